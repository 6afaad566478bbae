"""The CPU oracle restatement is pinned before it is trusted (CPU only).

* bitwise against the reference's own frozen golden vectors
  (proj/tests/golden/*.csv, test_golden.cpp:39-72), carried in
  tests/golden/golden_ref.json;
* bitwise against the reference library's dense_oracle on bf16-rounded inputs
  (fixtures made by tests/golden/make_golden.py from oracle/_ref);
* live against oracle/_ref when the reference is present in this container;
* the reference's known-answer tests (test_core.cpp:99-167).
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_ref.json")


def _doc():
    with open(GOLDEN) as f:
        return json.load(f)


def _unhex(rows):
    return np.array([[float.fromhex(v) for v in row] for row in rows], np.float64)


@pytest.mark.parametrize("stem,pattern", [("allgather", O.AG), ("reducescatter", O.RS)])
def test_oracle_reproduces_reference_golden_csv_bitwise(stem, pattern):
    g = _doc()["reference_csv"][stem]
    m, n, k, tp, seed = g["m"], g["n"], g["k"], g["tp"], g["seed"]
    a, b = zip(*[O.rank_inputs(pattern, m, n, k, tp, seed, r, round_bf16=False) for r in range(tp)])
    outs = O.dense_oracle(pattern, m, n, k, tp, a, b)
    for r in range(tp):
        want = _unhex(g["outputs"][r])
        assert outs[r].shape == want.shape
        assert np.array_equal(outs[r], want), f"rank {r}"


def test_oracle_matches_reference_on_bf16_inputs_bitwise():
    for case in _doc()["bf16_cases"]:
        pat, m, n, k, tp, seed = (case[x] for x in ("pattern", "m", "n", "k", "tp", "seed"))
        a, b = zip(*[O.rank_inputs(pat, m, n, k, tp, seed, r, round_bf16=True) for r in range(tp)])
        outs = O.dense_oracle(pat, m, n, k, tp, a, b)
        for r in range(tp):
            assert np.array_equal(outs[r], _unhex(case["outputs"][r])), (case["m"], case["pattern"], r)


def test_bits_and_doubles_streams_agree():
    """The bf16 bit stream uploaded to the GPU is exactly the oracle's rounded input."""
    for pat in (O.AG, O.RS):
        m, n, k, tp = 32, 48, 40, 4 if pat == O.AG else 4
        for r in range(tp):
            a, b = O.rank_inputs(pat, m, n, k, tp, 5, r, round_bf16=True)
            abits, btbits = O.rank_inputs_bits(pat, m, n, k, tp, 5, r)
            assert np.array_equal(O.bits_to_f64(abits), a)
            assert np.array_equal(O.bits_to_f64(btbits).T, b)


def test_bf16_rounding_is_round_to_nearest_even():
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-1, 1, 20000), [0.0, -0.0, 1.0, -1.0, 1e-30, 2.0 ** -130]])
    # exact ties between adjacent bf16 values at several exponents
    for e in (-3, -1, 0):
        base = 2.0 ** e
        ulp = base * 2.0 ** -7
        xs = np.concatenate([xs, base + ulp * (np.arange(8) + 0.5)])
    got = O.round_bf16(xs)
    # reference rounding: exact rational RNE computed with integer arithmetic on the double
    import math
    for x, g in zip(xs, got):
        if x == 0:
            assert g == 0
            continue
        mant, ex = math.frexp(abs(x))  # x = mant * 2^ex, mant in [0.5, 1)
        scaled = mant * 256  # 8 significant bits
        lo = math.floor(scaled)
        frac = scaled - lo
        if frac > 0.5 or (frac == 0.5 and lo % 2 == 1):
            lo += 1
        want = math.copysign(math.ldexp(lo / 256, ex), x)
        if abs(x) < 2.0 ** -126:  # bf16 subnormals: not produced by the Rng stream
            continue
        assert g == want, (x, g, want)


def test_known_answer_identity_and_twos():
    """test_core.cpp:99-133: identity product; all-twos reduce-scatter."""
    m = 4
    eye = np.eye(m)
    out = O.dense_oracle(O.AG, m, m, m, 1, [eye], [eye])
    assert np.array_equal(out[0], eye)
    # tp=2 RS: both partials all-ones [4,4] (A = ones[4,1], B = ones[1,4] with k/tp=1)
    ones_a = np.ones((4, 1))
    ones_b = np.ones((1, 4))
    outs = O.dense_oracle(O.RS, 4, 4, 2, 2, [ones_a, ones_a], [ones_b, ones_b])
    for o in outs:
        assert o.shape == (2, 4)
        assert np.all(o == 2.0)


def test_tp1_is_plain_matmul_and_mass_conservation():
    """test_core.cpp:135-167."""
    a, b = O.rank_inputs(O.AG, 8, 6, 5, 1, 9, 0, round_bf16=True)
    assert np.allclose(O.dense_oracle(O.AG, 8, 6, 5, 1, [a], [b])[0], a @ b, rtol=0, atol=1e-12)
    m, n, k, tp = 8, 6, 8, 4
    a, b = zip(*[O.rank_inputs(O.RS, m, n, k, tp, 9, r, round_bf16=True) for r in range(tp)])
    outs = O.dense_oracle(O.RS, m, n, k, tp, a, b)
    total = sum(x @ y for x, y in zip(a, b))
    assert np.isclose(sum(o.sum() for o in outs), total.sum(), rtol=0, atol=1e-9)


def test_row_sampled_oracle_equals_dense():
    m, n, k, tp = 32, 16, 24, 4
    a, b = zip(*[O.rank_inputs(O.AG, m, n, k, tp, 2, r, True) for r in range(tp)])
    dense = O.dense_oracle(O.AG, m, n, k, tp, a, b)
    rows = [0, 7, 8, 31]
    assert np.array_equal(O.ag_rows(m, n, k, tp, a, b[2], rows), dense[2][rows])
    a, b = zip(*[O.rank_inputs(O.RS, m, n, k, tp, 2, r, True) for r in range(tp)])
    dense = O.dense_oracle(O.RS, m, n, k, tp, a, b)
    assert np.array_equal(O.rs_rows(m, n, k, tp, a, b, 3, [0, 5, 7]), dense[3][[0, 5, 7]])


def test_max_rel_error_floor():
    """matrix.cpp:11-25: denominator floored at 1 (test_core.cpp metric floor)."""
    assert O.max_rel_error(np.array([0.0, 10.0]), np.array([0.5, 11.0])) == pytest.approx(0.5)
    assert O.max_rel_error(np.array([1e-9]), np.array([2e-9])) == pytest.approx(1e-9)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref needs /root/reference (build container only)")
def test_oracle_matches_live_reference_random_cases():
    rng = np.random.default_rng(42)
    for i in range(40):
        pat = i % 2
        tp = int(rng.choice([1, 2, 4, 8]))
        rpr = int(rng.integers(1, 5)) * 2
        m = rpr * tp
        if pat == O.AG:
            n = int(rng.integers(1, 5)) * tp
            k = int(rng.integers(1, 24))
        else:
            n = int(rng.integers(1, 7))
            k = tp * int(rng.integers(1, 7))
        seed = 100 + i
        a, b = zip(*[O.rank_inputs(pat, m, n, k, tp, seed, r, True) for r in range(tp)])
        ours = O.dense_oracle(pat, m, n, k, tp, a, b)
        ref = O.ref_dense_oracle(pat, m, n, k, tp, seed, round_bf16=True)
        for x, y in zip(ours, ref):
            assert np.array_equal(x, y)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref needs /root/reference (build container only)")
def test_reference_fused_engine_is_bitwise_equal_to_its_oracle():
    """The reference's own claim (test_golden.cpp:53-66), checked here because the
    CPU baseline times that engine."""
    for which, pat in ((O.FUSED_AG, O.AG), (O.FUSED_RS, O.RS), (O.NONOVERLAP, O.RS)):
        _, outs = O.ref_run(which, pat, 32, 16, 16, 4, 42, True, tm=2, tn=2, rpct=4)
        ref = O.ref_dense_oracle(pat, 32, 16, 16, 4, 42, round_bf16=True)
        for x, y in zip(outs, ref):
            assert np.array_equal(x, y)
