"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes access to the CPU checker:
  * liboracle.so      — plain-C restatement of the reference's oracle
                        (flux_oracle.c; Rng, bf16 rounding, dense/row-sampled
                        oracle, max_rel_error).
  * _ref/libref.so    — the reference itself compiled from /root/reference
                        (oracle/Makefile), used to pin the restatement and as
                        bench.py's "reference" CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")
REFERENCE_DIR = "/root/reference/proj"

AG, RS = 0, 1
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u16p = C.POINTER(C.c_uint16)
ROUND_FN = C.CFUNCTYPE(C.c_double, C.c_double)


def build(ref: bool | None = None) -> None:
    """make -C oracle (liboracle.so always; _ref only where /root/reference exists)."""
    targets = ["liboracle.so"]
    if ref is None:
        ref = os.path.isdir(REFERENCE_DIR)
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_orc = None
_ref = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        l = C.CDLL(ORACLE_SO)
        l.orc_round_bf16.restype = C.c_double
        l.orc_round_bf16.argtypes = [C.c_double]
        l.orc_bf16_bits.restype = C.c_uint16
        l.orc_bf16_bits.argtypes = [C.c_double]
        l.orc_fill_rank.restype = None
        l.orc_fill_rank.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_int, C.c_int, _dp, _dp]
        l.orc_fill_rank_bits.restype = None
        l.orc_fill_rank_bits.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_int, _u16p, _u16p]
        l.orc_bits_to_double.restype = None
        l.orc_bits_to_double.argtypes = [_u16p, _dp, C.c_size_t]
        l.orc_ag_rank.restype = None
        l.orc_ag_rank.argtypes = [C.c_int] * 4 + [C.POINTER(_dp), _dp, _dp, C.c_int, C.c_int]
        l.orc_rs_rows.restype = None
        l.orc_rs_rows.argtypes = [C.c_int] * 4 + [C.POINTER(_dp), C.POINTER(_dp), C.c_int, C.c_int, C.c_int, _dp, _dp]
        l.orc_max_rel_error.restype = C.c_double
        l.orc_max_rel_error.argtypes = [_dp, _dp, C.c_size_t]
        l.orc_normwise_error.restype = C.c_double
        l.orc_normwise_error.argtypes = [_dp, _dp, C.c_size_t]
        _orc = l
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference; `make -C oracle ref`)")
        l = C.CDLL(REF_SO)
        l.ref_dense_oracle.restype = C.c_int
        l.ref_dense_oracle.argtypes = [C.c_int] * 5 + [C.c_uint64, ROUND_FN, _dp]
        l.ref_run.restype = C.c_double
        l.ref_run.argtypes = [C.c_int] * 6 + [C.c_uint64, ROUND_FN] + [C.c_int] * 7 + [_dp]
        l.ref_tile_order.restype = C.c_int
        l.ref_tile_order.argtypes = [C.c_int] * 10 + [_ip, C.c_int, _ip, _ip]
        l.ref_comm_spec.restype = C.c_int
        l.ref_comm_spec.argtypes = [C.c_int] * 8 + [_ip, _ip, _ip, C.c_int]
        _ref = l
    return _ref


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# inputs (workspace.cpp:5-29 Rng stream)
# ---------------------------------------------------------------------------
def shapes(pattern: int, m: int, n: int, k: int, tp: int):
    """Reference layouts: (A shard rows, cols), (B shard rows, cols)."""
    if pattern == AG:
        return (m // tp, k), (k, n // tp)
    return (m, k // tp), (k // tp, n)


def rank_inputs(pattern: int, m: int, n: int, k: int, tp: int, seed: int, rank: int, round_bf16: bool = True):
    """Rank `rank`'s (A, B) in the reference layout as float64 arrays."""
    sa, sb = shapes(pattern, m, n, k, tp)
    a = np.empty(sa, np.float64)
    b = np.empty(sb, np.float64)
    orc().orc_fill_rank(pattern, m, n, k, tp, seed, rank, int(round_bf16), _ptr(a), _ptr(b))
    return a, b


def rank_inputs_bits(pattern: int, m: int, n: int, k: int, tp: int, seed: int, rank: int):
    """bf16 bit patterns in the device layout: A [rows, kk], B^T [cols, kk]."""
    sa, sb = shapes(pattern, m, n, k, tp)
    a = np.empty(sa, np.uint16)
    bt = np.empty((sb[1], sb[0]), np.uint16)
    orc().orc_fill_rank_bits(pattern, m, n, k, tp, seed, rank, _ptr(a, _u16p), _ptr(bt, _u16p))
    return a, bt


def bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def round_bf16(x: np.ndarray) -> np.ndarray:
    f = np.vectorize(orc().orc_round_bf16, otypes=[np.float64])
    return f(x)


# ---------------------------------------------------------------------------
# oracle outputs
# ---------------------------------------------------------------------------
def dense_oracle(pattern: int, m: int, n: int, k: int, tp: int, a_list, b_list):
    """dense_oracle (oracle.cpp:28-62) over explicit per-rank inputs (reference layout)."""
    a_list = [np.ascontiguousarray(a, np.float64) for a in a_list]
    b_list = [np.ascontiguousarray(b, np.float64) for b in b_list]
    ap = (_dp * tp)(*[_ptr(a) for a in a_list])
    outs = []
    if pattern == AG:
        for r in range(tp):
            o = np.empty((m, n // tp), np.float64)
            orc().orc_ag_rank(m, n, k, tp, ap, _ptr(b_list[r]), _ptr(o), 0, m)
            outs.append(o)
    else:
        bp = (_dp * tp)(*[_ptr(b) for b in b_list])
        scratch = np.empty(n, np.float64)
        for r in range(tp):
            o = np.empty((m // tp, n), np.float64)
            orc().orc_rs_rows(m, n, k, tp, ap, bp, r, 0, m // tp, _ptr(o), _ptr(scratch))
            outs.append(o)
    return outs


def ag_rows(m, n, k, tp, a_list, b_rank, rows):
    """Selected output rows of one AG rank (row-sampled parity at full size)."""
    a_list = [np.ascontiguousarray(a, np.float64) for a in a_list]
    ap = (_dp * tp)(*[_ptr(a) for a in a_list])
    b = np.ascontiguousarray(b_rank, np.float64)
    out = np.empty((len(rows), n // tp), np.float64)
    for i, r in enumerate(rows):
        orc().orc_ag_rank(m, n, k, tp, ap, _ptr(b), _ptr(out[i:i + 1]), int(r), 1)
    return out


def rs_rows(m, n, k, tp, a_list, b_list, owner, lrows):
    a_list = [np.ascontiguousarray(a, np.float64) for a in a_list]
    b_list = [np.ascontiguousarray(b, np.float64) for b in b_list]
    ap = (_dp * tp)(*[_ptr(a) for a in a_list])
    bp = (_dp * tp)(*[_ptr(b) for b in b_list])
    scratch = np.empty(n, np.float64)
    out = np.empty((len(lrows), n), np.float64)
    for i, r in enumerate(lrows):
        orc().orc_rs_rows(m, n, k, tp, ap, bp, owner, int(r), 1, _ptr(out[i:i + 1]), _ptr(scratch))
    return out


def max_rel_error(a: np.ndarray, b: np.ndarray) -> float:
    """max |a-b| / max(1,|a|,|b|) (matrix.cpp:11-25)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    return float(orc().orc_max_rel_error(_ptr(a), _ptr(b), a.size))


def normwise_error(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return float(orc().orc_normwise_error(_ptr(a), _ptr(b), a.size))


# ---------------------------------------------------------------------------
# the reference itself (oracle/_ref)
# ---------------------------------------------------------------------------
_ROUND_CB = None


def _round_cb():
    """The C rounding function itself (no Python in the per-element path)."""
    global _ROUND_CB
    if _ROUND_CB is None:
        _ROUND_CB = ROUND_FN(("orc_round_bf16", orc()))
    return _ROUND_CB


def _null_round():
    return C.cast(None, ROUND_FN)


def out_sizes(pattern, m, n, k, tp):
    return [(m, n // tp)] * tp if pattern == AG else [(m // tp, n)] * tp


def _split(flat, pattern, m, n, k, tp):
    outs, off = [], 0
    for (r, c) in out_sizes(pattern, m, n, k, tp):
        outs.append(flat[off:off + r * c].reshape(r, c))
        off += r * c
    return outs


def ref_dense_oracle(pattern, m, n, k, tp, seed, round_bf16=False):
    tot = sum(r * c for r, c in out_sizes(pattern, m, n, k, tp))
    flat = np.empty(tot, np.float64)
    rc = ref().ref_dense_oracle(pattern, m, n, k, tp, seed, _round_cb() if round_bf16 else _null_round(), _ptr(flat))
    if rc != 0:
        raise RuntimeError("reference dense_oracle failed")
    return _split(flat, pattern, m, n, k, tp)


FUSED_AG, FUSED_RS, NONOVERLAP = 0, 1, 2


def ref_run(which, pattern, m, n, k, tp, seed, round_bf16=False, tm=1, tn=1, rpct=0, transfer=0, write_mode=0,
            swizzle=True, workers=0, want_outputs=True):
    """Runs the reference engine; returns (seconds, outputs or None)."""
    rpct = rpct or m // tp
    flat = None
    if want_outputs:
        flat = np.empty(sum(r * c for r, c in out_sizes(pattern, m, n, k, tp)), np.float64)
    secs = ref().ref_run(which, pattern, m, n, k, tp, seed, _round_cb() if round_bf16 else _null_round(), tm, tn,
                         rpct, transfer, write_mode, int(swizzle), workers,
                         _ptr(flat) if flat is not None else C.cast(None, _dp))
    if secs < 0:
        raise RuntimeError("reference engine failed")
    return secs, (_split(flat, pattern, m, n, k, tp) if flat is not None else None)


def ref_tile_order(pattern, m, n, k, tp, tm, tn, kind, rank, shift=1, arrival=None):
    cnt = (m // tm) * ((n // tp if pattern == AG else n) // tn)
    rows, cols = (C.c_int * cnt)(), (C.c_int * cnt)()
    arr = (C.c_int * len(arrival))(*arrival) if arrival else None
    got = ref().ref_tile_order(pattern, m, n, k, tp, tm, tn, kind, rank, shift, arr, len(arrival or []), rows, cols)
    if got < 0:
        raise RuntimeError("reference tile_order raised")
    return list(zip(rows, cols))


def ref_comm_spec(pattern, m, n, k, tp, rank, rpct, transfer):
    cap = max(1, m)
    p, b, r = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)()
    got = ref().ref_comm_spec(pattern, m, n, k, tp, rank, rpct, transfer, p, b, r, cap)
    if got < 0:
        raise RuntimeError("reference make_comm_specs raised")
    return [(p[i], b[i], r[i]) for i in range(got)]
