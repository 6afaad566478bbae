"""Regenerates tests/golden/golden_ref.json from the REFERENCE (run in the build
container, where /root/reference exists; the GPU box only reads the JSON).

Contents:
  * reference_csv   — the reference's own frozen goldens
                      (/root/reference/proj/tests/golden/*.csv, ProblemSpec{16,16,16,4},
                      seed 42, gen_golden.cpp:17-25), copied value-for-value as
                      hex floats.
  * bf16_cases      — dense_oracle outputs of the reference library itself
                      (oracle/_ref, oracle.cpp:28-62) on the same Rng stream with
                      every input rounded to bf16: what the B200 kernels must
                      reproduce within the bf16/fp32 tolerance.
  * tile_orders     — the reference's tile_order (swizzle.cpp:75-80) for all kinds.
  * comm_specs      — the reference's make_comm_specs (engine.cpp:77-99).

Usage:  make -C oracle && python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

REF_GOLDEN = "/root/reference/proj/tests/golden"
OUT = os.path.join(HERE, "golden_ref.json")

BF16_CASES = [
    # (pattern, m, n, k, tp, seed)
    (O.AG, 16, 16, 16, 4, 42),
    (O.RS, 16, 16, 16, 4, 42),
    (O.AG, 64, 96, 80, 2, 3),
    (O.RS, 64, 96, 80, 2, 3),
    (O.AG, 128, 64, 40, 8, 11),
    (O.RS, 128, 64, 40, 8, 11),
]

ORDER_CASES = [
    # (pattern, m, n, k, tp, tm, tn)
    (O.AG, 16, 16, 16, 4, 2, 2),
    (O.RS, 16, 16, 16, 4, 2, 2),
    (O.AG, 64, 64, 8, 8, 4, 2),
    (O.RS, 48, 12, 6, 3, 4, 3),
]

SPEC_CASES = [
    # (pattern, m, n, k, tp, rpct)
    (O.AG, 16, 16, 16, 4, 4),
    (O.AG, 16, 16, 16, 4, 2),
    (O.AG, 64, 64, 8, 8, 2),
    (O.AG, 24, 6, 6, 3, 4),
]


def hexlist(a: np.ndarray):
    return [[float(v).hex() for v in row] for row in a]


def main() -> None:
    doc = {"generated_by": "tests/golden/make_golden.py", "reference_csv": {}, "bf16_cases": [],
           "tile_orders": [], "comm_specs": []}
    for stem in ("allgather", "reducescatter"):
        ranks = []
        for r in range(4):
            m = np.loadtxt(os.path.join(REF_GOLDEN, f"{stem}_rank{r}.csv"), delimiter=",", ndmin=2)
            ranks.append(hexlist(m))
        doc["reference_csv"][stem] = {"m": 16, "n": 16, "k": 16, "tp": 4, "seed": 42, "outputs": ranks}
    for (pat, m, n, k, tp, seed) in BF16_CASES:
        outs = O.ref_dense_oracle(pat, m, n, k, tp, seed, round_bf16=True)
        doc["bf16_cases"].append({"pattern": pat, "m": m, "n": n, "k": k, "tp": tp, "seed": seed,
                                  "outputs": [hexlist(o) for o in outs]})
    for (pat, m, n, k, tp, tm, tn) in ORDER_CASES:
        for kind in (0, 1, 2):
            for rank in range(tp):
                for shift in ((1, 2) if kind == 1 else (1,)):
                    order = O.ref_tile_order(pat, m, n, k, tp, tm, tn, kind, rank, shift)
                    doc["tile_orders"].append({"pattern": pat, "m": m, "n": n, "k": k, "tp": tp, "tm": tm, "tn": tn,
                                               "kind": kind, "rank": rank, "shift": shift, "order": order})
    for (pat, m, n, k, tp, rpct) in SPEC_CASES:
        for transfer in (0, 1):
            for rank in range(tp):
                doc["comm_specs"].append({"pattern": pat, "m": m, "n": n, "k": k, "tp": tp, "rpct": rpct,
                                          "transfer": transfer, "rank": rank,
                                          "order": O.ref_comm_spec(pat, m, n, k, tp, rank, rpct, transfer)})
    with open(OUT, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
