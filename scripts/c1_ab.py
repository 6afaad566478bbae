"""A/B of the C1 config (GEMM-RS M=N=K=1024, TP=2, ranks emulated on one GPU):
fused kernel time and the local GEMM, L2 flushed (write + read sweep) before
each launch; env knobs are read by the library at launch time."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06858_b200 as fx  # noqa: E402

p = fx.ProblemSpec(1024, 1024, 1024, 2, fx.GEMM_REDUCESCATTER)
comm = fx.Communicator(2, [0, 0], heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
cases = [("default", {}), ("no tail split", {"FLUX_TAIL_SPLIT": "0"}), ("no units", {"FLUX_RS_UNITS": "0"}),
         ("neither", {"FLUX_TAIL_SPLIT": "0", "FLUX_RS_UNITS": "0"}), ("cta_group 1", {"_cg": 1}),
         ("units warm-up", {"FLUX_DEBUG": "2048"}), ("warm-up cg1", {"FLUX_DEBUG": "2048", "_cg": 1})]
for name, env in cases:
    for k in ("FLUX_TAIL_SPLIT", "FLUX_RS_UNITS", "FLUX_DEBUG"):
        os.environ.pop(k, None)
    opts = fx.default_opts(cta_group=env.get("_cg", 0))
    for k, v in env.items():
        if not k.startswith("_"):
            os.environ[k] = v
    res = {}
    for what, fn in (("local", lambda: comm.local_gemm(p, opts, [s, s])),
                     ("fused", lambda: comm.gemm_rs(p, fx.TileShape(512, 1024), fx.WRITE_ALLTOALL, True, opts, [s, s]))):
        comm.set_timing(True)
        ts = []
        for i in range(15):
            flush.zero_()
            rd.max()
            fn()
            comm.sync()
            ts.append(comm.last_kernel_ms() * 1e3)
        res[what] = sorted(ts)[7]
    print(f"{name:14s} local {res['local']:6.1f} us  fused {res['fused']:6.1f} us", flush=True)
