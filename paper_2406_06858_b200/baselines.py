"""Library baselines the fused operators are measured against (NOT the product).

B1 "unfused" (reference run_nonoverlap, engine.cpp:558-605): the collective,
then the GEMM — cuBLAS (torch.matmul) for the GEMM and NCCL
(torch.distributed) for the collective when ranks are separate processes, or
device copies / adds when the ranks are emulated on one GPU.
B2 "decomposed" (reference run_medium_grained, engine.cpp:607-728, the
TransformerEngine-style chunked overlap): tp chunk GEMMs on the compute stream,
chunk transfers on a side stream, joined with events.
T_gemm (Eq. 1 "best non-split GEMM"): cuBLAS on the local shapes, no comm.
"""
from __future__ import annotations

import torch


class EmulatedAG:
    """tp ranks of an AllGather-GEMM on one device, torch-owned buffers."""

    def __init__(self, shards, weights):
        self.tp = len(shards)
        self.shards = shards                      # [rpr, k] per rank
        self.weights = weights                    # [n/tp, k] per rank (K-major)
        rpr, k = shards[0].shape
        self.rpr = rpr
        self.gathered = [torch.empty(rpr * self.tp, k, dtype=shards[0].dtype, device=shards[0].device)
                         for _ in range(self.tp)]
        self.out = [torch.empty(rpr * self.tp, w.shape[0], dtype=shards[0].dtype, device=w.device)
                    for w in weights]
        self.side = torch.cuda.Stream()

    def gemm_only(self):
        for r in range(self.tp):
            torch.matmul(self.gathered[r], self.weights[r].t(), out=self.out[r])

    def unfused(self):
        """B1: serial all-gather (rank order) then cuBLAS GEMM per rank."""
        for r in range(self.tp):
            for q in range(self.tp):
                self.gathered[r][q * self.rpr:(q + 1) * self.rpr].copy_(self.shards[q])
        self.gemm_only()

    def decomposed(self):
        """B2: per-chunk copies on a side stream overlapped with chunk GEMMs."""
        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        events = []
        with torch.cuda.stream(self.side):
            for step in range(self.tp):
                for r in range(self.tp):
                    q = (r + step) % self.tp
                    self.gathered[r][q * self.rpr:(q + 1) * self.rpr].copy_(self.shards[q])
                ev = torch.cuda.Event()
                ev.record(self.side)
                events.append(ev)
        for step in range(self.tp):
            cur.wait_event(events[step])
            for r in range(self.tp):
                q = (r + step) % self.tp
                rows = slice(q * self.rpr, (q + 1) * self.rpr)
                torch.matmul(self.gathered[r][rows], self.weights[r].t(), out=self.out[r][rows])


class EmulatedRS:
    """tp ranks of a GEMM-ReduceScatter on one device."""

    def __init__(self, a_shards, weights):
        self.tp = len(a_shards)
        self.a = a_shards                          # [m, k/tp]
        self.w = weights                           # [n, k/tp]
        m = a_shards[0].shape[0]
        n = weights[0].shape[0]
        self.rpr = m // self.tp
        dev = a_shards[0].device
        self.partials = [torch.empty(m, n, dtype=torch.bfloat16, device=dev) for _ in range(self.tp)]
        self.out = [torch.empty(self.rpr, n, dtype=torch.bfloat16, device=dev) for _ in range(self.tp)]
        self.acc = torch.empty(self.rpr, n, dtype=torch.float32, device=dev)

    def gemm_only(self):
        for r in range(self.tp):
            torch.matmul(self.a[r], self.w[r].t(), out=self.partials[r])

    def unfused(self):
        """B1: GEMM, then the reduce-scatter in source order (bf16 partials, as NCCL)."""
        self.gemm_only()
        for d in range(self.tp):
            rows = slice(d * self.rpr, (d + 1) * self.rpr)
            self.acc.zero_()
            for s in range(self.tp):
                self.acc.add_(self.partials[s][rows])
            self.out[d].copy_(self.acc)


class DistAG:
    """One rank of a multi-process AllGather-GEMM: NCCL all-gather + cuBLAS."""

    def __init__(self, shard, weight, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.tp = dist.get_world_size(group)
        self.shard, self.weight = shard, weight
        self.gathered = torch.empty(shard.shape[0] * self.tp, shard.shape[1], dtype=shard.dtype, device=shard.device)
        self.out = torch.empty(self.gathered.shape[0], weight.shape[0], dtype=shard.dtype, device=shard.device)

    def gemm_only(self):
        torch.matmul(self.gathered, self.weight.t(), out=self.out)

    def unfused(self):
        self.dist.all_gather_into_tensor(self.gathered, self.shard, group=self.group)
        self.gemm_only()


class DistRS:
    """One rank of a multi-process GEMM-ReduceScatter: cuBLAS + NCCL reduce-scatter."""

    def __init__(self, a, weight, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.tp = dist.get_world_size(group)
        self.a, self.w = a, weight
        self.partial = torch.empty(a.shape[0], weight.shape[0], dtype=a.dtype, device=a.device)
        self.out = torch.empty(a.shape[0] // self.tp, weight.shape[0], dtype=a.dtype, device=a.device)

    def gemm_only(self):
        torch.matmul(self.a, self.w.t(), out=self.partial)

    def unfused(self):
        self.gemm_only()
        self.dist.reduce_scatter_tensor(self.out, self.partial, group=self.group)
