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
    """One rank of a multi-process AllGather-GEMM: NCCL all-gather + cuBLAS (B1),
    and the decomposed B2: per-chunk NCCL broadcasts from each chunk's owner,
    issued asynchronously up front, each chunk's cuBLAS GEMM waiting only for
    its own chunk (run_medium_grained, engine.cpp:653-728, partitions = tp).
    host_collectives: stage through host tensors (gloo plumbing when the ranks
    share one GPU in tests; no timing meaning)."""

    def __init__(self, shard, weight, group=None, host_collectives=False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.host = host_collectives
        self.tp = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.shard, self.weight = shard, weight
        self.rpr = shard.shape[0]
        self.gathered = torch.empty(shard.shape[0] * self.tp, shard.shape[1], dtype=shard.dtype, device=shard.device)
        self.out = torch.empty(self.gathered.shape[0], weight.shape[0], dtype=shard.dtype, device=shard.device)

    def gemm_only(self):
        torch.matmul(self.gathered, self.weight.t(), out=self.out)

    def _all_gather(self):
        if self.host:
            parts = [torch.empty_like(self.shard, device="cpu") for _ in range(self.tp)]
            self.dist.all_gather(parts, self.shard.cpu(), group=self.group)
            self.gathered.copy_(torch.cat(parts).to(self.gathered.device))
        else:
            self.dist.all_gather_into_tensor(self.gathered, self.shard, group=self.group)

    def unfused(self):
        self._all_gather()
        self.gemm_only()

    def decomposed(self):
        if self.host:
            self.unfused()
            return
        self.gathered[self.rank * self.rpr:(self.rank + 1) * self.rpr].copy_(self.shard)
        works = []
        for c in range(self.tp):
            chunk = self.gathered[c * self.rpr:(c + 1) * self.rpr]
            works.append(self.dist.broadcast(chunk, src=c, group=self.group, async_op=True))
        for c in range(self.tp):
            works[c].wait()  # the compute stream waits for chunk c only
            rows = slice(c * self.rpr, (c + 1) * self.rpr)
            torch.matmul(self.gathered[rows], self.weight.t(), out=self.out[rows])


class DistRS:
    """One rank of a multi-process GEMM-ReduceScatter: cuBLAS + NCCL
    reduce-scatter (B1), and the decomposed B2: per-chunk cuBLAS GEMMs whose
    bf16 partial chunks are reduced to their owner asynchronously while the
    next chunk computes (run_medium_grained, engine.cpp:653-728)."""

    def __init__(self, a, weight, group=None, host_collectives=False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.host = host_collectives
        self.tp = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.a, self.w = a, weight
        self.rpr = a.shape[0] // self.tp
        self.partial = torch.empty(a.shape[0], weight.shape[0], dtype=a.dtype, device=a.device)
        self.out = torch.empty(a.shape[0] // self.tp, weight.shape[0], dtype=a.dtype, device=a.device)

    def gemm_only(self):
        torch.matmul(self.a, self.w.t(), out=self.partial)

    def unfused(self):
        self.gemm_only()
        if self.host:
            h = self.partial.float().cpu()
            self.dist.all_reduce(h, group=self.group)
            self.out.copy_(h[self.rank * self.rpr:(self.rank + 1) * self.rpr].to(self.out.device))
        else:
            self.dist.reduce_scatter_tensor(self.out, self.partial, group=self.group)

    def decomposed(self):
        if self.host:
            self.unfused()
            return
        works = []
        for c in range(self.tp):
            rows = slice(c * self.rpr, (c + 1) * self.rpr)
            torch.matmul(self.a[rows], self.w.t(), out=self.partial[rows])
            works.append(self.dist.reduce(self.partial[rows], dst=c, group=self.group, async_op=True))
        for w in works:
            w.wait()
        self.out.copy_(self.partial[self.rank * self.rpr:(self.rank + 1) * self.rpr])
