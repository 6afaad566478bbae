"""Python host mirror of the communicator and the fused operators.

Thin object layer over the C ABI (include/flux_b200.h) with the reference's
vocabulary: a communicator owns every rank's symmetric buffers (the reference
ShardedWorkspace + peer directory, workspace.hpp:22-43) and runs
`run_fused_allgather_gemm` / `run_fused_gemm_reducescatter`
(engine.hpp:101-111) on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

from . import _native as N


@dataclass(frozen=True)
class ProblemSpec:
    """overlap::ProblemSpec (problem.hpp:22-38)."""

    m: int
    n: int
    k: int
    tp: int = 1
    pattern: int = N.ALLGATHER_GEMM

    def c(self) -> N.Problem:
        return N.Problem(self.m, self.n, self.k, self.tp, self.pattern)

    def validate(self) -> None:
        N.check(N.lib().flux_problem_validate(C.byref(self.c()), None))

    def rows_per_rank(self) -> int:
        return self.m // self.tp

    def local_cols(self) -> int:
        return self.n // self.tp if self.pattern == N.ALLGATHER_GEMM else self.n

    def local_k(self) -> int:
        return self.k // self.tp if self.pattern == N.GEMM_REDUCESCATTER else self.k

    def owner_of_row(self, row: int) -> int:
        return row // self.rows_per_rank()

    def flops(self) -> float:
        """Whole-job algorithmic FLOPs (all ranks)."""
        return 2.0 * self.m * self.n * self.k


@dataclass(frozen=True)
class TileShape:
    """overlap::TileShape (problem.hpp:40-43)."""

    tm: int
    tn: int

    def c(self) -> N.Tile:
        return N.Tile(self.tm, self.tn)


def validate_tiling(problem: ProblemSpec, tile: TileShape) -> None:
    N.check(N.lib().flux_problem_validate(C.byref(problem.c()), C.byref(tile.c())))


def grid_for(problem: ProblemSpec, tile: TileShape) -> tuple[int, int, int]:
    a, b, r = C.c_int(), C.c_int(), C.c_int()
    N.check(N.lib().flux_grid_for(C.byref(problem.c()), C.byref(tile.c()), C.byref(a), C.byref(b), C.byref(r)))
    return a.value, b.value, r.value


def tile_order(problem: ProblemSpec, tile: TileShape, kind: int, rank: int, shift_offset: int = 1,
               arrival_blocks: Optional[Sequence[int]] = None) -> list[tuple[int, int]]:
    """tile_order(SwizzlePolicy, grid) (swizzle.cpp:75-80) as (row, col) pairs."""
    rows, cols, _ = grid_for(problem, tile)
    n = rows * cols
    out_r, out_c = (C.c_int * n)(), (C.c_int * n)()
    arr = (C.c_int * len(arrival_blocks))(*arrival_blocks) if arrival_blocks else None
    N.check(N.lib().flux_tile_order(C.byref(problem.c()), C.byref(tile.c()), kind, rank, shift_offset, arr,
                                    len(arrival_blocks or []), out_r, out_c))
    return list(zip(out_r, out_c))


def comm_order(rank: int, tp: int, rows_per_rank: int, rows_per_comm_tile: int) -> list[tuple[int, int, int]]:
    """comm_order(Topology{NVLinkRing}, ...) (topology.cpp:102-168): (peer, row_begin, rows)."""
    cap = max(1, tp * max(1, rows_per_rank // max(1, rows_per_comm_tile)))
    p, b, r, n = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)(), C.c_int()
    N.check(N.lib().flux_comm_order(rank, tp, rows_per_rank, rows_per_comm_tile, p, b, r, cap, C.byref(n)))
    return [(p[i], b[i], r[i]) for i in range(n.value)]


def make_comm_spec(problem: ProblemSpec, rank: int, rows_per_comm_tile: int, transfer: int) -> list[tuple[int, int, int]]:
    """make_comm_specs(...)[rank].order (engine.cpp:77-99), validated."""
    cap = max(1, problem.m)
    p, b, r, n = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)(), C.c_int()
    N.check(N.lib().flux_make_comm_spec(C.byref(problem.c()), rank, rows_per_comm_tile, transfer, p, b, r, cap,
                                        C.byref(n)))
    return [(p[i], b[i], r[i]) for i in range(n.value)]


class _CAI:
    """__cuda_array_interface__ holder so torch can view a library buffer."""

    def __init__(self, ptr: int, rows: int, cols: int, ld: int, typestr: str, esize: int):
        self.__cuda_array_interface__ = {
            "shape": (rows, cols), "strides": (ld * esize, esize), "typestr": typestr,
            "data": (ptr, False), "version": 3,
        }


def _mat(t) -> N.Matrix:
    if t is None:
        return N.Matrix(None, 0)
    assert t.dim() == 2 and t.stride(1) == 1, "operands must be row-major 2-D views"
    return N.Matrix(t.data_ptr(), t.stride(0))


def _operands(per_rank):
    """Per rank (a, b, c) or (a, b, c, aux) tensors (None = library buffer)."""
    arr = (N.Operands * len(per_rank))()
    for i, abc in enumerate(per_rank):
        t = tuple(abc) if abc is not None else (None, None, None)
        a, b, c = t[:3]
        aux = t[3] if len(t) > 3 else None
        arr[i] = N.Operands(_mat(a), _mat(b), _mat(c), _mat(aux))
    return arr


@dataclass(frozen=True)
class MlpSpec:
    """Chained tensor-parallel MLP (flux_mlp): x [m/tp, hidden] -> AG-GEMM with
    W_up + activation -> GEMM-RS with W_down -> out [m/tp, hidden]."""
    m: int
    hidden: int
    ffn: int
    tp: int
    activation: int = N.ACT_GELU

    def c(self) -> N.Mlp:
        return N.Mlp(self.m, self.hidden, self.ffn, self.tp, self.activation)

    def required_heap_bytes(self) -> int:
        return int(N.lib().flux_mlp_required_heap_bytes(C.byref(self.c())))


class Communicator:
    """Symmetric-heap communicator over `tp` ranks.

    Single-process mode: rank r lives on devices[r] (devices may repeat: ranks
    emulated on one GPU). IPC mode: one process per GPU, see `Communicator.ipc`.
    """

    def __init__(self, tp: int, devices: Optional[Sequence[int]] = None, heap_bytes: int = 0, *, _handle=None,
                 device: Optional[int] = None, nvls_bytes: int = 0):
        self.tp = tp
        self._h = C.c_void_p(_handle) if _handle is not None else C.c_void_p()
        if _handle is None:
            devs = (C.c_int * tp)(*(devices if devices is not None else [0] * tp))
            N.check(N.lib().flux_comm_create(tp, devs, C.byref(N.CommOpts(heap_bytes, nvls_bytes)), C.byref(self._h)))
        self.rank = N.lib().flux_comm_rank(self._h)
        # Device of every rank this process drives, and the device this process
        # drives when it is a single one (IPC mode, or every rank on one GPU).
        devs_l = list(devices) if devices is not None else [device if device is not None else 0] * tp
        self.devices = devs_l
        self.device = device if device is not None else (devs_l[0] if len(set(devs_l)) == 1 else None)

    @classmethod
    def ipc(cls, rank: int, tp: int, device: int, heap_bytes: int,
            all_gather_bytes: Callable[[bytes], list[bytes]], nvls_bytes: int = 0) -> "Communicator":
        """Multi-process constructor: `all_gather_bytes` exchanges handle blobs
        (e.g. torch.distributed.all_gather_object), the paper's init-phase IPC
        exchange. `nvls_bytes` > 0 also sets up the NVLS
        multicast region (rank 0's multicast handle reaches the peers as a file
        descriptor over a Unix socket); every rank raises the same error if the
        host does not expose it."""
        h = C.c_void_p()
        N.check(N.lib().flux_comm_create_ipc(rank, tp, device, C.byref(N.CommOpts(heap_bytes, 0)), C.byref(h)))
        nb = N.lib().flux_comm_ipc_blob_bytes()
        blob = C.create_string_buffer(nb)
        N.check(N.lib().flux_comm_ipc_handle(h, blob))
        blobs = all_gather_bytes(blob.raw)
        joined = C.create_string_buffer(b"".join(blobs), nb * tp)
        N.check(N.lib().flux_comm_ipc_connect(h, joined))
        comm = cls(tp, _handle=h.value, device=device)
        if nvls_bytes:
            try:
                comm._nvls_ipc_setup(rank, tp, nvls_bytes, all_gather_bytes)
            except Exception:
                comm.close()
                raise
        return comm

    def _nvls_ipc_setup(self, rank: int, tp: int, nvls_bytes: int, all_gather_bytes) -> None:
        """Every step ends with an exchange of per-rank status, so a failure on
        any rank raises the same error on all of them (nobody waits forever)."""
        lib = N.lib()

        def agree(status: bytes, payload: bytes = b"") -> list[bytes]:
            got = all_gather_bytes(status + b"\0" + payload)
            for r, g in enumerate(got):
                st = g.split(b"\0", 1)[0]
                if st != b"ok":
                    raise N.CudaError(f"rank {r}: " + st.decode(errors="replace"))
            return [g.split(b"\0", 1)[1] for g in got]

        status, server, name = b"ok", None, b""
        if rank == 0:
            fd = C.c_int(-1)
            try:
                if lib.flux_comm_nvls_ipc_export(self._h, nvls_bytes, C.byref(fd)) != N.OK:
                    status = lib.flux_last_error()
                else:
                    name = ("flux-nvls-%d-%s" % (os.getpid(), os.urandom(6).hex())).encode()
                    server = fd_server(name.decode(), fd.value)  # listening before the peers learn the name
            except OSError as e:
                status = ("fd hand-off socket: %s" % e).encode()
                if fd.value >= 0 and server is None:
                    os.close(fd.value)
        name0 = agree(status, name)[0]
        status = b"ok"
        try:
            if rank == 0:
                server.serve(tp - 1)
            else:
                fd = fd_receive(name0.decode())
                if lib.flux_comm_nvls_ipc_import(self._h, nvls_bytes, fd) != N.OK:
                    status = lib.flux_last_error()
            if status == b"ok" and lib.flux_comm_nvls_ipc_add_device(self._h) != N.OK:
                status = lib.flux_last_error()
        except OSError as e:
            status = ("fd hand-off: %s" % e).encode()
        agree(status)  # every GPU is in the object before anyone binds
        status = b"ok" if lib.flux_comm_nvls_ipc_bind(self._h) == N.OK else lib.flux_last_error()
        agree(status)  # every region mapped and zeroed before the first operator

    # ---- buffers -------------------------------------------------------------
    def buffer(self, rank: int, kind: int, problem: ProblemSpec) -> N.BufferDesc:
        d = N.BufferDesc()
        N.check(N.lib().flux_buffer(self._h, rank, kind, C.byref(problem.c()), C.byref(d)))
        return d

    def tensor(self, rank: int, kind: int, problem: ProblemSpec):
        """torch view (no copy) of a rank's buffer: bf16 or fp32, strided by the padded pitch."""
        import torch

        d = self.buffer(rank, kind, problem)
        dev = torch.device("cuda", self.devices[rank] if rank < len(self.devices) else 0)
        if d.dtype == N.F32:
            return torch.as_tensor(_CAI(d.ptr, d.rows, d.cols, d.ld, "<f4", 4), device=dev)
        t = torch.as_tensor(_CAI(d.ptr, d.rows, d.cols, d.ld, "<i2", 2), device=dev)
        return t.view(torch.bfloat16)

    def copy_in(self, rank: int, kind: int, problem: ProblemSpec, host_ptr: int, host_ld: int, stream=None):
        N.check(N.lib().flux_copy_in(self._h, rank, kind, C.byref(problem.c()), C.c_void_p(host_ptr), host_ld,
                                     C.c_void_p(stream) if stream else None))

    def copy_out(self, rank: int, kind: int, problem: ProblemSpec, host_ptr: int, host_ld: int, stream=None):
        N.check(N.lib().flux_copy_out(self._h, rank, kind, C.byref(problem.c()), C.c_void_p(host_ptr), host_ld,
                                      C.c_void_p(stream) if stream else None))

    # ---- operators -------------------------------------------------------------
    def ag_gemm(self, problem: ProblemSpec, tile: TileShape, rows_per_comm_tile: int = 0, transfer: int = N.PULL,
                swizzle: bool = True, opts: Optional[N.Opts] = None, streams=None) -> None:
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_ag_gemm(self._h, C.byref(problem.c()), C.byref(tile.c()), rows_per_comm_tile,
                                     transfer, int(swizzle), C.byref(o), N.stream_array(streams)))

    def ag_gemm_ex(self, problem: ProblemSpec, tile: TileShape, operands, rows_per_comm_tile: int = 0,
                   transfer: int = N.PULL, swizzle: bool = True, opts: Optional[N.Opts] = None, streams=None) -> None:
        """ag_gemm on caller-owned operands: `operands` is a list (one per rank
        this process drives) of (a, b, c) tensors or None (library buffer)."""
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_ag_gemm_ex(self._h, C.byref(problem.c()), C.byref(tile.c()), rows_per_comm_tile, transfer,
                                        int(swizzle), C.byref(o), N.stream_array(streams), _operands(operands)))

    def ag_gemm_ordered(self, problem: ProblemSpec, tile: TileShape, orders, rows_per_comm_tile: int,
                        transfer: int = N.PULL, swizzle: bool = True, opts: Optional[N.Opts] = None, streams=None,
                        operands=None) -> None:
        """run_fused_allgather_gemm with the caller's comm specs: `orders` holds,
        for every rank this process drives, its (peer, row_begin, rows) list."""
        o = opts if opts is not None else N.default_opts()
        count = len(orders[0]) if orders else 0
        flat = [d for order in orders for d in order]
        if any(len(order) != count for order in orders):
            raise N.ConfigError("all ranks' comm orders must have the same length")
        peer = (C.c_int * max(1, len(flat)))(*[d[0] for d in flat])
        begin = (C.c_int * max(1, len(flat)))(*[d[1] for d in flat])
        rows = (C.c_int * max(1, len(flat)))(*[d[2] for d in flat])
        N.check(N.lib().flux_ag_gemm_ordered(self._h, C.byref(problem.c()), C.byref(tile.c()), rows_per_comm_tile,
                                             transfer, int(swizzle), C.byref(o), N.stream_array(streams),
                                             _operands(operands) if operands else None, peer, begin, rows, count))

    def transfer_log(self, rank: int) -> list[dict]:
        """TransferRecords of the last traced copy-engine AllGather (flux_transfer_log)."""
        n = C.c_int()
        N.check(N.lib().flux_transfer_log(self._h, rank, None, 0, C.byref(n)))
        recs = (N.TransferRecord * max(1, n.value))()
        N.check(N.lib().flux_transfer_log(self._h, rank, recs, n.value, C.byref(n)))
        return [{"peer": r.peer, "row_begin": r.row_begin, "rows": r.rows, "copy_done_ns": r.copy_done_ns,
                 "flag_set_ns": r.flag_set_ns} for r in recs[:n.value]]

    def gemm_rs_ex(self, problem: ProblemSpec, tile: TileShape, operands, write_mode: int = N.WRITE_ALLTOALL,
                   swizzle: bool = True, opts: Optional[N.Opts] = None, streams=None) -> None:
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_gemm_rs_ex(self._h, C.byref(problem.c()), C.byref(tile.c()), write_mode, int(swizzle),
                                        C.byref(o), N.stream_array(streams), _operands(operands)))

    def gemm_rs(self, problem: ProblemSpec, tile: TileShape, write_mode: int = N.WRITE_ALLTOALL,
                swizzle: bool = True, opts: Optional[N.Opts] = None, streams=None) -> None:
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_gemm_rs(self._h, C.byref(problem.c()), C.byref(tile.c()), write_mode, int(swizzle),
                                     C.byref(o), N.stream_array(streams)))

    def mlp_forward(self, mlp: MlpSpec, operands, opts: Optional[N.Opts] = None, streams=None) -> None:
        """Per rank a dict with x, w_up, w_down, act, out (and optional pre)."""
        arr = (N.MlpOperands * len(operands))()
        for i, d in enumerate(operands):
            arr[i] = N.MlpOperands(*[_mat(d.get(k)) for k in ("x", "w_up", "w_down", "pre", "act", "out")])
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_mlp_forward(self._h, C.byref(mlp.c()), C.byref(o), N.stream_array(streams), arr))

    def mlp_backward_dx(self, mlp: MlpSpec, operands, opts: Optional[N.Opts] = None, streams=None) -> None:
        """Per rank a dict with dout, w_down_t, w_up_t, pre, dact, dx."""
        arr = (N.MlpGradOperands * len(operands))()
        for i, d in enumerate(operands):
            arr[i] = N.MlpGradOperands(*[_mat(d.get(k)) for k in ("dout", "w_down_t", "w_up_t", "pre", "dact", "dx")])
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_mlp_backward_dx(self._h, C.byref(mlp.c()), C.byref(o), N.stream_array(streams), arr))

    def local_gemm(self, problem: ProblemSpec, opts: Optional[N.Opts] = None, streams=None) -> None:
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_local_gemm(self._h, C.byref(problem.c()), C.byref(o), N.stream_array(streams)))

    def nonoverlap(self, problem: ProblemSpec, opts: Optional[N.Opts] = None, streams=None) -> None:
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_nonoverlap(self._h, C.byref(problem.c()), C.byref(o), N.stream_array(streams)))

    def medium_grained(self, problem: ProblemSpec, tile: TileShape, partitions: int, opts: Optional[N.Opts] = None,
                       streams=None) -> None:
        """run_medium_grained (engine.hpp:144-145): the decomposed (B2) baseline on the device."""
        o = opts if opts is not None else N.default_opts()
        N.check(N.lib().flux_medium_grained(self._h, C.byref(problem.c()), C.byref(tile.c()), partitions, C.byref(o),
                                            N.stream_array(streams)))

    def sync(self) -> None:
        N.check(N.lib().flux_sync(self._h))

    def last_launch_count(self) -> int:
        return N.lib().flux_last_launch_count(self._h)

    def set_timing(self, enable: bool = True) -> None:
        N.check(N.lib().flux_comm_set_timing(self._h, int(enable)))

    def last_kernel_ms(self) -> float:
        v = C.c_float()
        N.check(N.lib().flux_last_kernel_ms(self._h, C.byref(v)))
        return float(v.value)

    def inject_fault(self, kind: int, rank: int = 0, index: int = 0) -> None:
        """Arm a fault for the next operator (flux_comm_inject_fault): drop or
        double one signal of `rank`'s flag table."""
        N.check(N.lib().flux_comm_inject_fault(self._h, kind, rank, index))

    def set_check_double_set(self, enable: bool = True) -> None:
        N.check(N.lib().flux_comm_set_check_double_set(self._h, int(enable)))

    def drop_peer(self, from_rank: int, peer_rank: int) -> None:
        N.check(N.lib().flux_comm_drop_peer(self._h, from_rank, peer_rank))

    @property
    def nvls(self) -> bool:
        """True if the communicator owns an NVLS multicast region (nvls_bytes > 0)."""
        return bool(N.lib().flux_comm_nvls(self._h))

    def close(self) -> None:
        if self._h:
            N.lib().flux_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def required_heap_bytes(problem: ProblemSpec) -> int:
    return int(N.lib().flux_required_heap_bytes(C.byref(problem.c())))


def nvls_required_bytes(problem: ProblemSpec) -> int:
    """Per-rank NVLS region bytes the problem needs (Communicator(nvls_bytes=...))."""
    return int(N.lib().flux_nvls_required_bytes(C.byref(problem.c())))


TRACE_KINDS = {1: "compute_start", 2: "signal_set", 3: "tile_write", 4: "reduce", 5: "wait", 6: "launch"}


def read_trace(comm: Communicator, rank: int, problem: ProblemSpec, max_records: int = 1 << 18) -> list[dict]:
    """Device event trace of the last operator run with opts.trace=1, as the
    reference's CausalityEvent records (engine.hpp:37-63): kind, rank,
    tile_row, tile_col, target, logical_ts (order of the device timestamps),
    wall_ns (%globaltimer relative to the first event)."""
    buf = (C.c_uint64 * (2 * max_records))()
    n = C.c_size_t()
    N.check(N.lib().flux_trace_read(comm._h, rank, C.byref(problem.c()), buf, max_records, C.byref(n)))
    recs = []
    for i in range(n.value):
        ts, w = buf[2 * i], buf[2 * i + 1]
        recs.append({"event": TRACE_KINDS.get(w >> 60, "unknown"), "rank": (w >> 56) & 0xF,
                     "tile_row": (w >> 16) & 0xFFFF, "tile_col": w & 0xFFFF, "target": (w >> 32) & 0xFFFFFF,
                     "ts": ts})
    recs.sort(key=lambda r: r["ts"])
    t0 = recs[0]["ts"] if recs else 0
    for i, r in enumerate(recs):
        r["logical_ts"] = i + 1
        r["wall_ns"] = r["ts"] - t0  # "ts": absolute %globaltimer (comparable across ranks of one GPU)
    return recs


def write_jsonl(path: str, events: list[dict]) -> None:
    """The reference's JSONL schema (engine.cpp:101-109)."""
    import json

    with open(path, "w") as f:
        for e in events:
            f.write(json.dumps({k: e[k] for k in ("event", "rank", "tile_row", "tile_col", "target", "logical_ts",
                                                  "wall_ns")}) + "\n")


def chrome_trace(events: list[dict]) -> dict:
    """The device event trace (read_trace) in the Chrome trace-event format of
    the reference's write_chrome_trace (sim.cpp:597-610): {"traceEvents": [...]}
    with "ph": "X" complete events (ts / dur in us, pid = rank, tid = lane).
    Lanes: each CTA's lifetime (its launch records) is a span on tid = CTA
    index; the tile-level events (compute_start, signal_set, tile_write,
    reduce, copy_done) are zero-duration "X" events on tid = -1 (the rank's
    signal lane) named "<kind> (row,col)" with the target in args."""
    out = []
    starts = {}
    for e in events:
        us = e["wall_ns"] / 1000.0
        if e["event"] == "launch":
            key = (e["rank"], e["tile_row"])
            if e["tile_col"] == 0:
                starts[key] = us
            elif key in starts:
                t0 = starts.pop(key)
                out.append({"name": f"cta {e['tile_row']}", "ph": "X", "ts": t0, "dur": us - t0, "pid": e["rank"],
                            "tid": e["tile_row"]})
            continue
        out.append({"name": f"{e['event']} ({e['tile_row']},{e['tile_col']})", "ph": "X", "ts": us, "dur": 0,
                    "pid": e["rank"], "tid": -1, "args": {"target": e["target"], "logical_ts": e["logical_ts"]}})
    return {"traceEvents": out}


def write_chrome_trace(path: str, events: list[dict]) -> None:
    """write_chrome_trace (sim.cpp:597-610) for the device event trace."""
    import json

    with open(path, "w") as f:
        json.dump(chrome_trace(events), f)
        f.write("\n")


# ---------------------------------------------------------------------------
# file-descriptor hand-off between the processes of one node (NVLS multicast
# handles are POSIX file descriptors): an abstract-namespace Unix socket and
# SCM_RIGHTS (socket.send_fds / recv_fds).
# ---------------------------------------------------------------------------
class fd_server:
    """Listens on abstract socket `name`; serve(n) hands `fd` to n clients,
    then closes the socket and the fd."""

    def __init__(self, name: str, fd: int):
        import socket

        self.fd = fd
        self.sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        self.sock.bind("\0" + name)
        self.sock.listen(64)

    def serve(self, n: int, timeout_s: float = 60.0) -> None:
        import socket

        self.sock.settimeout(timeout_s)
        try:
            for _ in range(n):
                conn, _ = self.sock.accept()
                with conn:
                    socket.send_fds(conn, [b"fd"], [self.fd])
                    conn.recv(1)  # the client holds its copy before we close ours
        finally:
            self.sock.close()
            os.close(self.fd)


def fd_receive(name: str, timeout_s: float = 60.0) -> int:
    """The file descriptor served on abstract socket `name` (a new fd in this process)."""
    import socket
    import time

    deadline = time.monotonic() + timeout_s
    while True:
        s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        try:
            s.connect("\0" + name)
            break
        except OSError:
            s.close()
            if time.monotonic() > deadline:
                raise
            time.sleep(0.01)
    with s:
        _, fds, _, _ = socket.recv_fds(s, 16, 1)
        s.sendall(b"k")
    if not fds:
        raise OSError("no file descriptor received on " + name)
    return fds[0]

