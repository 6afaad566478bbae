"""ctypes binding of the C ABI in include/flux_b200.h.

This module is the only place Python touches the native library. It fails
loudly when `libflux_b200.so` is missing: there is no Python or CPU fallback
for the operators.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libflux_b200.so")

# Return codes (flux_status) -> reference exception taxonomy (errors.hpp:9-31).
OK, ERR_CONFIG, ERR_SHAPE, ERR_DIRECTORY, ERR_DEADLOCK, ERR_BOUNDS, ERR_CUDA, ERR_RUNTIME = range(8)
ALLGATHER_GEMM, GEMM_REDUCESCATTER = 0, 1
PULL, PUSH = 0, 1
WRITE_ALLTOALL, FUSED_REDUCE = 0, 1
SWIZZLE_NAIVE, SWIZZLE_RANK_SHIFTED, SWIZZLE_ARRIVAL_ALIGNED = 0, 1, 2
BF16, F32 = 0, 1
BUF_A_SHARD, BUF_B_SHARD, BUF_A_AGG, BUF_C_OUT, BUF_STAGING, BUF_C_OUT_F32 = 0, 1, 2, 3, 4, 5
ACT_NONE, ACT_GELU, ACT_RELU, ACT_SILU, ACT_SWIGLU = 0, 1, 2, 3, 4
ABI_VERSION = 8
FAULT_NONE, FAULT_DROP_SIGNAL, FAULT_DOUBLE_SIGNAL = 0, 1, 2
B_NK, B_KN = 0, 1
DECODE_AUTO, DECODE_TILE, DECODE_STREAM = 0, 1, 2  # flux_decode_kernel
NVLS_OFF, NVLS_MULTICAST, NVLS_EMULATED = 0, 1, 2  # flux_nvls


class FluxError(RuntimeError):
    code = -1


class ConfigError(FluxError):
    code = ERR_CONFIG


class ShapeError(FluxError):
    code = ERR_SHAPE


class DirectoryError(FluxError):
    code = ERR_DIRECTORY


class DeadlockError(FluxError):
    code = ERR_DEADLOCK


class BoundsError(FluxError):
    code = ERR_BOUNDS


class CudaError(FluxError):
    code = ERR_CUDA


class SignalError(FluxError):
    """std::runtime_error of the reference: a flag set twice (engine.cpp:401-403)."""
    code = ERR_RUNTIME


_EXC = {ERR_CONFIG: ConfigError, ERR_SHAPE: ShapeError, ERR_DIRECTORY: DirectoryError,
        ERR_DEADLOCK: DeadlockError, ERR_BOUNDS: BoundsError, ERR_CUDA: CudaError, ERR_RUNTIME: SignalError}


class Problem(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("tp", C.c_int), ("pattern", C.c_int)]


class Tile(C.Structure):
    _fields_ = [("tm", C.c_int), ("tn", C.c_int)]


class Opts(C.Structure):
    _fields_ = [("workers_per_rank", C.c_int), ("deterministic_reduce", C.c_int),
                ("poll_budget", C.c_longlong), ("wall_budget_s", C.c_double),
                ("interleave_seed", C.c_uint64), ("shift_offset", C.c_int), ("out_dtype", C.c_int),
                ("emulated_order", C.c_int), ("cta_group", C.c_int), ("ag_engine", C.c_int), ("trace", C.c_int),
                ("activation", C.c_int), ("activation_grad", C.c_int), ("rs_partials", C.c_int),
                ("b_layout", C.c_int), ("graph_safe", C.c_int), ("decode_kernel", C.c_int),
                ("nvls", C.c_int)]


class CommOpts(C.Structure):
    _fields_ = [("heap_bytes", C.c_size_t), ("nvls_bytes", C.c_size_t)]


class Matrix(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("ld", C.c_int)]


class Operands(C.Structure):
    _fields_ = [("a", Matrix), ("b", Matrix), ("c", Matrix), ("aux", Matrix)]


class Mlp(C.Structure):
    _fields_ = [("m", C.c_int), ("hidden", C.c_int), ("ffn", C.c_int), ("tp", C.c_int), ("activation", C.c_int)]


class MlpOperands(C.Structure):
    _fields_ = [("x", Matrix), ("w_up", Matrix), ("w_down", Matrix), ("pre", Matrix), ("act", Matrix),
                ("out", Matrix)]


class MlpGradOperands(C.Structure):
    _fields_ = [("dout", Matrix), ("w_down_t", Matrix), ("w_up_t", Matrix), ("pre", Matrix), ("dact", Matrix),
                ("dx", Matrix)]


class TransferRecord(C.Structure):
    """flux_transfer_record (reference TransferRecord, engine.hpp:79-85)."""
    _fields_ = [("peer", C.c_int), ("row_begin", C.c_int), ("rows", C.c_int), ("copy_done_ns", C.c_int64),
                ("flag_set_ns", C.c_int64)]


class BufferDesc(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("rows", C.c_int), ("cols", C.c_int), ("ld", C.c_int),
                ("dtype", C.c_int)]


_P = C.POINTER
_SIGS = {
    "flux_last_error": (C.c_char_p, []),
    "flux_abi_version": (C.c_int, []),
    "flux_device_sm_count": (C.c_int, [C.c_int]),
    "flux_default_opts": (None, [_P(Opts)]),
    "flux_problem_validate": (C.c_int, [_P(Problem), _P(Tile)]),
    "flux_grid_for": (C.c_int, [_P(Problem), _P(Tile), _P(C.c_int), _P(C.c_int), _P(C.c_int)]),
    "flux_tile_order": (C.c_int, [_P(Problem), _P(Tile), C.c_int, C.c_int, C.c_int, _P(C.c_int), C.c_int,
                                  _P(C.c_int), _P(C.c_int)]),
    "flux_comm_order": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P(C.c_int), _P(C.c_int), _P(C.c_int),
                                  C.c_int, _P(C.c_int)]),
    "flux_make_comm_spec": (C.c_int, [_P(Problem), C.c_int, C.c_int, C.c_int, _P(C.c_int), _P(C.c_int),
                                      _P(C.c_int), C.c_int, _P(C.c_int)]),
    "flux_required_heap_bytes": (C.c_size_t, [_P(Problem)]),
    "flux_comm_create": (C.c_int, [C.c_int, _P(C.c_int), _P(CommOpts), _P(C.c_void_p)]),
    "flux_comm_create_ipc": (C.c_int, [C.c_int, C.c_int, C.c_int, _P(CommOpts), _P(C.c_void_p)]),
    "flux_comm_ipc_blob_bytes": (C.c_size_t, []),
    "flux_comm_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "flux_comm_ipc_connect": (C.c_int, [C.c_void_p, C.c_void_p]),
    "flux_ipc_blobs_check": (C.c_int, [C.c_void_p, C.c_int, C.c_size_t]),
    "flux_comm_destroy": (C.c_int, [C.c_void_p]),
    "flux_comm_tp": (C.c_int, [C.c_void_p]),
    "flux_comm_rank": (C.c_int, [C.c_void_p]),
    "flux_comm_drop_peer": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "flux_buffer": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _P(Problem), _P(BufferDesc)]),
    "flux_copy_in": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _P(Problem), C.c_void_p, C.c_int, C.c_void_p]),
    "flux_copy_out": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _P(Problem), C.c_void_p, C.c_int, C.c_void_p]),
    "flux_ag_gemm": (C.c_int, [C.c_void_p, _P(Problem), _P(Tile), C.c_int, C.c_int, C.c_int, _P(Opts),
                               _P(C.c_void_p)]),
    "flux_gemm_rs": (C.c_int, [C.c_void_p, _P(Problem), _P(Tile), C.c_int, C.c_int, _P(Opts), _P(C.c_void_p)]),
    "flux_ag_gemm_ex": (C.c_int, [C.c_void_p, _P(Problem), _P(Tile), C.c_int, C.c_int, C.c_int, _P(Opts),
                                  _P(C.c_void_p), _P(Operands)]),
    "flux_gemm_rs_ex": (C.c_int, [C.c_void_p, _P(Problem), _P(Tile), C.c_int, C.c_int, _P(Opts), _P(C.c_void_p),
                                  _P(Operands)]),
    "flux_ag_engine": (C.c_int, [_P(Problem), C.c_int, _P(Opts)]),
    "flux_local_gemm": (C.c_int, [C.c_void_p, _P(Problem), _P(Opts), _P(C.c_void_p)]),
    "flux_nonoverlap": (C.c_int, [C.c_void_p, _P(Problem), _P(Opts), _P(C.c_void_p)]),
    "flux_medium_grained": (C.c_int, [C.c_void_p, _P(Problem), _P(Tile), C.c_int, _P(Opts), _P(C.c_void_p)]),
    "flux_sync": (C.c_int, [C.c_void_p]),
    "flux_last_launch_count": (C.c_int, [C.c_void_p]),
    "flux_comm_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "flux_last_kernel_ms": (C.c_int, [C.c_void_p, _P(C.c_float)]),
    "flux_trace_read": (C.c_int, [C.c_void_p, C.c_int, _P(Problem), C.c_void_p, C.c_size_t, _P(C.c_size_t)]),
    "flux_mlp_forward": (C.c_int, [C.c_void_p, _P(Mlp), _P(Opts), _P(C.c_void_p), _P(MlpOperands)]),
    "flux_mlp_backward_dx": (C.c_int, [C.c_void_p, _P(Mlp), _P(Opts), _P(C.c_void_p), _P(MlpGradOperands)]),
    "flux_mlp_required_heap_bytes": (C.c_size_t, [_P(Mlp)]),
    "flux_comm_inject_fault": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int]),
    "flux_map_tile": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P(C.c_int), C.c_int, C.c_int, C.c_int, C.c_int,
                                C.c_int, _P(C.c_int), _P(C.c_int)]),
    "flux_validate_comm_spec": (C.c_int, [_P(Problem), C.c_int, C.c_int, C.c_int, _P(C.c_int), _P(C.c_int),
                                          _P(C.c_int), C.c_int]),
    "flux_ag_gemm_ordered": (C.c_int, [C.c_void_p, _P(Problem), _P(Tile), C.c_int, C.c_int, C.c_int, _P(Opts),
                                       _P(C.c_void_p), _P(Operands), _P(C.c_int), _P(C.c_int), _P(C.c_int), C.c_int]),
    "flux_transfer_log": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, _P(C.c_int)]),
    "flux_comm_set_check_double_set": (C.c_int, [C.c_void_p, C.c_int]),
    "flux_nvls_probe": (C.c_int, [C.c_int, _P(C.c_int), C.c_char_p, C.c_int]),
    "flux_nvls_required_bytes": (C.c_size_t, [_P(Problem)]),
    "flux_comm_nvls": (C.c_int, [C.c_void_p]),
    "flux_comm_nvls_ipc_export": (C.c_int, [C.c_void_p, C.c_size_t, _P(C.c_int)]),
    "flux_comm_nvls_ipc_import": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int]),
    "flux_comm_nvls_ipc_add_device": (C.c_int, [C.c_void_p]),
    "flux_comm_nvls_ipc_bind": (C.c_int, [C.c_void_p]),
}

# Symbols include/flux_b200.h declares (tests check the library exports all of them).
EXPORTED = sorted(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """Loads libflux_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        path = os.environ.get("FLUX_LIB_PATH", LIB_PATH)  # profiling variants only
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_2406_06858_b200.build` "
                "(the fused operators have no CPU fallback)")
        l = C.CDLL(path, mode=C.RTLD_LOCAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        if l.flux_abi_version() != ABI_VERSION:
            raise ImportError(f"{path}: ABI version {l.flux_abi_version()} != {ABI_VERSION} (rebuild the library)")
        _lib = l
    return _lib


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().flux_last_error().decode(errors="replace")
        raise _EXC.get(rc, FluxError)(msg)


def default_opts(**kw) -> Opts:
    o = Opts()
    lib().flux_default_opts(C.byref(o))
    names = {f[0] for f in Opts._fields_}
    for k, v in kw.items():
        if k not in names:
            raise TypeError(f"unknown flux_opts field {k!r}")
        setattr(o, k, v)
    return o


def nvls_probe(devices) -> tuple[bool, str]:
    """(supported, reason): can an NVLS multicast object be created over `devices`?"""
    devs = (C.c_int * len(devices))(*devices)
    why = C.create_string_buffer(256)
    ok = lib().flux_nvls_probe(len(devices), devs, why, 256)
    return bool(ok), why.value.decode(errors="replace")


def stream_array(streams):
    """List of raw cudaStream_t ints -> void*[]; None -> NULL (library streams).
    An explicit 0 (torch's legacy default stream) becomes cudaStreamLegacy (0x1):
    the C ABI reads a NULL entry as "use the library's stream"."""
    if streams is None:
        return None
    arr = (C.c_void_p * len(streams))(*[s if s else 1 for s in streams])
    return arr
