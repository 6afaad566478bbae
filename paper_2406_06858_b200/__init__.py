"""B200-native fused AllGather-GEMM / GEMM-ReduceScatter (Flux, arXiv 2406.06858).

The operators live in the native library libflux_b200.so (C ABI:
include/flux_b200.h); this package is the Python host mirror of the
reference's operator API over that ABI.
"""
from . import _native
from ._native import (ALLGATHER_GEMM, GEMM_REDUCESCATTER, PULL, PUSH, WRITE_ALLTOALL, FUSED_REDUCE,
                      SWIZZLE_NAIVE, SWIZZLE_RANK_SHIFTED, SWIZZLE_ARRIVAL_ALIGNED, BF16, F32,
                      ConfigError, ShapeError, DirectoryError, DeadlockError, BoundsError, CudaError, SignalError,
                      FluxError, default_opts, ACT_NONE, ACT_GELU, ACT_RELU, ACT_SILU, ACT_SWIGLU, B_NK, B_KN,
                      DECODE_AUTO, DECODE_TILE, DECODE_STREAM, NVLS_OFF, NVLS_MULTICAST, NVLS_EMULATED, nvls_probe,
                      FAULT_NONE, FAULT_DROP_SIGNAL, FAULT_DOUBLE_SIGNAL)
from .comm import (Communicator, MlpSpec, ProblemSpec, TileShape, comm_order, grid_for, make_comm_spec,
                   required_heap_bytes, nvls_required_bytes, tile_order, validate_tiling)

__all__ = [n for n in dir() if not n.startswith("_")]
