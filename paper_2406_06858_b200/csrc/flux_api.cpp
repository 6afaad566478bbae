// C ABI of the B200 fused operators: problem validation, schedules, the
// symmetric-heap communicator, and the AllGather-GEMM / GEMM-ReduceScatter
// drivers. See include/flux_b200.h for the contract and DESIGN.md for the
// data layout.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "flux_b200.h"
#include "flux_internal.hpp"

using namespace fluxb200;

namespace {

// ---------------------------------------------------------------------------
// errors (reference errors.hpp:9-31 -> status codes)
// ---------------------------------------------------------------------------
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define FLUX_CUDA(expr)                                                                    \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return fail(FLUX_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define FLUX_TRY(expr)          \
    do {                        \
        int _rc = (expr);       \
        if (_rc != FLUX_OK) return _rc; \
    } while (0)

std::string S(long long v) { return std::to_string(v); }

// ---------------------------------------------------------------------------
// driver entry points (no link-time dependency on libcuda)
// ---------------------------------------------------------------------------
struct Driver {
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    PFN_cuStreamWriteValue32_v11070 write32 = nullptr;
    PFN_cuStreamWaitValue32_v11070 wait32 = nullptr;
    PFN_cuMemsetD32Async_v3020 memset32 = nullptr;
    bool ok = false;
};

Driver& driver() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.write32 = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(fn);
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.wait32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(fn);
        if (cudaGetDriverEntryPoint("cuMemsetD32Async", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.memset32 = reinterpret_cast<PFN_cuMemsetD32Async_v3020>(fn);
        d.ok = d.encode && d.write32 && d.wait32 && d.memset32;
    });
    return d;
}

int need_driver() {
    if (!driver().ok) return fail(FLUX_ERR_CUDA, "CUDA driver entry points unavailable (no GPU driver?)");
    return FLUX_OK;
}

// NVLS: multicast objects and VMM (driver API, loaded on first use).
struct NvlsDriver {
    PFN_cuDeviceGet_v2000 dev_get = nullptr;
    PFN_cuDeviceGetAttribute_v2000 attr = nullptr;
    PFN_cuGetErrorString_v6000 err_str = nullptr;
    PFN_cuMulticastCreate_v12010 mc_create = nullptr;
    PFN_cuMulticastAddDevice_v12010 mc_add = nullptr;
    PFN_cuMulticastBindMem_v12010 mc_bind = nullptr;
    PFN_cuMulticastUnbind_v12010 mc_unbind = nullptr;
    PFN_cuMulticastGetGranularity_v12010 mc_gran = nullptr;
    PFN_cuMemCreate_v10020 mem_create = nullptr;
    PFN_cuMemRelease_v10020 mem_release = nullptr;
    PFN_cuMemAddressReserve_v10020 va_reserve = nullptr;
    PFN_cuMemAddressFree_v10020 va_free = nullptr;
    PFN_cuMemMap_v10020 map = nullptr;
    PFN_cuMemUnmap_v10020 unmap = nullptr;
    PFN_cuMemSetAccess_v10020 set_access = nullptr;
    PFN_cuMemExportToShareableHandle_v10020 export_handle = nullptr;
    PFN_cuMemImportFromShareableHandle_v10020 import_handle = nullptr;
    bool ok = false;
};

NvlsDriver& nvls_driver() {
    static NvlsDriver d;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            *fn = nullptr;
            if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
                *fn = nullptr;
            return *fn != nullptr;
        };
        bool ok = true;
        ok &= get("cuDeviceGet", reinterpret_cast<void**>(&d.dev_get));
        ok &= get("cuDeviceGetAttribute", reinterpret_cast<void**>(&d.attr));
        ok &= get("cuGetErrorString", reinterpret_cast<void**>(&d.err_str));
        ok &= get("cuMulticastCreate", reinterpret_cast<void**>(&d.mc_create));
        ok &= get("cuMulticastAddDevice", reinterpret_cast<void**>(&d.mc_add));
        ok &= get("cuMulticastBindMem", reinterpret_cast<void**>(&d.mc_bind));
        ok &= get("cuMulticastUnbind", reinterpret_cast<void**>(&d.mc_unbind));
        ok &= get("cuMulticastGetGranularity", reinterpret_cast<void**>(&d.mc_gran));
        ok &= get("cuMemCreate", reinterpret_cast<void**>(&d.mem_create));
        ok &= get("cuMemRelease", reinterpret_cast<void**>(&d.mem_release));
        ok &= get("cuMemAddressReserve", reinterpret_cast<void**>(&d.va_reserve));
        ok &= get("cuMemAddressFree", reinterpret_cast<void**>(&d.va_free));
        ok &= get("cuMemMap", reinterpret_cast<void**>(&d.map));
        ok &= get("cuMemUnmap", reinterpret_cast<void**>(&d.unmap));
        ok &= get("cuMemSetAccess", reinterpret_cast<void**>(&d.set_access));
        ok &= get("cuMemExportToShareableHandle", reinterpret_cast<void**>(&d.export_handle));
        ok &= get("cuMemImportFromShareableHandle", reinterpret_cast<void**>(&d.import_handle));
        d.ok = ok;
    });
    return d;
}

std::string cu_err(CUresult r) {
    const char* s = nullptr;
    if (nvls_driver().err_str) nvls_driver().err_str(r, &s);
    return s ? std::string(s) : ("CUresult " + std::to_string(static_cast<int>(r)));
}

int write_value(cudaStream_t s, void* addr, uint32_t v) {
    CUresult r = driver().write32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                                  CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(FLUX_ERR_CUDA, "cuStreamWriteValue32 failed (" + S(r) + ")");
    return FLUX_OK;
}

// Stream-side wait for an epoch-stamped word (wrap-safe >=). The wait is
// followed by a flush of outstanding remote writes where the device supports
// it, so data written by peers before they stamped the word is visible to the
// work queued after the wait.
int wait_value_geq(cudaStream_t s, const void* addr, uint32_t v) {
    if (v == 0) return FLUX_OK;  // epoch 0 is always satisfied
    // The flush capability is a property of the device the stream belongs to
    // (callers set it current): cached per device, -1 = not probed yet.
    static std::atomic<int> flush_cap[64] = {};
    static std::once_flag init;
    std::call_once(init, [] {
        for (auto& f : flush_cap) f.store(-1);
    });
    int dev = 0;
    cudaGetDevice(&dev);
    unsigned flush = 0;
    if (dev >= 0 && dev < 64) {
        int cap = flush_cap[dev].load(std::memory_order_acquire);
        if (cap < 0) {
            int can = 0;
            cudaDeviceGetAttribute(&can, cudaDevAttrCanFlushRemoteWrites, dev);
            cap = can ? 1 : 0;
            flush_cap[dev].store(cap, std::memory_order_release);
        }
        flush = cap ? static_cast<unsigned>(CU_STREAM_WAIT_VALUE_FLUSH) : 0u;
    }
    CUresult r = driver().wait32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                                 CU_STREAM_WAIT_VALUE_GEQ | flush);
    if (r != CUDA_SUCCESS) return fail(FLUX_ERR_CUDA, "cuStreamWaitValue32 failed (" + S(r) + ")");
    return FLUX_OK;
}

// ---------------------------------------------------------------------------
// problem validation: ProblemSpec::validate / validate_tiling (problem.cpp:15-38)
// ---------------------------------------------------------------------------
int validate_problem(const flux_problem* p) {
    if (!p) return fail(FLUX_ERR_CONFIG, "null problem");
    if (p->m <= 0 || p->n <= 0 || p->k <= 0) return fail(FLUX_ERR_CONFIG, "problem dimensions must be positive");
    if (p->tp <= 0) return fail(FLUX_ERR_CONFIG, "tp must be positive");
    if (p->pattern != FLUX_ALLGATHER_GEMM && p->pattern != FLUX_GEMM_REDUCESCATTER)
        return fail(FLUX_ERR_CONFIG, "unknown pattern");
    if (p->m % p->tp != 0)
        return fail(FLUX_ERR_CONFIG, "m=" + S(p->m) + " not divisible by tp=" + S(p->tp));
    if (p->pattern == FLUX_ALLGATHER_GEMM && p->n % p->tp != 0)
        return fail(FLUX_ERR_CONFIG,
                    "AllGatherGemm requires n divisible by tp (weight is column-sharded); n=" + S(p->n) +
                        " tp=" + S(p->tp));
    if (p->pattern == FLUX_GEMM_REDUCESCATTER && p->k % p->tp != 0)
        return fail(FLUX_ERR_CONFIG,
                    "GemmReduceScatter requires k divisible by tp (weight is row-sharded); k=" + S(p->k) +
                        " tp=" + S(p->tp));
    return FLUX_OK;
}

int rows_per_rank(const flux_problem* p) { return p->m / p->tp; }
int local_cols(const flux_problem* p) { return p->pattern == FLUX_ALLGATHER_GEMM ? p->n / p->tp : p->n; }
int local_k(const flux_problem* p) { return p->pattern == FLUX_GEMM_REDUCESCATTER ? p->k / p->tp : p->k; }

int validate_tiling(const flux_problem* p, const flux_tile* t) {
    FLUX_TRY(validate_problem(p));
    if (!t) return fail(FLUX_ERR_CONFIG, "null tile");
    if (t->tm <= 0 || t->tn <= 0) return fail(FLUX_ERR_CONFIG, "tile extents must be positive");
    const int rpr = rows_per_rank(p);
    if (t->tm > rpr || rpr % t->tm != 0)
        return fail(FLUX_ERR_CONFIG, "tm=" + S(t->tm) + " must divide m/tp=" + S(rpr));
    const int lc = local_cols(p);
    if (lc % t->tn != 0)
        return fail(FLUX_ERR_CONFIG, "tn=" + S(t->tn) + " must divide the local output cols=" + S(lc));
    return FLUX_OK;
}

// ---------------------------------------------------------------------------
// schedules: block order (swizzle.cpp:23-47), comm order (topology.cpp:46-55,102-178)
// ---------------------------------------------------------------------------
std::vector<int> block_order(int kind, int rank, int tp, int shift, const std::vector<int>& arrival) {
    std::vector<int> b;
    if (kind == FLUX_SWIZZLE_ARRIVAL_ALIGNED) {
        if (!arrival.empty()) return arrival;
        b.push_back(rank);
        for (int d = 1; d < tp; ++d) b.push_back((rank + d) % tp);
    } else {  // RankShifted: start after `shift`, local block last for shift = 1
        for (int d = 0; d < tp; ++d) b.push_back(((rank + shift) % tp + d) % tp);
    }
    return b;
}

struct Desc {
    int peer, row_begin, rows;
};

// NVLinkRing pull order: peers rank+1, rank+2, ..., each block cut into comm tiles.
std::vector<Desc> ring_order(int rank, int tp, int rpr, int rpct) {
    std::vector<Desc> out;
    for (int d = 1; d < tp; ++d) {
        const int peer = (rank + d) % tp;
        for (int off = 0; off < rpr; off += rpct) out.push_back({peer, peer * rpr + off, rpct});
    }
    return out;
}

// Peers in order of first appearance (topology.cpp:170-178).
std::vector<int> peer_order(const std::vector<Desc>& order, int rank, int rpr) {
    std::vector<int> seq;
    for (const Desc& d : order) {
        const int block = d.row_begin / rpr;
        if (block == rank) continue;
        if (std::find(seq.begin(), seq.end(), block) == seq.end()) seq.push_back(block);
    }
    return seq;
}

// CommTileSpec::validate (engine.cpp:40-75).
int validate_comm_spec(const flux_problem* p, int rank, int rpct, int transfer, const std::vector<Desc>& order) {
    const int rpr = rows_per_rank(p);
    if (rpct <= 0 || rpr % rpct != 0)
        return fail(FLUX_ERR_CONFIG, "rows_per_comm_tile=" + S(rpct) + " must divide m/tp=" + S(rpr));
    const int ct = rpr / rpct;
    std::vector<int> seen(p->m / rpct, 0);
    for (const Desc& d : order) {
        if (d.rows != rpct || d.row_begin % rpct != 0 || d.row_begin < 0 || d.row_begin + d.rows > p->m)
            return fail(FLUX_ERR_BOUNDS, "transfer descriptor rows [" + S(d.row_begin) + ",+" + S(d.rows) + ") invalid");
        ++seen[d.row_begin / rpct];
    }
    for (int t = 0; t < static_cast<int>(seen.size()); ++t) {
        const bool local = t / ct == rank;
        if (transfer == FLUX_PULL) {
            if (!local && seen[t] != 1)
                return fail(FLUX_ERR_CONFIG, "comm order must cover non-local comm tile " + S(t) +
                                                 " exactly once (saw " + S(seen[t]) + ")");
            if (local && seen[t] != 0) return fail(FLUX_ERR_CONFIG, "comm order must not include local comm tiles");
        } else {
            if (local && seen[t] != p->tp - 1)
                return fail(FLUX_ERR_CONFIG, "push order must carry local comm tile " + S(t) + " to every peer");
            if (!local && seen[t] != 0) return fail(FLUX_ERR_CONFIG, "push order may only move local comm tiles");
        }
    }
    return FLUX_OK;
}

// make_comm_specs for one rank (engine.cpp:77-99).
int make_spec(const flux_problem* p, int rank, int rpct, int transfer, std::vector<Desc>& out) {
    FLUX_TRY(validate_problem(p));
    const int rpr = rows_per_rank(p);
    if (rpct <= 0 || rpr % rpct != 0)
        return fail(FLUX_ERR_CONFIG, "rows_per_comm_tile=" + S(rpct) + " must divide rows_per_rank=" + S(rpr));
    if (rank < 0 || rank >= p->tp) return fail(FLUX_ERR_CONFIG, "rank " + S(rank) + " >= tp");
    std::vector<Desc> pull = ring_order(rank, p->tp, rpr, rpct);
    if (transfer == FLUX_PULL) {
        out = pull;
    } else if (transfer == FLUX_PUSH) {
        out.clear();
        for (int peer : peer_order(pull, rank, rpr))
            for (int off = 0; off < rpr; off += rpct) out.push_back({peer, rank * rpr + off, rpct});
    } else {
        return fail(FLUX_ERR_CONFIG, "unknown transfer mode");
    }
    return validate_comm_spec(p, rank, rpct, transfer, out);
}

// Row-block visit order used by the AG kernel (engine.cpp:475-505), from every
// rank's comm spec for `transfer` (the reference's defaults or the caller's).
std::vector<int> ag_block_order(const flux_problem* p, int rank, int transfer, bool swizzle,
                                const std::vector<std::vector<Desc>>& specs) {
    const int tp = p->tp, rpr = rows_per_rank(p);
    if (!swizzle) {
        std::vector<int> b;
        for (int i = 0; i < tp; ++i) b.push_back(i);
        return b;
    }
    if (transfer == FLUX_PULL) {  // arrival_aligned_policy: local first, then peer_order(comm)
        std::vector<int> b{rank};
        for (int q : peer_order(specs[rank], rank, rpr)) b.push_back(q);
        for (int q = 0; q < tp; ++q)  // (a valid Pull spec names every peer; defensive)
            if (std::find(b.begin(), b.end(), q) == b.end()) b.push_back(q);
        return b;
    }
    // Push: sources sorted by how early their list targets this rank.
    std::vector<std::pair<int, int>> arrivals;
    for (int s = 0; s < tp; ++s) {
        if (s == rank) continue;
        const std::vector<Desc>& spec = specs[s];
        for (size_t i = 0; i < spec.size(); ++i)
            if (spec[i].peer == rank) {
                arrivals.emplace_back(static_cast<int>(i), s);
                break;
            }
    }
    std::sort(arrivals.begin(), arrivals.end());
    std::vector<int> b{rank};
    for (auto& a : arrivals) b.push_back(a.second);
    for (int s = 0; s < tp; ++s)
        if (std::find(b.begin(), b.end(), s) == b.end()) b.push_back(s);
    return b;
}

// The reference's comm specs of every rank (make_comm_specs, engine.cpp:77-99).
int default_specs(const flux_problem* p, int rpct, int transfer, std::vector<std::vector<Desc>>& out) {
    out.assign(p->tp, {});
    for (int r = 0; r < p->tp; ++r) FLUX_TRY(make_spec(p, r, rpct, transfer, out[r]));
    return FLUX_OK;
}

// Device tile sequence of one rank over the kBM x kBN grid. When ownership
// blocks align with device tile rows the reference's block-then-column-major
// order is reproduced (swizzle.cpp:51-73); otherwise tiles straddle blocks and
// the order is a grouped raster (every rank walks the same sequence).
//
// Blocks of few tile rows re-stream every column panel of B per block, so
// `group_blocks` consecutive blocks of the visit order may share one
// column-major sweep (a super-block); `last_alone` keeps the final block on its
// own (RS: the owner's local block must stay last).
std::vector<uint32_t> device_sequence(int m, int ncols, int rpr, const std::vector<int>& blocks, int tile_m,
                                      int group_blocks = 1, bool last_alone = false) {
    const int slot = 0;
    const int tiles_m = (m + tile_m - 1) / tile_m, tiles_n = (ncols + kBN - 1) / kBN;
    std::vector<uint32_t> seq;
    seq.reserve(static_cast<size_t>(tiles_m) * tiles_n);
    if (!blocks.empty() && rpr % tile_m == 0) {
        const int rpb = rpr / tile_m;
        const int nb = static_cast<int>(blocks.size());
        const int grouped = last_alone ? nb - 1 : nb;
        for (int b0 = 0; b0 < nb;) {
            const int g = b0 < grouped ? std::min(std::max(1, group_blocks), grouped - b0) : 1;
            for (int c = 0; c < tiles_n; ++c)
                for (int bi = b0; bi < b0 + g; ++bi)
                    for (int r = 0; r < rpb; ++r) seq.push_back(pack_tile(slot, blocks[bi] * rpb + r, c));
            b0 += g;
        }
    } else {
        // Grouped raster: bands of kRasterRows tile rows walked column by column,
        // so one wave of CTAs shares a few A row-panels and B column-panels in L2
        // (plain row-major re-streams all of B for every tile row).
        constexpr int kRasterRows = 8;
        for (int r0 = 0; r0 < tiles_m; r0 += kRasterRows)
            for (int c = 0; c < tiles_n; ++c)
                for (int r = r0; r < std::min(tiles_m, r0 + kRasterRows); ++r) seq.push_back(pack_tile(slot, r, c));
    }
    return seq;
}

// Blocks per super-block. AG keeps the reference's strict block order (a
// super-block would make early tiles wait for later transfers; measured
// slower); RS sweeps at least 4 tile rows per column panel of B (measured
// ~3 % faster on L-RS). FLUX_GROUP_BLOCKS overrides both.
int group_blocks(int rpr, int tile_m, bool ag) {
    if (const char* env = std::getenv("FLUX_GROUP_BLOCKS")) return std::max(1, std::atoi(env));
    if (ag) return 1;
    const int rpb = std::max(1, rpr / tile_m);
    return std::max(1, 4 / rpb);
}

// ---------------------------------------------------------------------------
// symmetric heap layout (identical on every rank)
// ---------------------------------------------------------------------------
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
int pad_to(int v, int a) { return (v + a - 1) / a * a; }

struct Region {
    size_t off = 0;
    int rows = 0, cols = 0, ld = 0, dtype = FLUX_BF16;
    size_t bytes() const { return static_cast<size_t>(rows) * ld * (dtype == FLUX_F32 ? 4 : 2); }
};

struct Layout {
    Region a_shard, b, a_agg, c, c32, staging;
    size_t trace_off = 0;
    size_t tail_ws_off = 0;
    long long stage_plane = 0, stage_parity = 0;
    int ld_stage = 0;
    size_t total = 0;
};

Layout layout_for(const flux_problem* p) {
    Layout L;
    const int rpr = rows_per_rank(p), lc = local_cols(p), lk = local_k(p);
    size_t off = kDataOffset;
    auto place = [&](Region& r, int rows, int cols, int dtype, int pad) {
        r.off = off;
        r.rows = rows;
        r.cols = cols;
        r.ld = pad_to(cols, pad);
        r.dtype = dtype;
        off = align_up(off + std::max<size_t>(r.bytes(), 1), 4096);
    };
    if (p->pattern == FLUX_ALLGATHER_GEMM) {
        place(L.a_shard, rpr, lk, FLUX_BF16, 64);
        place(L.a_agg, p->m, lk, FLUX_BF16, 64);
        place(L.b, lc, lk, FLUX_BF16, 64);
        place(L.c32, p->m, lc, FLUX_F32, 32);  // C region sized for fp32; bf16 view shares it
    } else {
        place(L.a_shard, p->m, lk, FLUX_BF16, 64);
        place(L.b, lc, lk, FLUX_BF16, 64);
        place(L.c32, rpr, lc, FLUX_F32, 32);
        L.ld_stage = pad_to(lc, kBN);  // a plane also holds tile-major 128 x 256 partials (RS mode)
        L.stage_plane = static_cast<long long>(rpr) * L.ld_stage;
        L.stage_parity = L.stage_plane * p->tp;
        L.staging.off = off;
        L.staging.rows = 2 * p->m;  // 2 parities x tp planes x rpr rows
        L.staging.cols = lc;
        L.staging.ld = L.ld_stage;
        L.staging.dtype = FLUX_F32;
        off = align_up(off + static_cast<size_t>(2) * L.stage_parity * 4, 4096);
    }
    L.tail_ws_off = off;  // tail-split K-slice partials of one launch (Plain / AG)
    off = align_up(off + static_cast<size_t>(kTailWsCtas) * kBM * kBN * 4, 4096);
    L.c = L.c32;
    L.c.dtype = FLUX_BF16;
    L.trace_off = off;  // device event trace ring (flux_opts.trace)
    off += kTraceBytes;
    L.total = off;
    return L;
}

// ---------------------------------------------------------------------------
// communicator
// ---------------------------------------------------------------------------
struct RankState {
    int device = 0;
    char* heap = nullptr;     // address of this rank's heap in our VA (own or peer-mapped)
    bool owned = false;       // allocated by us (free on destroy) vs IPC-opened
    bool local = false;       // we drive this rank (launch work for it)
    cudaStream_t stream = nullptr;       // default compute stream
    cudaStream_t copy_stream = nullptr;  // copy-engine transfer loop
    cudaEvent_t start_evt = nullptr, kernel_evt = nullptr, copy_evt = nullptr;
    bool kernel_evt_valid = false;
};

constexpr uint32_t kIpcMagic = 0xF1u << 24 | 0xB200u;

struct IpcBlob {
    uint32_t magic;
    int32_t rank, tp, device;
    uint64_t heap_bytes;
    int32_t pid;
    int32_t pad;
    cudaIpcMemHandle_t handle;
};

}  // namespace

struct flux_comm {
    int tp = 0;
    int my_rank = -1;  // IPC mode
    bool ipc = false;
    bool connected = false;
    size_t heap_bytes = 0;
    uint32_t epoch = 0;
    std::vector<RankState> ranks;
    std::vector<std::vector<bool>> directory;  // [from][peer] usable
    int last_launches = 0;
    bool timing = false;                          // bracket fused launches with events
    uint64_t ag_sig = 0;                          // in-kernel AG: piece layout of the counters
    uint32_t ag_mult = 0;                         // in-kernel AG: operators since the counter reset
    uint32_t launch_seq = 0;                      // fused launches so far (tags the tail-split counters)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kernel_events;  // per device group
    int kernel_events_used = 0;
    // Device copies of tile schedules / piece tables, keyed by (device, content
    // hash), bounded (least recently used evicted; tables a CUDA graph captured
    // are kept for the communicator's lifetime).
    struct OrderEntry {
        int device = 0;
        uint64_t hash = 0;
        std::vector<uint32_t> table;
        uint32_t* dev = nullptr;     // device copy
        uint32_t* staged = nullptr;  // pinned host copy the asynchronous upload reads
        uint64_t last_use = 0;
        bool captured = false;
    };
    std::vector<OrderEntry> order_cache;
    uint64_t order_clock = 0;
    uint32_t* err_host = nullptr;  // host-mapped error mirror [tp][8] (device waits write it on timeout)
    // Copy-engine transfer log of the last traced AllGather (TransferRecord).
    struct XferEntry {
        int rank = 0, peer = 0, row_begin = 0, rows = 0;
        cudaEvent_t base = nullptr, copy_ev = nullptr, flag_ev = nullptr;
    };
    std::vector<XferEntry> xfer_log;
    std::vector<cudaEvent_t> xfer_events;  // pool
    size_t xfer_used = 0;
    // Fault injection (flux_comm_inject_fault): armed for the next operator,
    // active while that operator enqueues its work.
    int fault_kind = 0, fault_rank = 0, fault_index = 0;
    int act_fault_kind = 0, act_fault_rank = 0, act_fault_index = 0;
    bool check_double = false;      // flux_comm_set_check_double_set
    // Graph-safe operators on a one-process-per-GPU communicator: ordered by
    // device-side rank barriers instead of host stream memops (see graph_ipc_op).
    bool graph_ipc = false;         // a graph-safe operator is being enqueued
    bool last_was_graph = false;    // the previous operator was graph-safe (eager ones fence first)
    std::string host_error;         // host-detected failure of the last operator (flag set twice)
    // NVLS multicast region (flux_comm_opts.nvls_bytes): one multicast object over
    // every rank's GPU; each rank's VMM allocation is bound to it and mapped at
    // uc[r] (its unicast address); mc is the multicast address of the region.
    struct Nvls {
        size_t bytes = 0;
        unsigned long long mc_handle = 0;
        std::vector<unsigned long long> mem;
        std::vector<unsigned long long> uc;
        unsigned long long mc = 0;
        bool bound = false;
    } nvls;
};

namespace {

int check_comm(flux_comm* c) {
    if (!c) return fail(FLUX_ERR_CONFIG, "null communicator");
    if (c->ipc && !c->connected) return fail(FLUX_ERR_DIRECTORY, "IPC communicator not connected");
    return FLUX_OK;
}

// Message of a device error record {code, info0, info1, info2} of rank r
// (the reference's DeadlockError / "set twice" texts, engine.cpp:149-162,401-403).
std::string error_text(const uint32_t* err, int r) {
    if (err[5] != 0) r = static_cast<int>(err[5]) - 1;  // the failing rank (records are shared by a launch)
    if (err[0] == kErrAgFlagTimeout)
        return "deadlock budget exhausted waiting for signal " + S(err[1]) + " for tile (" + S(err[2] >> 16) + "," +
               S(err[2] & 0xFFFF) + ") on rank " + S(r);
    if (err[0] == kErrDoubleSet) return "flag " + S(err[1]) + " on rank " + S(err[2]) + " set twice";
    if (err[0] == kErrBarrierTimeout)
        return "deadlock budget exhausted at the rank barrier of a graph-safe operator (barrier " + S(err[1]) +
               ", waiting for " + S(err[3]) + " arrivals) on rank " + S(r);
    return "deadlock budget exhausted waiting for partial of tile " + S(err[1]) + " from source " + S(err[2]) +
           " on rank " + S(r);
}

int code_of(uint32_t device_code) { return device_code == kErrDoubleSet ? FLUX_ERR_RUNTIME : FLUX_ERR_DEADLOCK; }

// Operator entry: the communicator is usable and no earlier operator left a
// device failure behind. Device waits that time out write their record into a
// host-mapped mirror as well, so this check needs no synchronisation; the
// failure stays reported until flux_sync clears it. Also activates a fault
// armed by flux_comm_inject_fault for this operator.
int begin_op(flux_comm* c) {
    FLUX_TRY(check_comm(c));
    if (c->err_host) {
        for (int r = 0; r < c->tp; ++r) {
            if (!c->ranks[r].local) continue;
            const volatile uint32_t* h = c->err_host + 8 * r;
            if (h[0] != 0) {
                const uint32_t e[6] = {h[0], h[1], h[2], h[3], h[4], h[5]};
                return fail(code_of(e[0]), "a previous operator failed on the device (" + error_text(e, r) +
                                               "); flux_sync reports and clears it");
            }
        }
    }
    c->act_fault_kind = c->fault_kind;
    c->act_fault_rank = c->fault_rank;
    c->act_fault_index = c->fault_index;
    c->fault_kind = 0;
    c->host_error.clear();
    return FLUX_OK;
}

// Operator exit: a host-detected failure (a copy-engine flag the transfer loop
// set twice, engine.cpp:401-403) is raised once every piece of work is enqueued.
int end_op(flux_comm* c) {
    // An injected fault leaves the in-kernel AllGather's monotonic piece
    // counters off their targets (a piece never counted, or counted twice):
    // the next operator re-zeroes them (layout signature reset).
    if (c->act_fault_kind != 0) c->ag_sig = 0;
    c->act_fault_kind = 0;
    if (!c->host_error.empty()) return fail(FLUX_ERR_RUNTIME, c->host_error);
    return FLUX_OK;
}

// ---------------------------------------------------------------------------
// NVLS multicast region: one multicast object over the ranks' GPUs, one VMM
// allocation per GPU bound to it, each mapped at a unicast address, and the
// object mapped once at a multicast address every GPU may access.
// ---------------------------------------------------------------------------
void nvls_release(flux_comm::Nvls& nv, const std::vector<int>& devs) {
    NvlsDriver& d = nvls_driver();
    if (!d.ok) return;
    if (nv.mc) {
        d.unmap(nv.mc, nv.bytes);
        d.va_free(nv.mc, nv.bytes);
    }
    for (size_t r = 0; r < nv.mem.size(); ++r) {
        if (!nv.mem[r]) continue;  // (one process per GPU: only this rank's memory is ours)
        CUdevice cd = 0;
        d.dev_get(&cd, devs[r]);
        if (nv.bound && nv.mc_handle) d.mc_unbind(static_cast<CUmemGenericAllocationHandle>(nv.mc_handle), cd, 0, nv.bytes);
        if (r < nv.uc.size() && nv.uc[r]) {
            d.unmap(nv.uc[r], nv.bytes);
            d.va_free(nv.uc[r], nv.bytes);
        }
        if (nv.mem[r]) d.mem_release(static_cast<CUmemGenericAllocationHandle>(nv.mem[r]));
    }
    if (nv.mc_handle) d.mem_release(static_cast<CUmemGenericAllocationHandle>(nv.mc_handle));
    nv = flux_comm::Nvls{};
}

// Creates the region over `devs` (distinct GPUs, one per rank). On failure
// everything created so far is released and `why` names the failing step.
int nvls_create(flux_comm::Nvls& nv, const std::vector<int>& devs, size_t want, std::string& why) {
    NvlsDriver& d = nvls_driver();
    if (!d.ok) {
        why = "multicast / VMM driver entry points unavailable";
        return FLUX_ERR_CUDA;
    }
    const int n = static_cast<int>(devs.size());
    std::vector<CUdevice> cds(n);
    for (int r = 0; r < n; ++r) {
        for (int q = 0; q < r; ++q)
            if (devs[q] == devs[r]) {
                why = "ranks " + S(q) + " and " + S(r) + " share GPU " + S(devs[r]) + " (NVLS needs one rank per GPU)";
                return FLUX_ERR_CONFIG;
            }
        CUresult e = d.dev_get(&cds[r], devs[r]);
        int mc = 0;
        if (e == CUDA_SUCCESS) e = d.attr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cds[r]);
        if (e != CUDA_SUCCESS || !mc) {
            why = "GPU " + S(devs[r]) + ": multicast not supported" + (e != CUDA_SUCCESS ? " (" + cu_err(e) + ")" : "");
            return FLUX_ERR_CUDA;
        }
    }
    auto step = [&](CUresult e, const char* what) {
        if (e == CUDA_SUCCESS) return true;
        why = std::string(what) + ": " + cu_err(e);
        return false;
    };
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = static_cast<unsigned>(n);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = std::max<size_t>(want, 1);
    size_t gran = 0;
    bool ok = step(d.mc_gran(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    if (ok) {
        gran = std::max<size_t>(gran, size_t(2) << 20);
        nv.bytes = (std::max<size_t>(want, 1) + gran - 1) / gran * gran;
        mp.size = nv.bytes;
        CUmemGenericAllocationHandle h = 0;
        ok = step(d.mc_create(&h, &mp), "cuMulticastCreate");
        nv.mc_handle = h;
    }
    for (int r = 0; ok && r < n; ++r) ok = step(d.mc_add(static_cast<CUmemGenericAllocationHandle>(nv.mc_handle), cds[r]), "cuMulticastAddDevice");
    nv.mem.assign(n, 0);
    nv.uc.assign(n, 0);
    for (int r = 0; ok && r < n; ++r) {
        CUmemAllocationProp ap;
        std::memset(&ap, 0, sizeof(ap));
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = devs[r];
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        CUmemGenericAllocationHandle mh = 0;
        ok = step(d.mem_create(&mh, nv.bytes, &ap, 0), "cuMemCreate");
        nv.mem[r] = mh;
        CUdeviceptr va = 0;
        if (ok) ok = step(d.va_reserve(&va, nv.bytes, gran, 0, 0), "cuMemAddressReserve");
        if (ok) ok = step(d.map(va, nv.bytes, 0, mh, 0), "cuMemMap");
        if (ok) nv.uc[r] = va;
        else if (va) d.va_free(va, nv.bytes);
        CUmemAccessDesc ad;
        std::memset(&ad, 0, sizeof(ad));
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.location.id = devs[r];
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        if (ok) ok = step(d.set_access(nv.uc[r], nv.bytes, &ad, 1), "cuMemSetAccess (unicast)");
    }
    for (int r = 0; ok && r < n; ++r) {
        ok = step(d.mc_bind(static_cast<CUmemGenericAllocationHandle>(nv.mc_handle), 0,
                            static_cast<CUmemGenericAllocationHandle>(nv.mem[r]), 0, nv.bytes, 0),
                  "cuMulticastBindMem");
        if (ok) nv.bound = true;
    }
    if (ok) {
        CUdeviceptr va = 0;
        ok = step(d.va_reserve(&va, nv.bytes, gran, 0, 0), "cuMemAddressReserve (multicast)");
        if (ok) ok = step(d.map(va, nv.bytes, 0, static_cast<CUmemGenericAllocationHandle>(nv.mc_handle), 0),
                          "cuMemMap (multicast)");
        if (ok) nv.mc = va;
        else if (va) d.va_free(va, nv.bytes);
        std::vector<CUmemAccessDesc> ads(n);
        for (int r = 0; r < n; ++r) {
            std::memset(&ads[r], 0, sizeof(ads[r]));
            ads[r].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            ads[r].location.id = devs[r];
            ads[r].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        }
        if (ok) ok = step(d.set_access(nv.mc, nv.bytes, ads.data(), static_cast<size_t>(n)), "cuMemSetAccess (multicast)");
    }
    for (int r = 0; ok && r < n; ++r) {
        if (cudaSetDevice(devs[r]) != cudaSuccess ||
            cudaMemset(reinterpret_cast<void*>(nv.uc[r]), 0, nv.bytes) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            why = "zeroing the NVLS region failed";
            ok = false;
        }
    }
    if (!ok) {
        nvls_release(nv, devs);
        return FLUX_ERR_CUDA;
    }
    return FLUX_OK;
}

int check_directory(flux_comm* c, int from, int peer) {
    if (from < 0 || from >= c->tp || peer < 0 || peer >= c->tp)
        return fail(FLUX_ERR_DIRECTORY, "directory lookup out of range: rank " + S(from) + " -> peer " + S(peer));
    if (!c->directory[from][peer] || c->ranks[peer].heap == nullptr)
        return fail(FLUX_ERR_DIRECTORY,
                    "missing peer buffer: rank " + S(from) + " has no directory entry for peer " + S(peer));
    return FLUX_OK;
}

int init_rank_streams(RankState& r) {
    FLUX_CUDA(cudaSetDevice(r.device));
    FLUX_CUDA(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
    FLUX_CUDA(cudaStreamCreateWithFlags(&r.copy_stream, cudaStreamNonBlocking));
    FLUX_CUDA(cudaEventCreateWithFlags(&r.start_evt, cudaEventDisableTiming));
    FLUX_CUDA(cudaEventCreateWithFlags(&r.kernel_evt, cudaEventDisableTiming));
    FLUX_CUDA(cudaEventCreateWithFlags(&r.copy_evt, cudaEventDisableTiming));
    return FLUX_OK;
}

int alloc_heap(RankState& r, size_t bytes) {
    FLUX_CUDA(cudaSetDevice(r.device));
    void* p = nullptr;
    FLUX_CUDA(cudaMalloc(&p, bytes));
    FLUX_CUDA(cudaMemset(p, 0, bytes));
    FLUX_CUDA(cudaDeviceSynchronize());
    r.heap = static_cast<char*>(p);
    r.owned = true;
    return FLUX_OK;
}

// Host-mapped, zeroed error mirror ([tp][4] u32; UVA: the host pointer is the
// device address).
int alloc_err_host(flux_comm* c) {
    void* h = nullptr;
    FLUX_CUDA(cudaHostAlloc(&h, sizeof(uint32_t) * 8 * kMaxRanks, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(h, 0, sizeof(uint32_t) * 8 * kMaxRanks);
    c->err_host = static_cast<uint32_t*>(h);
    return FLUX_OK;
}

template <class T>
T* at(const RankState& r, size_t off) {
    return reinterpret_cast<T*>(r.heap + off);
}

int make_tmap(CUtensorMap* m, const void* base, int rows, int cols, int ld, int box_rows) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = driver().encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FLUX_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + S(r) + ")");
    return FLUX_OK;
}

int sm_count(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
    return v;
}

// Ranks this process drives, grouped by device (one fused launch per device).
std::vector<std::vector<int>> device_groups(flux_comm* c) {
    std::vector<std::vector<int>> groups;
    std::vector<int> devs;
    for (int r = 0; r < c->tp; ++r) {
        if (!c->ranks[r].local) continue;
        auto it = std::find(devs.begin(), devs.end(), c->ranks[r].device);
        if (it == devs.end()) {
            devs.push_back(c->ranks[r].device);
            groups.push_back({r});
        } else {
            groups[it - devs.begin()].push_back(r);
        }
    }
    return groups;
}

cudaStream_t stream_for(flux_comm* c, int rank, void* const* streams) {
    if (streams) {
        const int idx = c->ipc ? 0 : rank;
        if (streams[idx]) return static_cast<cudaStream_t>(streams[idx]);
    }
    return c->ranks[rank].stream;
}

// Tile schedules are immutable: upload each distinct table once per device and
// reuse it (no host sync on the launch path).
int mark_op_done(flux_comm* c, void* const* streams, uint32_t e) {
    if (!c->ipc || c->graph_ipc) return FLUX_OK;  // graph-safe: device barriers order the operators
    for (int r = 0; r < c->tp; ++r) {
        if (!c->ranks[r].local) continue;
        FLUX_CUDA(cudaSetDevice(c->ranks[r].device));
        cudaStream_t s = stream_for(c, r, streams);
        FLUX_TRY(write_value(s, c->ranks[r].heap + kCtrlDone, e));
        FLUX_TRY(write_value(s, c->ranks[r].heap + kCtrlKdone, e));
    }
    return FLUX_OK;
}

constexpr size_t kOrderCacheCap = 256;

uint64_t fnv1a(const std::vector<uint32_t>& v) {
    uint64_t h = 1469598103934665603ull ^ v.size();
    for (uint32_t x : v) {
        h ^= x;
        h *= 1099511628211ull;
    }
    return h;
}

void free_order_entry(flux_comm::OrderEntry& e) {
    cudaSetDevice(e.device);
    if (e.dev) cudaFree(e.dev);  // synchronises the device: no enqueued kernel still reads it
    if (e.staged) cudaFreeHost(e.staged);
    e.dev = nullptr;
    e.staged = nullptr;
}

// Device copy of a schedule table for `device`, uploaded asynchronously on
// `stream` (from a pinned copy that lives as long as the entry) on first use.
// A miss costs one cudaMalloc; no host synchronisation on the launch path, and
// a miss during CUDA-graph capture becomes a memcpy node of the graph (the
// entry is then never evicted).
int upload_order(flux_comm* c, int device, const std::vector<uint32_t>& order, uint32_t** out, cudaStream_t stream) {
    const uint64_t h = fnv1a(order);
    ++c->order_clock;
    for (auto& e : c->order_cache) {
        if (e.device == device && e.hash == h && e.table == order) {
            e.last_use = c->order_clock;
            *out = e.dev;
            return FLUX_OK;
        }
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (stream) FLUX_CUDA(cudaStreamIsCapturing(stream, &cap));
    if (c->order_cache.size() >= kOrderCacheCap && cap == cudaStreamCaptureStatusNone) {
        size_t victim = c->order_cache.size();
        for (size_t i = 0; i < c->order_cache.size(); ++i)
            if (!c->order_cache[i].captured &&
                (victim == c->order_cache.size() || c->order_cache[i].last_use < c->order_cache[victim].last_use))
                victim = i;
        if (victim < c->order_cache.size()) {
            free_order_entry(c->order_cache[victim]);
            c->order_cache.erase(c->order_cache.begin() + static_cast<long>(victim));
        }
    }
    FLUX_CUDA(cudaSetDevice(device));
    flux_comm::OrderEntry e;
    e.device = device;
    e.hash = h;
    e.table = order;
    e.last_use = c->order_clock;
    e.captured = cap != cudaStreamCaptureStatusNone;
    const size_t bytes = std::max<size_t>(1, order.size()) * sizeof(uint32_t);
    FLUX_CUDA(cudaMalloc(&e.dev, bytes));
    FLUX_CUDA(cudaHostAlloc(&e.staged, bytes, cudaHostAllocPortable));
    if (!order.empty()) std::memcpy(e.staged, order.data(), order.size() * sizeof(uint32_t));
    FLUX_CUDA(cudaMemcpyAsync(e.dev, e.staged, bytes, cudaMemcpyHostToDevice, stream));
    *out = e.dev;
    c->order_cache.push_back(std::move(e));
    return FLUX_OK;
}

enum { kInterleaveStep = 0, kInterleaveRank = 1, kInterleaveRankTail = 2, kInterleaveBlock = 3 };

// CTAs per MMA tile: CTA pairs (256-row tiles, cta_group::2) unless ownership
// blocks only align with 128-row tiles; opts.cta_group forces 1 or 2.
int choose_cg(const flux_problem* p, const flux_opts& o) {
    if (o.cta_group == 1 || o.cta_group == 2) return o.cta_group;
    const int rpr = rows_per_rank(p);
    if (rpr % (2 * kBM) == 0) return 2;
    if (rpr % kBM == 0) return 1;
    return p->m >= 2 * kBM ? 2 : 1;
}

struct OpCommon {
    flux_opts o;
    uint64_t timeout_ns;
    int fused_reduce = 0;  // RS FusedReduce in arrival order (red.add into the owner accumulator)
    int rs_units = 0;  // RS summed by the owners' reduction units (decode-sized blocks, sub-wave problems)
    int rs_chain = 0;         // RS with every rank in one launch: chained partial sums (kernel)
    const flux_operands* ops = nullptr;  // caller-provided operands (per rank; one entry in IPC mode)
};

// Cross-process operator boundary (IPC mode): every operator stamps `done` and
// `kdone` with its epoch after its kernel, so a later operator of any kind can
// wait for "peers finished epoch e-1" regardless of what e-1 was.
int mark_op_done(flux_comm* c, void* const* streams, uint32_t e);

// Caller-provided operand views of rank r (nullptr fields = library buffers).
const flux_operands* operands_of(flux_comm* c, const OpCommon& oc, int r) {
    if (!oc.ops) return nullptr;
    return c->ipc ? &oc.ops[0] : &oc.ops[r];
}

OpCommon common_opts(const flux_opts* opts) {
    OpCommon oc;
    if (opts) oc.o = *opts;
    else flux_default_opts(&oc.o);
    double s = oc.o.wall_budget_s > 0 ? oc.o.wall_budget_s : 10.0;
    oc.timeout_ns = static_cast<uint64_t>(s * 1e9);
    return oc;
}

// Streaming decode kernel eligibility: decode-sized GEMM rows (<= 128), modes
// Plain / AG / RSUnits, K-major weights, no gated (SwiGLU) or saved / derivative
// epilogues; opts.decode_kernel: 0 auto (below), 1 never, 2 whenever eligible.
bool stream_kernel_ok(flux_comm* c, const flux_problem* p, int mode, const OpCommon& oc, int m_rows, int nslots,
                      int sk_nt, const std::vector<int>& g) {
    if (oc.o.decode_kernel == FLUX_DECODE_TILE) return false;
    if (mode != kModePlain && mode != kModeAG && mode != kModeRSUnits) return false;
    if (m_rows > 128 || m_rows < 1) return false;
    if (oc.o.activation == FLUX_ACT_SWIGLU || oc.o.activation_grad != FLUX_ACT_NONE) return false;
    if (oc.o.b_layout == FLUX_B_KN) return false;
    for (int r : g) {
        const flux_operands* ops = operands_of(c, oc, r);
        if (ops && ops->aux.ptr) return false;
    }
    if (static_cast<long long>(nslots) * sk_nt > kSkCtrCap / 2) return false;
    // 32-bit stream-K arithmetic on the device: work x (CTAs + 1) < 2^31.
    const long long work = static_cast<long long>(nslots) * sk_nt * ((local_k(p) + kBK - 1) / kBK);
    if (work * (sm_count(c->ranks[g[0]].device) + 1) >= (1LL << 31)) return false;
    if (mode == kModeRSUnits && static_cast<size_t>(sk_nt) * p->tp > kRsFlagCap) return false;
    // GEMM-RS finishes a tile's owner rows in the epilogue that completed it, after
    // the other sources' flags. With one rank per launch every CTA walks tiles in
    // increasing n-tile order on every rank, so the waits form no cycle. With
    // several ranks in one launch and CTAs holding more than one tile, a CTA's
    // range wraps from one slot's last tiles to the next slot's first (a wait on
    // tile 63 of every slot ahead of tile 0 of the next): that mix stays on the
    // tile kernel (its owner units never block the GEMM).
    if (mode == kModeRSUnits && nslots > 1 && static_cast<long long>(nslots) * sk_nt > sm_count(c->ranks[g[0]].device))
        return false;
    if (std::getenv("FLUX_STREAM_KERNEL")) return std::atoi(std::getenv("FLUX_STREAM_KERNEL")) != 0;  // A/B
    if (oc.o.decode_kernel == FLUX_DECODE_STREAM) return true;
    // Auto: one rank per GPU (the deployed TP layout) with at most 64 rows. Measured
    // (scripts/stream_check.py, one GPU's Llama-2-70B TP=8 decode share, L2 flushed):
    // M=16 AG up-proj 37.9 -> 29.7 us, RS down-proj 52.2 -> 44.0, RS attn-out 48.2 ->
    // 37.9; M=64 35.8 -> 31.7; at M=128, and with eight ranks emulated in one launch,
    // the tile kernel was as fast or faster. Up to 128 rows since the GEMM-RS finish
    // keeps four row groups per thread in flight and the cluster reduction is
    // spread over the cluster with compact slots (one GPU's share at M=128,
    // scripts/rs_ab.py, tile / stream: RS attn-out 42.0 / 35.8 us, RS down-proj
    // 52.2 / 42.0, AG up-proj 33.8 / 29.7).
    return nslots == 1 && m_rows <= 128;
}

// Launch one fused kernel per device group. `mode` selects the role.
int launch_groups(flux_comm* c, const flux_problem* p, int mode, const OpCommon& oc, void* const* streams,
                  const std::vector<std::vector<uint32_t>>& seq_of_rank, int rpct, int interleave,
                  int cg, bool plain_on_agg = false, long long partial_off = -1, int rs_tail = 0,
                  const std::function<int(const std::vector<int>&, GemmParams&)>& extra = nullptr) {
    const bool plain_f32_to_staging = partial_off >= 0;
    const Layout L = layout_for(p);
    const int lk = local_k(p), lc = local_cols(p);
    const int m_rows = p->m;  // per-rank GEMM rows (AG: gathered m; RS: full m)
    auto groups = device_groups(c);
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        const auto& g = groups[gi];
        if (g.size() > static_cast<size_t>(kMaxRanks)) return fail(FLUX_ERR_CONFIG, "too many ranks on one device");
        const int dev = c->ranks[g[0]].device;
        FLUX_CUDA(cudaSetDevice(dev));
        cudaStream_t lead = stream_for(c, g[0], streams);
        GemmParams prm;
        std::memset(&prm, 0, sizeof(prm));
        // Streaming decode kernel (flux_stream_kernel) for decode-sized M.
        const int sk_mp = std::max(16, (m_rows + 15) / 16 * 16);
        const int sk_nt = (lc + kSkRows - 1) / kSkRows;
        const bool use_stream = stream_kernel_ok(c, p, mode, oc, m_rows, static_cast<int>(g.size()), sk_nt, g);
        const int a_box = use_stream ? sk_mp : kBM, b_box = use_stream ? kSkRows : kBN / cg;
        for (size_t li = 0; li < g.size(); ++li) {
            const RankState& rs = c->ranks[g[li]];
            const flux_operands* ops = operands_of(c, oc, g[li]);
            // AG at tp = 1: the gathered A is the rank's own shard; the GEMM reads it
            // there and waits for nothing (the shard still lands in a_agg).
            const bool direct = mode == kModeAG && p->tp == 1;
            const Region& A = ((mode == kModeAG && !direct) || plain_on_agg) ? L.a_agg : L.a_shard;
            if (mode == kModeAG && !direct && oc.o.nvls == FLUX_NVLS_MULTICAST)  // a_agg in the NVLS region
                FLUX_TRY(make_tmap(&prm.tma_a[li], reinterpret_cast<char*>(c->nvls.uc[g[li]]) + kNvlsDataOffset, A.rows,
                                   lk, A.ld, a_box));
            else if (A.off == L.a_shard.off && ops && ops->a.ptr)
                FLUX_TRY(make_tmap(&prm.tma_a[li], ops->a.ptr, A.rows, lk, ops->a.ld, a_box));
            else
                FLUX_TRY(make_tmap(&prm.tma_a[li], rs.heap + A.off, A.rows, lk, A.ld, a_box));
            if (ops && ops->b.ptr && oc.o.b_layout == FLUX_B_KN)  // [k, n]: 64 (N) x 64 (K) boxes, MN-major
                FLUX_TRY(make_tmap(&prm.tma_b[li], ops->b.ptr, lk, lc, ops->b.ld, kBK));
            else if (ops && ops->b.ptr) FLUX_TRY(make_tmap(&prm.tma_b[li], ops->b.ptr, lc, lk, ops->b.ld, b_box));
            else FLUX_TRY(make_tmap(&prm.tma_b[li], rs.heap + L.b.off, lc, lk, L.b.ld, b_box));
            if (plain_f32_to_staging) {
                prm.c[li] = rs.heap + partial_off;  // full [m, n] partial
                prm.ldc_l[li] = L.ld_stage;
            } else if (ops && ops->c.ptr) {
                prm.c[li] = ops->c.ptr;
                prm.ldc_l[li] = ops->c.ld;
            } else {
                prm.c[li] = rs.heap + L.c32.off;
                prm.ldc_l[li] = L.c32.ld;
            }
            if (mode == kModePlain || mode == kModeAG) {
                prm.act = oc.o.activation;
                prm.act_grad = oc.o.activation_grad;
                if (ops && ops->aux.ptr) {
                    prm.aux[li] = ops->aux.ptr;
                    prm.ld_aux[li] = ops->aux.ld;
                    prm.aux_save = oc.o.activation_grad == FLUX_ACT_NONE ? 1 : 0;
                }
            }
            prm.global_rank[li] = g[li];
            prm.ag_flags[li] = at<uint32_t>(rs, kAgFlagOffset);
            prm.ctrl[li] = at<uint32_t>(rs, kCtrlErr);
        }
        if (mode == kModeRS || mode == kModeRSUnits) {
            for (int r = 0; r < c->tp; ++r) {
                prm.staging[r] = reinterpret_cast<float*>(c->ranks[r].heap + L.staging.off);
                prm.rs_flags[r] = at<uint32_t>(c->ranks[r], kRsFlagOffset);
                prm.fr_acc[r] = reinterpret_cast<float*>(c->ranks[r].heap + L.staging.off +
                                                         static_cast<size_t>(c->epoch & 1u) * L.stage_parity * 4);
                prm.fr_ready[r] = at<uint32_t>(c->ranks[r], kCtrlFrReady);
            }
        }
        // Interleave the per-rank sequences into one device schedule.
        std::vector<uint32_t> order;
        const size_t T = seq_of_rank[g[0]].size();
        order.reserve(T * g.size());
        // kInterleaveStep: position-major across ranks (every tile waits only on
        //   tiles at lower positions). kInterleaveRank: each rank's GEMM in turn
        //   (its operands stay L2-resident). kInterleaveRankTail: rank-major, but
        //   every rank's last `tail` tiles (its own RS block, which waits on the
        //   other ranks' partials) are moved behind all other tiles.
        auto push = [&](size_t li, size_t i) {
            const uint32_t e = seq_of_rank[g[li]][i];
            order.push_back((e & 0x0FFFFFFFu) | (uint32_t(li) << 28));
        };
        if (interleave == kInterleaveBlock && g.size() > 1) {
            // Blocks of positions, every rank's tiles of a block in turn: a
            // position's partials are complete after its block instead of after
            // the last rank's whole GEMM, so the owners' reduction (decode RS)
            // runs concurrently with later blocks. ~One wave per block.
            const char* env = std::getenv("FLUX_RS_BLOCK");
            const int clusters = std::max(1, sm_count(dev) / cg);
            size_t bs = std::max<size_t>(1, static_cast<size_t>(clusters) / g.size());
            if (env) bs = std::atoi(env) > 0 ? static_cast<size_t>(std::atoi(env)) : T;
            for (size_t i0 = 0; i0 < T; i0 += bs)
                for (size_t li = 0; li < g.size(); ++li)
                    for (size_t i = i0; i < std::min(T, i0 + bs); ++i) push(li, i);
        } else if (interleave == kInterleaveStep || g.size() == 1) {
            for (size_t i = 0; i < T; ++i)
                for (size_t li = 0; li < g.size(); ++li) push(li, i);
        } else {
            const size_t tail = interleave == kInterleaveRankTail ? std::min<size_t>(T, static_cast<size_t>(rs_tail)) : 0;
            for (size_t li = 0; li < g.size(); ++li)
                for (size_t i = 0; i < T - tail; ++i) push(li, i);
            for (size_t li = 0; li < g.size(); ++li)
                for (size_t i = T - tail; i < T; ++i) push(li, i);
        }
        uint32_t* order_dev = nullptr;
        FLUX_TRY(upload_order(c, dev, order, &order_dev, lead));
        prm.order = order_dev;
        prm.num_tiles = static_cast<int>(order.size());
        prm.ag_direct = mode == kModeAG && p->tp == 1 ? 1 : 0;
        prm.m = m_rows;
        prm.n = lc;
        prm.k = lk;
        prm.ldc = L.c32.ld;
        prm.out_f32 = oc.o.out_dtype == FLUX_F32 ? 1 : 0;
        prm.tiles_n = (lc + kBN - 1) / kBN;
        prm.tp = p->tp;
        prm.rpr = rows_per_rank(p);
        prm.rpct = rpct > 0 ? rpct : prm.rpr;
        prm.ld_stage = L.ld_stage;
        prm.stage_plane = L.stage_plane;
        prm.stage_parity = L.stage_parity;
        prm.epoch = c->epoch;
        prm.timeout_ns = oc.timeout_ns;
        prm.jitter_seed = oc.o.interleave_seed;
        prm.fused_reduce = mode == kModeRS ? oc.fused_reduce : 0;
        prm.rs_chain = mode == kModeRS ? oc.rs_chain : 0;
        prm.b_mn = oc.o.b_layout == FLUX_B_KN ? 1 : 0;
        prm.part_bf16 = (mode == kModeRS || mode == kModeRSUnits) && !oc.fused_reduce && oc.o.rs_partials == FLUX_BF16 ? 1 : 0;
        for (int q = 0; q < kMaxRanks; ++q) prm.slot_of[q] = -1;
        for (size_t li = 0; li < g.size(); ++li) prm.slot_of[g[li]] = static_cast<int>(li);
        prm.rs_units = mode == kModeRSUnits ? 1 : 0;
        // Reduction units of 16 owner rows, or 8 when 16 would give fewer than
        // four per CTA (finer units balance better; measured: decode M=256
        // 153 -> 144 us, M=512 slightly better with 16).
        {
            const int rpr = rows_per_rank(p), tiles_n_all = use_stream ? sk_nt : (lc + kBN - 1) / kBN;
            const long long units16 = static_cast<long long>(g.size()) * ((rpr + 15) / 16) * tiles_n_all;
            prm.red_rows = units16 < 4LL * sm_count(dev) ? 8 : 16;
            // Warm the units' code before the partials land (they otherwise run it
            // for the first time after the GEMM, fetched from DRAM on a cold L2) when
            // at most two ranks share the launch — one rank per GPU, C1: one GPU's
            // RS share M=128 60.6 -> 51.4 us, C1 50.2 -> 42.0 us; with eight emulated
            // ranks the dry pass competes with the GEMM (+1-2 %), so it stays off.
            prm.red_warm = g.size() <= 2 ? 1 : 0;
            if (use_stream) prm.tiles_n = sk_nt;  // RS flags per (128-column n-tile, source)
        }
        prm.red_ctr = at<uint32_t>(c->ranks[g[0]], kCtrlRedCtr);
        prm.red_exit = at<uint32_t>(c->ranks[g[0]], kCtrlRedExit);
        if (const char* env = std::getenv("FLUX_DEBUG")) prm.dbg = std::atoi(env);  // profiling ablations only
        prm.err_host = c->err_host;
        prm.fault_kind = c->act_fault_kind;
        prm.fault_rank = c->act_fault_rank;
        prm.fault_index = c->act_fault_index;
        prm.check_double = c->check_double ? 1 : 0;
        // Join the other local ranks' streams into the launch stream.
        for (size_t li = 0; li < g.size(); ++li) {
            cudaStream_t s = stream_for(c, g[li], streams);
            if (s != lead) {
                FLUX_CUDA(cudaEventRecord(c->ranks[g[li]].start_evt, s));
                FLUX_CUDA(cudaStreamWaitEvent(lead, c->ranks[g[li]].start_evt, 0));
            }
        }
        if (oc.o.trace) {
            prm.trace_cap = static_cast<uint32_t>(kTraceBytes / 16);
            for (size_t li = 0; li < g.size(); ++li) {
                RankState& rs = c->ranks[g[li]];
                prm.trace[li] = reinterpret_cast<unsigned long long*>(rs.heap + L.trace_off);
                prm.trace_cursor[li] = at<uint32_t>(rs, kCtrlTraceCursor);
                FLUX_CUDA(cudaMemsetAsync(prm.trace_cursor[li], 0, 4, lead));
            }
        }
        if (extra) FLUX_TRY(extra(g, prm));
        // Flag producers all on this GPU's SMs (not the copy engines): gpu-scope acquires.
        prm.all_local = static_cast<int>(g.size()) == p->tp && (mode != kModeAG || prm.sm_transfer) ? 1 : 0;
        // Tail split (Plain / AG): a persistent grid of W clusters runs T tiles in
        // ceil(T / W) waves; the last T mod W tiles would leave most clusters
        // idle for a whole tile, so each runs as S <= 8 K-slices instead.
        prm.tail_splits = 0;
        // GEMM-RS with owner reduction units (decode-sized blocks, sub-wave
        // problems such as one GPU's decode share) splits the same way: the
        // slices are summed before the partial is staged for its owners.
        if (!use_stream && (mode == kModePlain || mode == kModeAG || mode == kModeRSUnits) &&
            oc.o.activation != FLUX_ACT_SWIGLU) {
            const char* env = std::getenv("FLUX_TAIL_SPLIT");
            const int W = std::max(1, sm_count(dev) / cg), T = prm.num_tiles;
            const int R = T % W, kb = (lk + kBK - 1) / kBK;
            // Short K (a tile's mainloop of a few microseconds) does not pay for the
            // slices' park-and-sum: C1 (RS 1024^3, TP=2, K/TP = 512) local GEMM
            // 20.5 -> 14.4 us without the split.
            const int S = R > 0 && kb >= 24 ? std::min({kTailMaxSplits, W / R, kb}) : 1;
            if (S >= 2 && R * cg <= kTailCtrCap && R * S * cg <= kTailWsCtas && !(env && std::atoi(env) == 0)) {
                const RankState& lead_rank = c->ranks[g[0]];
                prm.tail_base = T - R;
                prm.tail_splits = S;
                prm.num_tiles = prm.tail_base + R * S;
                prm.tail_seq = ++c->launch_seq;
                prm.tail_ws = reinterpret_cast<float*>(lead_rank.heap + L.tail_ws_off);
                prm.tail_ctr = at<uint32_t>(lead_rank, kTailCtrOffset);
            }
        }
        // Every SM takes part even without a GEMM tile of its own: decode RS runs
        // reduction units, the in-kernel AllGather moves pieces (decode AG M=128:
        // 124 -> 116 us).
        const bool full = mode == kModeRSUnits || (mode == kModeAG && (prm.sm_transfer || prm.nvls));
        const int grid = full ? cg * std::max(1, sm_count(dev) / cg)
                              : cg * std::max(1, std::min(prm.num_tiles, sm_count(dev) / cg));
        // Dynamic tile scheduler (FLUX_DYN_SCHED=1): clusters fetch tiles from a
        // counter in the lead rank's control block instead of a static stride.
        if (const char* env = std::getenv("FLUX_DYN_SCHED"); env && std::atoi(env) != 0 && grid / cg > 1) {
            const RankState& lead_rank = c->ranks[g[0]];
            prm.dyn_ctr = at<uint32_t>(lead_rank, kCtrlDynCtr);
            prm.dyn_exit = at<uint32_t>(lead_rank, kCtrlDynExit);
        }
        std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
        if (c->timing) {
            if (static_cast<int>(c->kernel_events.size()) <= c->kernel_events_used) {
                std::pair<cudaEvent_t, cudaEvent_t> pr;
                FLUX_CUDA(cudaEventCreate(&pr.first));
                FLUX_CUDA(cudaEventCreate(&pr.second));
                c->kernel_events.push_back(pr);
            }
            ev = &c->kernel_events[c->kernel_events_used++];
            FLUX_CUDA(cudaEventRecord(ev->first, lead));
        }
        if (use_stream) {
            const int kbn = (lk + kBK - 1) / kBK;
            const int sms = std::max(1, sm_count(dev));
            prm.sk_mp = sk_mp;
            prm.sk_nt = sk_nt;
            prm.sk_kb = kbn;
            prm.sk_work = static_cast<long long>(g.size()) * sk_nt * kbn;
            // At most kSkMaxSegsHost K-segments per n-tile: every CTA takes at least
            // ceil(kb / (max - 1)) k-blocks.
            const long long min_run = (kbn + kSkMaxSegsHost - 2) / (kSkMaxSegsHost - 1);
            prm.sk_ctas = static_cast<int>(std::max<long long>(1, std::min<long long>(sms, prm.sk_work / min_run)));
            // Enough n-tiles for ~0.4 of the SMs: one whole tile per CTA (no K-segment
            // fixup after the stream). Measured on one GPU's Llama-2-70B TP=8 decode
            // share, M=16, L2 flushed: RS attn-out (64 tiles) 26.6 -> 18.5 us, RS
            // down-proj 32.8 -> 26.6 us; split K-segments stay for fewer tiles (AG
            // up-proj share: 28 tiles).
            const long long tiles_all = static_cast<long long>(g.size()) * sk_nt;
            if (tiles_all * 5 >= 2LL * sms && tiles_all <= sms) prm.sk_ctas = static_cast<int>(tiles_all);
            if (const char* env = std::getenv("FLUX_SK_CTAS"))  // A/B: CTAs of the stream-K partition
                prm.sk_ctas = static_cast<int>(std::max<long long>(1, std::min<long long>({sms, prm.sk_work, std::atoll(env)})));
            prm.sk_acc_cols = 16;
            while (prm.sk_acc_cols < sk_mp) prm.sk_acc_cols *= 2;
            const int stage_bytes = stream_smem_bytes(mode, sk_mp, 1) - stream_smem_bytes(mode, sk_mp, 0);
            prm.sk_cluster = 1;
            // Cluster split-K: with at most half as many n-tiles as SMs, clusters of
            // c CTAs (c = 8, 4, 2; every CTA >= 2 k-blocks) split each tile's K and
            // meet in the leader's shared memory (no global fixup round trip). Every
            // cluster must be resident at once (cross-cluster waits: AllGather pieces,
            // RS flags), checked with the occupancy API. FLUX_SK_CLUSTER=c forces c
            // (1 = off) for A/B runs.
            {
                const char* envc = std::getenv("FLUX_SK_CLUSTER");
                const int forced = envc ? std::atoi(envc) : 0;
                const bool full_grid = mode == kModeAG && (prm.sm_transfer || prm.nvls);
                for (int cl : {8, 4, 2}) {
                    if (forced > 0 && cl != forced) continue;
                    if (tiles_all * cl > sms || kbn < 2 * cl) continue;
                    int st = std::min(kSkMaxStages, (kSkSmemMax - stream_smem_bytes(mode, sk_mp, 0, cl)) / stage_bytes);
                    // Ring mode (one tile per cluster): the leader's drained stage ring holds
                    // the slots, so the dedicated buffer's stages come back (M = 64 AG:
                    // cluster of 4 with 3 -> 8 stages).
                    const int st_ring = std::min(kSkMaxStages, (kSkSmemMax - stream_smem_bytes(mode, sk_mp, 0)) / stage_bytes);
                    // Distributed ring (AG / Plain, > 16 rows, kernel `dist`): each CTA's
                    // slots hold only its own 16-row chunks (M = 128 AG: clusters of 4).
                    const int nchunk = (std::min(m_rows, sk_mp) + 15) / 16;
                    const bool dist = mode != kModeRSUnits && m_rows > 16;
                    const int slot_rows = dist ? 16 * ((nchunk + cl - 1) / cl) + 4 : sk_mp + 4;
                    const bool ring = st < 8 && static_cast<long long>(st_ring) * stage_bytes >=
                                                    static_cast<long long>(cl - 1) * kSkRows * slot_rows * 4;
                    if (ring) st = st_ring;
                    if (st < 4) continue;
                    GemmParams q = prm;
                    q.sk_cluster = cl;
                    q.sk_stages = st;
                    q.sk_red_ring = ring ? 1 : 0;
                    const int maxc = stream_max_clusters(mode, q, cl, stream_smem_bytes(mode, sk_mp, st, ring ? 1 : cl));
                    const int launched = full_grid ? std::min(sms / cl, maxc) : static_cast<int>(tiles_all);
                    if (maxc < launched || launched < tiles_all) continue;
                    if (forced == 0 && tiles_all * 2 > sms) continue;  // auto: only when tiles <= SMs / 2
                    prm.sk_cluster = cl;
                    prm.sk_ctas = static_cast<int>(tiles_all) * cl;
                    prm.sk_stages = st;
                    prm.sk_red_ring = ring ? 1 : 0;
                    break;
                }
            }
            if (prm.sk_cluster == 1)
                prm.sk_stages = std::min(kSkMaxStages, (kSkSmemMax - stream_smem_bytes(mode, sk_mp, 0)) / stage_bytes);
            // AG: weight stages streamed before the gathered rows land. A few hide the
            // transfer; a full ring of them queues the transfer's own loads behind the
            // weight stream (one GPU's decode AG: rows landed 9 us in with 10 stages).
            prm.sk_pref = std::min(prm.sk_stages, 3);
            if (const char* env = std::getenv("FLUX_SK_PREFETCH")) prm.sk_pref = std::max(1, std::min(prm.sk_stages, std::atoi(env)));
            const RankState& lead_rank = c->ranks[g[0]];
            prm.tail_seq = ++c->launch_seq;
            prm.tail_ws = reinterpret_cast<float*>(lead_rank.heap + L.tail_ws_off);
            prm.sk_ctr = at<uint32_t>(lead_rank, kSkCtrOffset);
            prm.tail_splits = 0;
            // The in-kernel AllGather runs on every SM (whole clusters, all resident).
            int sgrid = (mode == kModeAG && (prm.sm_transfer || prm.nvls)) ? sms : prm.sk_ctas;
            const int smem_launch = stream_smem_bytes(mode, sk_mp, prm.sk_stages, prm.sk_red_ring ? 1 : prm.sk_cluster);
            if (prm.sk_cluster > 1 && sgrid != prm.sk_ctas)
                sgrid = std::min(sms / prm.sk_cluster, stream_max_clusters(mode, prm, prm.sk_cluster, smem_launch)) * prm.sk_cluster;
            FLUX_CUDA(launch_stream(mode, prm, sgrid, smem_launch, lead));
        } else {
            FLUX_CUDA(launch_gemm(mode, cg, prm, grid, lead));
        }
        if (ev) FLUX_CUDA(cudaEventRecord(ev->second, lead));
        ++c->last_launches;
        FLUX_CUDA(cudaEventRecord(c->ranks[g[0]].kernel_evt, lead));
        for (size_t li = 0; li < g.size(); ++li) {
            RankState& rs = c->ranks[g[li]];
            rs.kernel_evt_valid = true;
            cudaStream_t s = stream_for(c, g[li], streams);
            if (li > 0) FLUX_CUDA(cudaEventRecord(rs.kernel_evt, lead));
            if (s != lead) FLUX_CUDA(cudaStreamWaitEvent(s, c->ranks[g[0]].kernel_evt, 0));
        }
    }
    return FLUX_OK;
}

int local_ranks_only(flux_comm* c, std::vector<int>& out) {
    out.clear();
    for (int r = 0; r < c->tp; ++r)
        if (c->ranks[r].local) out.push_back(r);
    return FLUX_OK;
}

}  // namespace

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

const char* flux_last_error(void) { return g_last_error.c_str(); }
int flux_abi_version(void) { return FLUX_ABI_VERSION; }

int flux_device_sm_count(int device) { return sm_count(device); }

void flux_default_opts(flux_opts* o) {
    if (!o) return;
    o->workers_per_rank = 0;
    o->deterministic_reduce = 1;
    o->poll_budget = 10000000LL;
    o->wall_budget_s = 10.0;
    o->interleave_seed = 0;
    o->shift_offset = 1;
    o->out_dtype = FLUX_BF16;
    o->emulated_order = 0;
    o->cta_group = 0;
    o->ag_engine = 0;
    o->trace = 0;
    o->activation = FLUX_ACT_NONE;
    o->activation_grad = FLUX_ACT_NONE;
    o->rs_partials = FLUX_F32;
    o->b_layout = FLUX_B_NK;
    o->graph_safe = 0;
    o->decode_kernel = FLUX_DECODE_AUTO;
    o->nvls = FLUX_NVLS_OFF;
}

int flux_problem_validate(const flux_problem* problem, const flux_tile* tile) {
    if (!tile) return validate_problem(problem);
    return validate_tiling(problem, tile);
}

int flux_grid_for(const flux_problem* p, const flux_tile* t, int* tile_rows, int* tile_cols, int* row_blocks) {
    FLUX_TRY(validate_tiling(p, t));
    if (tile_rows) *tile_rows = p->m / t->tm;
    if (tile_cols) *tile_cols = local_cols(p) / t->tn;
    if (row_blocks) *row_blocks = p->tp;
    return FLUX_OK;
}

int flux_map_tile(int kind, int rank, int tp, int shift_offset, const int* arrival_blocks, int n_arrival,
                  int tile_rows, int tile_cols, int row_blocks, int index, int* out_row, int* out_col) {
    const int tiles = tile_rows * tile_cols;
    if (index < 0 || index >= tiles)
        return fail(FLUX_ERR_BOUNDS, "tile index " + S(index) + " out of range [0," + S(tiles) + ")");
    if (kind == FLUX_SWIZZLE_NAIVE) {  // map_tile Naive: row-major (swizzle.cpp:54-56)
        *out_row = index / tile_cols;
        *out_col = index % tile_cols;
        return FLUX_OK;
    }
    if (kind != FLUX_SWIZZLE_RANK_SHIFTED && kind != FLUX_SWIZZLE_ARRIVAL_ALIGNED)
        return fail(FLUX_ERR_CONFIG, "unknown swizzle kind");
    if (row_blocks != tp) return fail(FLUX_ERR_CONFIG, "grid row blocks != policy tp");
    std::vector<int> arrival(arrival_blocks ? arrival_blocks : nullptr,
                             arrival_blocks ? arrival_blocks + n_arrival : nullptr);
    const std::vector<int> blocks = block_order(kind, rank, tp, shift_offset, arrival);
    if (static_cast<int>(blocks.size()) != row_blocks)
        return fail(FLUX_ERR_CONFIG, "arrival block list does not cover the grid (" + S(blocks.size()) +
                                         " blocks for " + S(row_blocks) + ")");
    const int rpb = tile_rows / row_blocks, per_block = rpb * tile_cols;
    const int block = blocks[index / per_block];
    const int within = index % per_block;
    *out_row = block * rpb + within % rpb;  // column-major within the block (swizzle.cpp:67-72)
    *out_col = within / rpb;
    return FLUX_OK;
}

int flux_tile_order(const flux_problem* p, const flux_tile* t, int kind, int rank, int shift_offset,
                    const int* arrival_blocks, int n_arrival, int* out_rows, int* out_cols) {
    FLUX_TRY(validate_tiling(p, t));
    const int tile_rows = p->m / t->tm, tile_cols = local_cols(p) / t->tn, tiles = tile_rows * tile_cols;
    for (int i = 0; i < tiles; ++i)
        FLUX_TRY(flux_map_tile(kind, rank, p->tp, shift_offset, arrival_blocks, n_arrival, tile_rows, tile_cols, p->tp,
                               i, &out_rows[i], &out_cols[i]));
    return FLUX_OK;
}

int flux_validate_comm_spec(const flux_problem* p, int rank, int rows_per_comm_tile, int transfer, const int* peer,
                            const int* row_begin, const int* rows, int count) {
    FLUX_TRY(validate_problem(p));
    if (rank < 0 || rank >= p->tp) return fail(FLUX_ERR_CONFIG, "rank " + S(rank) + " >= tp");
    if (transfer != FLUX_PULL && transfer != FLUX_PUSH) return fail(FLUX_ERR_CONFIG, "unknown transfer mode");
    std::vector<Desc> order;
    for (int i = 0; i < count; ++i) order.push_back({peer[i], row_begin[i], rows[i]});
    return validate_comm_spec(p, rank, rows_per_comm_tile, transfer, order);
}

int flux_comm_order(int rank, int tp, int rpr, int rpct, int* out_peer, int* out_row_begin, int* out_rows, int max,
                    int* count) {
    if (rank < 0 || rank >= tp) return fail(FLUX_ERR_CONFIG, "rank " + S(rank) + " >= tp");
    if (rpct <= 0 || rpr % rpct != 0)
        return fail(FLUX_ERR_CONFIG, "rows_per_comm_tile=" + S(rpct) + " must divide rows_per_rank=" + S(rpr));
    std::vector<Desc> o = ring_order(rank, tp, rpr, rpct);
    const int n = std::min<int>(max, static_cast<int>(o.size()));
    for (int i = 0; i < n; ++i) {
        out_peer[i] = o[i].peer;
        out_row_begin[i] = o[i].row_begin;
        out_rows[i] = o[i].rows;
    }
    if (count) *count = static_cast<int>(o.size());
    return FLUX_OK;
}

int flux_make_comm_spec(const flux_problem* p, int rank, int rpct, int transfer, int* out_peer, int* out_row_begin,
                        int* out_rows, int max, int* count) {
    std::vector<Desc> o;
    FLUX_TRY(make_spec(p, rank, rpct, transfer, o));
    const int n = std::min<int>(max, static_cast<int>(o.size()));
    for (int i = 0; i < n; ++i) {
        out_peer[i] = o[i].peer;
        out_row_begin[i] = o[i].row_begin;
        out_rows[i] = o[i].rows;
    }
    if (count) *count = static_cast<int>(o.size());
    return FLUX_OK;
}

size_t flux_required_heap_bytes(const flux_problem* p) {
    if (validate_problem(p) != FLUX_OK) return 0;
    return layout_for(p).total;
}

size_t flux_nvls_required_bytes(const flux_problem* p) {
    if (validate_problem(p) != FLUX_OK) return 0;
    const Layout L = layout_for(p);
    const size_t data = p->pattern == FLUX_ALLGATHER_GEMM ? L.a_agg.bytes() : static_cast<size_t>(2) * L.stage_parity * 4;
    return kNvlsDataOffset + data;
}

int flux_nvls_probe(int n, const int* devices, char* why, int why_len) {
    std::string msg;
    int ok = 0;
    if (n < 1 || n > kMaxRanks || !devices) {
        msg = "need 1..8 devices";
    } else if (!driver().ok) {
        msg = "no CUDA driver";
    } else {
        std::vector<int> devs(devices, devices + n);
        flux_comm::Nvls nv;
        if (nvls_create(nv, devs, size_t(2) << 20, msg) == FLUX_OK) {
            ok = 1;
            msg = "ok";
            nvls_release(nv, devs);
        }
    }
    if (why && why_len > 0) {
        std::strncpy(why, msg.c_str(), static_cast<size_t>(why_len) - 1);
        why[why_len - 1] = 0;
    }
    return ok;
}

int flux_comm_nvls(const flux_comm* c) { return c && c->nvls.mc ? 1 : 0; }

// NVLS for one process per GPU: the multicast object is created by rank 0 and
// its POSIX file-descriptor handle passed to the peers by the caller (a Unix
// socket with SCM_RIGHTS, comm.py); each rank then adds its GPU, and once every
// rank has (the caller's barrier), binds its own VMM memory and maps the region.
static int nvls_ipc_geometry(flux_comm* c, size_t want, size_t* bytes, size_t* gran) {
    NvlsDriver& d = nvls_driver();
    if (!d.ok) return fail(FLUX_ERR_CUDA, "NVLS unavailable: multicast / VMM driver entry points unavailable");
    if (!c || !c->ipc || !c->connected) return fail(FLUX_ERR_CONFIG, "NVLS IPC setup needs a connected IPC communicator");
    if (c->tp < 2) return fail(FLUX_ERR_CONFIG, "NVLS unavailable: needs tp >= 2");
    if (c->nvls.mc_handle) return fail(FLUX_ERR_CONFIG, "the communicator already has an NVLS region");
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = static_cast<unsigned>(c->tp);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = std::max<size_t>(want, 1);
    CUresult e = d.mc_gran(gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (e != CUDA_SUCCESS) return fail(FLUX_ERR_CUDA, "NVLS unavailable: cuMulticastGetGranularity: " + cu_err(e));
    *gran = std::max<size_t>(*gran, size_t(2) << 20);
    *bytes = (std::max<size_t>(want, 1) + *gran - 1) / *gran * *gran;
    return FLUX_OK;
}

int flux_comm_nvls_ipc_export(flux_comm* c, size_t want, int* fd_out) {
    size_t bytes = 0, gran = 0;
    FLUX_TRY(nvls_ipc_geometry(c, want, &bytes, &gran));
    if (c->my_rank != 0 || !fd_out) return fail(FLUX_ERR_CONFIG, "rank 0 creates and exports the multicast object");
    NvlsDriver& d = nvls_driver();
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = static_cast<unsigned>(c->tp);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    CUmemGenericAllocationHandle h = 0;
    CUresult e = d.mc_create(&h, &mp);
    if (e != CUDA_SUCCESS) return fail(FLUX_ERR_CUDA, "NVLS unavailable: cuMulticastCreate: " + cu_err(e));
    int fd = -1;
    e = d.export_handle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (e != CUDA_SUCCESS) {
        d.mem_release(h);
        return fail(FLUX_ERR_CUDA, "NVLS unavailable: cuMemExportToShareableHandle: " + cu_err(e));
    }
    c->nvls = flux_comm::Nvls{};
    c->nvls.bytes = bytes;
    c->nvls.mc_handle = h;
    *fd_out = fd;
    return FLUX_OK;
}

int flux_comm_nvls_ipc_import(flux_comm* c, size_t want, int fd) {
    size_t bytes = 0, gran = 0;
    FLUX_TRY(nvls_ipc_geometry(c, want, &bytes, &gran));
    if (c->my_rank == 0) return fail(FLUX_ERR_CONFIG, "rank 0 exports the multicast object; the others import it");
    NvlsDriver& d = nvls_driver();
    CUmemGenericAllocationHandle h = 0;
    CUresult e = d.import_handle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    if (e != CUDA_SUCCESS) return fail(FLUX_ERR_CUDA, "NVLS unavailable: cuMemImportFromShareableHandle: " + cu_err(e));
    c->nvls = flux_comm::Nvls{};
    c->nvls.bytes = bytes;
    c->nvls.mc_handle = h;
    return FLUX_OK;
}

int flux_comm_nvls_ipc_add_device(flux_comm* c) {
    if (!c || !c->ipc || !c->nvls.mc_handle) return fail(FLUX_ERR_CONFIG, "no multicast object to add this GPU to");
    NvlsDriver& d = nvls_driver();
    CUdevice cd = 0;
    CUresult e = d.dev_get(&cd, c->ranks[c->my_rank].device);
    if (e == CUDA_SUCCESS) e = d.mc_add(static_cast<CUmemGenericAllocationHandle>(c->nvls.mc_handle), cd);
    if (e != CUDA_SUCCESS) return fail(FLUX_ERR_CUDA, "NVLS unavailable: cuMulticastAddDevice: " + cu_err(e));
    return FLUX_OK;
}

int flux_comm_nvls_ipc_bind(flux_comm* c) {
    if (!c || !c->ipc || !c->nvls.mc_handle) return fail(FLUX_ERR_CONFIG, "no multicast object to bind");
    NvlsDriver& d = nvls_driver();
    flux_comm::Nvls& nv = c->nvls;
    const int me = c->my_rank, dev = c->ranks[me].device;
    const size_t gran = size_t(2) << 20;
    nv.mem.assign(c->tp, 0);
    nv.uc.assign(c->tp, 0);
    std::vector<int> devs(c->tp, dev);
    auto bail = [&](CUresult e, const char* what) {
        const std::string msg = std::string("NVLS unavailable: ") + what + ": " + cu_err(e);
        nvls_release(nv, devs);
        return fail(FLUX_ERR_CUDA, msg);
    };
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle mh = 0;
    CUresult e = d.mem_create(&mh, nv.bytes, &ap, 0);
    if (e != CUDA_SUCCESS) return bail(e, "cuMemCreate");
    nv.mem[me] = mh;
    CUdeviceptr va = 0;
    if ((e = d.va_reserve(&va, nv.bytes, gran, 0, 0)) != CUDA_SUCCESS) return bail(e, "cuMemAddressReserve");
    if ((e = d.map(va, nv.bytes, 0, mh, 0)) != CUDA_SUCCESS) {
        d.va_free(va, nv.bytes);
        return bail(e, "cuMemMap");
    }
    nv.uc[me] = va;
    CUmemAccessDesc ad;
    std::memset(&ad, 0, sizeof(ad));
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = dev;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if ((e = d.set_access(va, nv.bytes, &ad, 1)) != CUDA_SUCCESS) return bail(e, "cuMemSetAccess (unicast)");
    if ((e = d.mc_bind(static_cast<CUmemGenericAllocationHandle>(nv.mc_handle), 0, mh, 0, nv.bytes, 0)) != CUDA_SUCCESS)
        return bail(e, "cuMulticastBindMem");
    nv.bound = true;
    CUdeviceptr mva = 0;
    if ((e = d.va_reserve(&mva, nv.bytes, gran, 0, 0)) != CUDA_SUCCESS) return bail(e, "cuMemAddressReserve (multicast)");
    if ((e = d.map(mva, nv.bytes, 0, static_cast<CUmemGenericAllocationHandle>(nv.mc_handle), 0)) != CUDA_SUCCESS) {
        d.va_free(mva, nv.bytes);
        return bail(e, "cuMemMap (multicast)");
    }
    nv.mc = mva;
    if ((e = d.set_access(mva, nv.bytes, &ad, 1)) != CUDA_SUCCESS) return bail(e, "cuMemSetAccess (multicast)");
    if (cudaSetDevice(dev) != cudaSuccess || cudaMemset(reinterpret_cast<void*>(va), 0, nv.bytes) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        nvls_release(nv, devs);
        return fail(FLUX_ERR_CUDA, "NVLS unavailable: zeroing the region failed");
    }
    return FLUX_OK;
}

int flux_comm_create(int tp, const int* devices, const flux_comm_opts* opts, flux_comm** out) {
    if (!out) return fail(FLUX_ERR_CONFIG, "null output");
    *out = nullptr;
    if (tp <= 0 || tp > kMaxRanks) return fail(FLUX_ERR_CONFIG, "tp must be in [1, " + S(kMaxRanks) + "]");
    FLUX_TRY(need_driver());
    auto* c = new flux_comm();
    c->tp = tp;
    c->heap_bytes = (opts && opts->heap_bytes) ? opts->heap_bytes : (size_t(1) << 30);
    c->ranks.resize(tp);
    c->directory.assign(tp, std::vector<bool>(tp, true));
    for (int r = 0; r < tp; ++r) {
        RankState& rs = c->ranks[r];
        rs.device = devices ? devices[r] : 0;
        rs.local = true;
        int rc = alloc_heap(rs, c->heap_bytes);
        if (rc == FLUX_OK && r == 0) rc = alloc_err_host(c);
        if (rc == FLUX_OK) rc = init_rank_streams(rs);
        if (rc != FLUX_OK) {
            std::string msg = g_last_error;
            flux_comm_destroy(c);
            return fail(rc, msg);
        }
    }
    // Peer access between distinct devices (NVLink P2P).
    for (int a = 0; a < tp; ++a)
        for (int b = 0; b < tp; ++b) {
            const int da = c->ranks[a].device, db = c->ranks[b].device;
            if (da == db) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, da, db);
            if (!can) {
                c->directory[a][b] = false;
                continue;
            }
            cudaSetDevice(da);
            cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) c->directory[a][b] = false;
            cudaGetLastError();
        }
    if (opts && opts->nvls_bytes > 0) {
        std::vector<int> devs(tp);
        for (int r = 0; r < tp; ++r) devs[r] = c->ranks[r].device;
        std::string why;
        const int rc = tp < 2 ? FLUX_ERR_CONFIG : nvls_create(c->nvls, devs, opts->nvls_bytes, why);
        if (rc != FLUX_OK) {
            flux_comm_destroy(c);
            return fail(rc, "NVLS unavailable: " + (tp < 2 ? std::string("needs tp >= 2") : why));
        }
    }
    c->connected = true;
    *out = c;
    return FLUX_OK;
}

int flux_comm_create_ipc(int rank, int tp, int device, const flux_comm_opts* opts, flux_comm** out) {
    if (!out) return fail(FLUX_ERR_CONFIG, "null output");
    *out = nullptr;
    if (tp <= 0 || tp > kMaxRanks) return fail(FLUX_ERR_CONFIG, "tp must be in [1, " + S(kMaxRanks) + "]");
    if (rank < 0 || rank >= tp) return fail(FLUX_ERR_CONFIG, "rank " + S(rank) + " >= tp");
    FLUX_TRY(need_driver());
    auto* c = new flux_comm();
    c->tp = tp;
    c->ipc = true;
    c->my_rank = rank;
    if (opts && opts->nvls_bytes > 0) {
        delete c;
        return fail(FLUX_ERR_CONFIG, "one process per GPU: set up NVLS with flux_comm_nvls_ipc_export / _import / "
                                     "_add_device / _bind after flux_comm_ipc_connect (nvls_bytes must be 0 here)");
    }
    c->heap_bytes = (opts && opts->heap_bytes) ? opts->heap_bytes : (size_t(1) << 30);
    c->ranks.resize(tp);
    c->directory.assign(tp, std::vector<bool>(tp, false));
    RankState& me = c->ranks[rank];
    me.device = device;
    me.local = true;
    int rc = alloc_heap(me, c->heap_bytes);
    if (rc == FLUX_OK) rc = alloc_err_host(c);
    if (rc == FLUX_OK) rc = init_rank_streams(me);
    if (rc != FLUX_OK) {
        std::string msg = g_last_error;
        flux_comm_destroy(c);
        return fail(rc, msg);
    }
    c->directory[rank][rank] = true;
    *out = c;
    return FLUX_OK;
}

size_t flux_comm_ipc_blob_bytes(void) { return sizeof(IpcBlob); }

int flux_comm_ipc_handle(flux_comm* c, void* blob) {
    if (!c || !c->ipc) return fail(FLUX_ERR_CONFIG, "not an IPC communicator");
    IpcBlob b;
    std::memset(&b, 0, sizeof(b));
    b.magic = kIpcMagic;
    b.rank = c->my_rank;
    b.tp = c->tp;
    b.device = c->ranks[c->my_rank].device;
    b.heap_bytes = c->heap_bytes;
    b.pid = static_cast<int32_t>(getpid());
    FLUX_CUDA(cudaSetDevice(b.device));
    FLUX_CUDA(cudaIpcGetMemHandle(&b.handle, c->ranks[c->my_rank].heap));
    std::memcpy(blob, &b, sizeof(b));
    return FLUX_OK;
}

int flux_ipc_blobs_check(const void* blobs, int tp, size_t heap_bytes) {
    if (!blobs || tp <= 0) return fail(FLUX_ERR_CONFIG, "bad blob set");
    for (int r = 0; r < tp; ++r) {
        IpcBlob b;
        std::memcpy(&b, static_cast<const char*>(blobs) + r * sizeof(IpcBlob), sizeof(b));
        if (b.magic != kIpcMagic) return fail(FLUX_ERR_DIRECTORY, "peer " + S(r) + " blob has a bad magic");
        if (b.rank != r) return fail(FLUX_ERR_DIRECTORY, "blob " + S(r) + " carries rank " + S(b.rank));
        if (b.tp != tp) return fail(FLUX_ERR_CONFIG, "peer " + S(r) + " has tp=" + S(b.tp) + ", expected " + S(tp));
        if (b.heap_bytes != heap_bytes)
            return fail(FLUX_ERR_CONFIG, "peer " + S(r) + " heap is " + S(b.heap_bytes) + " bytes, expected " +
                                             S(heap_bytes) + " (heaps must be symmetric)");
    }
    return FLUX_OK;
}

int flux_comm_ipc_connect(flux_comm* c, const void* blobs) {
    if (!c || !c->ipc) return fail(FLUX_ERR_CONFIG, "not an IPC communicator");
    FLUX_TRY(flux_ipc_blobs_check(blobs, c->tp, c->heap_bytes));
    FLUX_CUDA(cudaSetDevice(c->ranks[c->my_rank].device));
    for (int r = 0; r < c->tp; ++r) {
        if (r == c->my_rank) continue;
        IpcBlob b;
        std::memcpy(&b, static_cast<const char*>(blobs) + r * sizeof(IpcBlob), sizeof(b));
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(FLUX_ERR_DIRECTORY, "rank " + S(c->my_rank) + " cannot map peer " + S(r) + " heap: " +
                                                cudaGetErrorString(e));
        }
        c->ranks[r].heap = static_cast<char*>(p);
        c->ranks[r].device = b.device;
        c->ranks[r].owned = false;
        c->directory[c->my_rank][r] = true;
    }
    c->connected = true;
    return FLUX_OK;
}

int flux_comm_destroy(flux_comm* c) {
    if (!c) return FLUX_OK;
    for (int r = 0; r < c->tp; ++r) {
        RankState& rs = c->ranks[r];
        if (!rs.heap && !rs.stream) continue;
        cudaSetDevice(rs.local ? rs.device : c->ranks[c->my_rank >= 0 ? c->my_rank : r].device);
        if (rs.stream) cudaStreamSynchronize(rs.stream);
        if (rs.copy_stream) cudaStreamSynchronize(rs.copy_stream);
        if (rs.heap) {
            if (rs.owned) cudaFree(rs.heap);
            else cudaIpcCloseMemHandle(rs.heap);
        }
        if (rs.stream) cudaStreamDestroy(rs.stream);
        if (rs.copy_stream) cudaStreamDestroy(rs.copy_stream);
        if (rs.start_evt) cudaEventDestroy(rs.start_evt);
        if (rs.kernel_evt) cudaEventDestroy(rs.kernel_evt);
        if (rs.copy_evt) cudaEventDestroy(rs.copy_evt);
    }
    for (auto& e : c->order_cache) free_order_entry(e);
    for (auto& pr : c->kernel_events) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    if (c->err_host) cudaFreeHost(c->err_host);
    for (cudaEvent_t x : c->xfer_events) cudaEventDestroy(x);
    if (c->nvls.mc_handle) {
        std::vector<int> devs;
        for (int r = 0; r < c->tp; ++r) devs.push_back(c->ranks[r].device);
        nvls_release(c->nvls, devs);
    }
    delete c;
    return FLUX_OK;
}

int flux_comm_tp(const flux_comm* c) { return c ? c->tp : 0; }
int flux_comm_rank(const flux_comm* c) { return c ? c->my_rank : -1; }

int flux_comm_drop_peer(flux_comm* c, int from_rank, int peer_rank) {
    if (!c) return fail(FLUX_ERR_CONFIG, "null communicator");
    if (from_rank < 0 || from_rank >= c->tp || peer_rank < 0 || peer_rank >= c->tp)
        return fail(FLUX_ERR_DIRECTORY, "directory lookup out of range");
    c->directory[from_rank][peer_rank] = false;
    return FLUX_OK;
}

int flux_buffer(flux_comm* c, int rank, int kind, const flux_problem* p, flux_buffer_desc* out) {
    FLUX_TRY(check_comm(c));
    FLUX_TRY(validate_problem(p));
    if (p->tp != c->tp) return fail(FLUX_ERR_SHAPE, "problem tp=" + S(p->tp) + " but communicator tp=" + S(c->tp));
    if (rank < 0 || rank >= c->tp || !c->ranks[rank].local)
        return fail(FLUX_ERR_DIRECTORY, "rank " + S(rank) + " is not driven by this process");
    const Layout L = layout_for(p);
    if (L.total > c->heap_bytes)
        return fail(FLUX_ERR_SHAPE, "problem needs " + S(L.total) + " heap bytes, communicator has " + S(c->heap_bytes));
    const Region* r = nullptr;
    switch (kind) {
        case FLUX_BUF_A_SHARD: r = &L.a_shard; break;
        case FLUX_BUF_B_SHARD: r = &L.b; break;
        case FLUX_BUF_A_AGG: r = p->pattern == FLUX_ALLGATHER_GEMM ? &L.a_agg : nullptr; break;
        case FLUX_BUF_C_OUT: r = &L.c; break;
        case FLUX_BUF_STAGING: r = p->pattern == FLUX_GEMM_REDUCESCATTER ? &L.staging : nullptr; break;
        case 5: r = &L.c32; break;  // fp32 view of C
        default: return fail(FLUX_ERR_CONFIG, "unknown buffer kind " + S(kind));
    }
    if (!r) return fail(FLUX_ERR_CONFIG, "buffer kind " + S(kind) + " does not exist for this pattern");
    out->ptr = c->ranks[rank].heap + r->off;
    out->rows = r->rows;
    out->cols = r->cols;
    out->ld = r->ld;
    out->dtype = r->dtype;
    return FLUX_OK;
}

static int copy_2d(flux_comm* c, int rank, int kind, const flux_problem* p, void* host, int host_ld, void* stream,
                   bool in) {
    flux_buffer_desc d;
    FLUX_TRY(flux_buffer(c, rank, kind, p, &d));
    const size_t es = d.dtype == FLUX_F32 ? 4 : 2;
    if (host_ld < d.cols) return fail(FLUX_ERR_SHAPE, "host_ld smaller than the buffer width");
    FLUX_CUDA(cudaSetDevice(c->ranks[rank].device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->ranks[rank].stream;
    if (in)
        FLUX_CUDA(cudaMemcpy2DAsync(d.ptr, d.ld * es, host, host_ld * es, d.cols * es, d.rows, cudaMemcpyHostToDevice, s));
    else
        FLUX_CUDA(cudaMemcpy2DAsync(host, host_ld * es, d.ptr, d.ld * es, d.cols * es, d.rows, cudaMemcpyDeviceToHost, s));
    return FLUX_OK;
}

int flux_copy_in(flux_comm* c, int rank, int kind, const flux_problem* p, const void* host, int host_ld, void* stream) {
    return copy_2d(c, rank, kind, p, const_cast<void*>(host), host_ld, stream, true);
}
int flux_copy_out(flux_comm* c, int rank, int kind, const flux_problem* p, void* host, int host_ld, void* stream) {
    return copy_2d(c, rank, kind, p, host, host_ld, stream, false);
}

static int check_heap(flux_comm* c, const flux_problem* p) {
    if (p->tp != c->tp) return fail(FLUX_ERR_SHAPE, "workspace has " + S(c->tp) + " ranks, problem tp=" + S(p->tp));
    const size_t need = layout_for(p).total;
    if (need > c->heap_bytes)
        return fail(FLUX_ERR_SHAPE, "problem needs " + S(need) + " heap bytes per rank, communicator has " + S(c->heap_bytes));
    const int lc = local_cols(p), lk = local_k(p);
    if (p->m / kBM >= (1 << 14) || lc / kBN >= (1 << 14)) return fail(FLUX_ERR_CONFIG, "problem too large for the tile schedule");
    if (lk > (1 << 28)) return fail(FLUX_ERR_CONFIG, "k too large");
    return FLUX_OK;
}

// AllGather transfer engine: 1 copy engines, 2 in-kernel (the GEMM's SMs).
static bool ag_sm_engine_ok(const flux_problem* p, int transfer) {
    return (transfer == FLUX_PULL || transfer == FLUX_PUSH) && local_k(p) % 8 == 0 &&
           (p->m + kBM - 1) / kBM < static_cast<int>(kAgGroupCap);
}
static int ag_engine_for(const flux_problem* p, int transfer, int requested, int rpct = 0, int ranks_per_device = 1) {
    if (requested == 1 || requested == 2) return requested;
    // Many small comm tiles on one copy stream cost ~8 us of copy + flag-write
    // overhead each (measured: L-AG emulated, rpct 64 -> 448 copies, 3x slower):
    // move them on the SMs instead.
    const int rpr = rows_per_rank(p);
    if (rpct > 0 && ag_sm_engine_ok(p, transfer) && (p->tp - 1) * (rpr / rpct) * ranks_per_device > 128) return 2;
    // Auto: in-kernel transfers up to 32 MiB of gathered A (decode / small
    // problems: one launch, no host work per comm tile), copy engines above.
    // Measured on L-AG (64 MiB): within +-5 % of each other, the sign depending
    // on what runs around them (scripts/ab_engine.py vs bench.py round-robin).
    const size_t gathered = static_cast<size_t>(p->m) * local_k(p) * 2;
    return ag_sm_engine_ok(p, transfer) && gathered <= (size_t(32) << 20) ? 2 : 1;
}

int flux_ag_engine(const flux_problem* p, int transfer, const flux_opts* opts) {
    if (!p) return fail(FLUX_ERR_CONFIG, "null problem");
    return ag_engine_for(p, transfer, opts ? opts->ag_engine : 0);
}

// B layout contract: KN needs caller-provided B on every local rank (the
// library's B buffer is [n, k]) and whole 64-column atoms.
static int check_b_layout(flux_comm* c, const flux_problem* p, const flux_opts* opts, const flux_operands* ops) {
    if (!opts || opts->b_layout == FLUX_B_NK) return FLUX_OK;
    if (opts->b_layout != FLUX_B_KN) return fail(FLUX_ERR_CONFIG, "unknown b_layout");
    std::vector<int> mine;
    local_ranks_only(c, mine);
    for (int r : mine) {
        const flux_operands* o = ops ? (c->ipc ? ops : ops + r) : nullptr;
        if (!o || !o->b.ptr) return fail(FLUX_ERR_CONFIG, "b_layout KN needs caller-provided B ([k, n] row-major)");
    }
    if (local_cols(p) % 64 != 0) return fail(FLUX_ERR_SHAPE, "b_layout KN needs the local n to be a multiple of 64");
    return FLUX_OK;
}

// Epilogue activation contract (flux_activation, include/flux_b200.h).
static int check_activation(flux_comm* c, const flux_problem* p, const flux_opts* opts, const flux_operands* ops) {
    if (!opts) return FLUX_OK;
    const int a = opts->activation, g = opts->activation_grad;
    if (a < FLUX_ACT_NONE || a > FLUX_ACT_SWIGLU || g < FLUX_ACT_NONE || g > FLUX_ACT_SWIGLU)
        return fail(FLUX_ERR_CONFIG, "unknown activation");
    if (a == FLUX_ACT_NONE && g == FLUX_ACT_NONE) return FLUX_OK;
    if (a != FLUX_ACT_NONE && g != FLUX_ACT_NONE) return fail(FLUX_ERR_CONFIG, "activation and activation_grad are exclusive");
    if (p->pattern != FLUX_ALLGATHER_GEMM)
        return fail(FLUX_ERR_CONFIG, "epilogue activations belong to the AllGather-GEMM (the GEMM-RS partials are pre-reduction)");
    std::vector<int> mine;
    local_ranks_only(c, mine);
    for (size_t i = 0; i < mine.size(); ++i) {
        const flux_operands* o = ops ? (c->ipc ? ops : ops + mine[i]) : nullptr;
        const bool aux = o && o->aux.ptr;
        if (g != FLUX_ACT_NONE && !aux) return fail(FLUX_ERR_CONFIG, "activation_grad needs the saved pre-activation (operands.aux)");
    }
    if (a == FLUX_ACT_SWIGLU && local_cols(p) % kBN != 0)
        return fail(FLUX_ERR_SHAPE, "SWIGLU needs n/tp % 256 == 0 (128 gate + 128 up columns per group)");
    if (g == FLUX_ACT_SWIGLU && local_cols(p) % (kBN / 2) != 0)
        return fail(FLUX_ERR_SHAPE, "SWIGLU backward needs n/tp % 128 == 0 (C and aux hold 2n/tp grouped columns)");
    return FLUX_OK;
}

// ---------------------------------------------------------------------------
// CUDA-graph-safe operators (flux_opts.graph_safe). Between operators the host
// tracks device state: epoch-stamped flags, the in-kernel AllGather's monotonic
// piece counters (targets scale with the operators run since their reset) and
// the tail-split counters' launch tags. A replayed graph repeats the epoch and
// targets it was captured with, so a graph-safe operator zeroes the words it
// uses before its kernel: flags stamped by eager operators since the capture
// carry later epochs and would satisfy the replay's waits. Nothing is needed
// afterwards: its stamps carry an epoch older than any later eager operator's,
// the in-kernel AllGather runs on a separate counter set (kAgCtrGraphOffset,
// target = one operator's pieces), tail-split tags differ per eager launch and
// the work counters re-arm themselves. No host stream memops are issued:
// AllGather runs on the in-kernel transfer engine.
// ---------------------------------------------------------------------------
static int ag_gemm_impl(flux_comm* c, const flux_problem* p, const flux_tile* tile, int rpct, int transfer,
                        int swizzle_on, const flux_opts* opts, void* const* streams, const flux_operands* operands,
                        const std::vector<std::vector<Desc>>* custom = nullptr);
static int gemm_rs_impl(flux_comm* c, const flux_problem* p, const flux_tile* tile, int write_mode, int swizzle_on,
                        const flux_opts* opts, void* const* streams, const flux_operands* operands);
static int local_gemm_impl(flux_comm* c, const flux_problem* p, const flux_opts* opts, void* const* streams);

static int graph_zero(flux_comm* c, const flux_problem* p, void* const* streams) {
    ZeroParams z;
    std::memset(&z, 0, sizeof(z));
    auto add = [&](size_t off, size_t bytes) {
        z.off[z.nranges] = static_cast<uint32_t>(off);
        z.bytes[z.nranges] = static_cast<uint32_t>(bytes);
        ++z.nranges;
    };
    // ready / done / kdone / fr_ready / trace / work counters; across processes the
    // first four are the eager operators' cross-process epoch stamps and stay.
    if (c->ipc) add(kCtrlTraceCursor, kCtrlRedExit + 4 - kCtrlTraceCursor);
    else add(kCtrlReady, kCtrlRedExit + 4 - kCtrlReady);
    add(kAgFlagOffset, std::min<size_t>(kAgFlagCap, static_cast<size_t>(p->m)) * 4);
    add(kAgCtrGraphOffset, (static_cast<size_t>((p->m + kBM - 1) / kBM) + 1) * 4);
    add(kTailCtrOffset, static_cast<size_t>(2 * kTailCtrCap) * 4);  // arrival + RS-units staged counters
    add(kSkCtrOffset, static_cast<size_t>(kSkCtrCap) * 4);  // streaming decode kernel's n-tile counters
    if (p->pattern == FLUX_GEMM_REDUCESCATTER) {
        // Flags per (tile, source): 128 x 256 tiles, or 128-column n-tiles (streaming kernel).
        const size_t tiles = std::max(static_cast<size_t>((p->m + kBM - 1) / kBM) * ((p->n + kBN - 1) / kBN),
                                      static_cast<size_t>((p->n + kSkRows - 1) / kSkRows));
        add(kRsFlagOffset, std::min(kRsFlagCap, tiles * p->tp) * 4);
    }
    for (const auto& g : device_groups(c)) {
        ZeroParams zg = z;
        for (size_t li = 0; li < g.size(); ++li) zg.heap[li] = c->ranks[g[li]].heap;
        FLUX_CUDA(cudaSetDevice(c->ranks[g[0]].device));
        FLUX_CUDA(launch_zero_ranges(zg, static_cast<int>(g.size()), stream_for(c, g[0], streams)));
    }
    return FLUX_OK;
}

// Validates a graph-safe request and returns the options the operator runs with.
static int graph_opts(flux_comm* c, const flux_problem* p, const flux_opts* opts, int transfer, flux_opts* out) {
    if (opts) *out = *opts;
    else flux_default_opts(out);
    if (!out->graph_safe) return FLUX_OK;
    FLUX_TRY(check_comm(c));
    if (!p) return fail(FLUX_ERR_CONFIG, "null problem");
    if (p->pattern == FLUX_ALLGATHER_GEMM && transfer >= 0) {
        if (out->ag_engine == 1 || !ag_sm_engine_ok(p, transfer))
            return fail(FLUX_ERR_CONFIG, "graph_safe AllGather needs the in-kernel transfer engine (k % 8 == 0)");
        out->ag_engine = 2;
    }
    return FLUX_OK;
}

// Every operator runs between begin_op (pending device failure check, fault
// activation) and end_op (host-detected failures).
static int run_op(flux_comm* c, const std::function<int()>& body) {
    FLUX_TRY(begin_op(c));
    const int rc = body();
    if (rc != FLUX_OK) {
        if (c->act_fault_kind != 0) c->ag_sig = 0;
        c->act_fault_kind = 0;
        return rc;
    }
    return end_op(c);
}

// NVLS operator checks (opts.nvls) and the fields every NVLS launch carries.
static int nvls_check(flux_comm* c, const flux_problem* p, const flux_opts& o) {
    if (o.nvls != FLUX_NVLS_MULTICAST && o.nvls != FLUX_NVLS_EMULATED) return fail(FLUX_ERR_CONFIG, "unknown nvls mode");
    if (o.graph_safe) return fail(FLUX_ERR_CONFIG, "graph_safe operators do not use NVLS");
    if (o.nvls == FLUX_NVLS_MULTICAST) {
        if (!c->nvls.mc)
            return fail(FLUX_ERR_CONFIG, "FLUX_NVLS_MULTICAST needs a communicator created with nvls_bytes > 0");
        const size_t need = flux_nvls_required_bytes(p);
        if (need > c->nvls.bytes)
            return fail(FLUX_ERR_SHAPE, "problem needs " + S(need) + " NVLS bytes per rank, communicator has " + S(c->nvls.bytes));
    }
    return FLUX_OK;
}

// Regions of every rank the NVLS protocol addresses: the multicast region
// (nvls = 1), or the regular heap buffers of the same role (nvls = 2).
static void nvls_fill(flux_comm* c, const flux_problem* p, const flux_opts& o, GemmParams& prm) {
    const Layout L = layout_for(p);
    prm.nvls = o.nvls;
    const bool hw = o.nvls == FLUX_NVLS_MULTICAST;
    for (int q = 0; q < p->tp; ++q) {
        char* base = hw ? reinterpret_cast<char*>(q < static_cast<int>(c->nvls.uc.size()) ? c->nvls.uc[q] : 0)
                        : c->ranks[q].heap;
        if (!base) {  // a peer's region in another process: reached only through the multicast address
            prm.nvls_data[q] = nullptr;
            prm.nvls_flags[q] = nullptr;
            continue;
        }
        const size_t data = hw ? kNvlsDataOffset : (p->pattern == FLUX_ALLGATHER_GEMM ? L.a_agg.off : L.staging.off);
        prm.nvls_data[q] = base + data;
        prm.nvls_flags[q] = reinterpret_cast<uint32_t*>(base + (hw ? kNvlsFlagOffset : kAgFlagOffset));
    }
    prm.nvls_data_mc = hw ? reinterpret_cast<char*>(c->nvls.mc) + kNvlsDataOffset : nullptr;
    prm.nvls_flags_mc = hw ? reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c->nvls.mc) + kNvlsFlagOffset) : nullptr;
    prm.nvls_ld_bytes = static_cast<long long>(L.a_agg.ld) * 2;
}

// WAR across devices before an NVLS operator: multicast stores and reductions
// touch every rank's region, so each rank's launch follows every peer's
// previous kernel (in-process peers on other GPUs: events; other processes:
// their `done` stamp of the previous epoch).
static int nvls_war(flux_comm* c, const std::vector<int>& mine, void* const* streams, uint32_t e) {
    for (int r : mine) {
        RankState& rs = c->ranks[r];
        FLUX_CUDA(cudaSetDevice(rs.device));
        cudaStream_t s = stream_for(c, r, streams);
        for (int q = 0; q < c->tp; ++q) {
            if (q == r) continue;
            if (!c->ranks[q].local) FLUX_TRY(wait_value_geq(s, c->ranks[q].heap + kCtrlDone, e - 1));
            else if (c->ranks[q].device != rs.device && c->ranks[q].kernel_evt_valid)
                FLUX_CUDA(cudaStreamWaitEvent(s, c->ranks[q].kernel_evt, 0));
        }
    }
    return FLUX_OK;
}

static int ag_gemm_ex_body(flux_comm* c, const flux_problem* p, const flux_tile* tile, int rpct, int transfer,
                           int swizzle_on, const flux_opts* opts, void* const* streams, const flux_operands* operands);
static int gemm_rs_ex_body(flux_comm* c, const flux_problem* p, const flux_tile* tile, int write_mode, int swizzle_on,
                           const flux_opts* opts, void* const* streams, const flux_operands* operands);
static int local_gemm_body(flux_comm* c, const flux_problem* p, const flux_opts* opts, void* const* streams);
static int nonoverlap_body(flux_comm* c, const flux_problem* p, const flux_opts* opts, void* const* streams);
static int medium_grained_body(flux_comm* c, const flux_problem* p, const flux_tile* tile, int partitions,
                               const flux_opts* opts, void* const* streams);

int flux_ag_gemm_ex(flux_comm* c, const flux_problem* p, const flux_tile* tile, int rpct, int transfer, int swizzle_on,
                    const flux_opts* opts, void* const* streams, const flux_operands* operands) {
    return run_op(c, [&] { return ag_gemm_ex_body(c, p, tile, rpct, transfer, swizzle_on, opts, streams, operands); });
}
int flux_gemm_rs_ex(flux_comm* c, const flux_problem* p, const flux_tile* tile, int write_mode, int swizzle_on,
                    const flux_opts* opts, void* const* streams, const flux_operands* operands) {
    return run_op(c, [&] { return gemm_rs_ex_body(c, p, tile, write_mode, swizzle_on, opts, streams, operands); });
}
int flux_local_gemm(flux_comm* c, const flux_problem* p, const flux_opts* opts, void* const* streams) {
    return run_op(c, [&] { return local_gemm_body(c, p, opts, streams); });
}
int flux_nonoverlap(flux_comm* c, const flux_problem* p, const flux_opts* opts, void* const* streams) {
    return run_op(c, [&] { return nonoverlap_body(c, p, opts, streams); });
}
int flux_medium_grained(flux_comm* c, const flux_problem* p, const flux_tile* tile, int partitions,
                        const flux_opts* opts, void* const* streams) {
    return run_op(c, [&] { return medium_grained_body(c, p, tile, partitions, opts, streams); });
}

// Device-side barrier across the processes of an IPC communicator, enqueued on
// this rank's stream (monotonic counters in the control blocks, never reset).
static int rank_barrier(flux_comm* c, void* const* streams, uint32_t epoch) {
    const int me = c->my_rank;
    RankState& rs = c->ranks[me];
    FLUX_CUDA(cudaSetDevice(rs.device));
    BarrierParams b;
    std::memset(&b, 0, sizeof(b));
    b.gen = at<uint32_t>(rs, kCtrlBarGen);
    b.arr = at<uint32_t>(rs, kCtrlBarArr);
    for (int q = 0; q < c->tp; ++q) b.peer_arr[q] = at<uint32_t>(c->ranks[q], kCtrlBarArr);
    b.err = at<uint32_t>(rs, kCtrlErr);
    b.err_host = c->err_host;
    b.tp = c->tp;
    b.me = me;
    b.epoch = epoch;
    b.timeout_ns = 10000000000ull;
    FLUX_CUDA(launch_rank_barrier(b, stream_for(c, me, streams)));
    return FLUX_OK;
}

// A graph-safe operator on a one-process-per-GPU communicator. Captured in a
// CUDA graph it replays with the epoch and targets it was captured with, so
// instead of the eager operators' host stream memops (epoch stamps and waits,
// which a replay would repeat with stale values) it is bracketed by device
// barriers: A — every rank has finished its previous operator; zero this
// rank's flags and counters; B — every rank has zeroed (no peer stamps a flag
// before its owner cleared it); then the kernel. It reuses the current epoch
// (its stamps are older than any later eager operator's) and leaves the host
// epoch unchanged, so eager operators' cross-process stamps stay consistent;
// the next eager operator enters barrier A first (see eager_after_graph).
static int graph_ipc_op(flux_comm* c, const flux_problem* p, void* const* streams, const std::function<int()>& impl) {
    if (c->epoch == 0) c->epoch = 1;  // graph stamps must stay behind every later eager epoch
    const uint32_t e = c->epoch;
    FLUX_TRY(rank_barrier(c, streams, e));
    FLUX_TRY(graph_zero(c, p, streams));
    FLUX_TRY(rank_barrier(c, streams, e));
    c->graph_ipc = true;
    c->epoch = e - 1;  // the operator bumps it back to e
    const int rc = impl();
    c->graph_ipc = false;
    c->epoch = e;
    c->last_was_graph = true;
    return rc;
}

// An eager operator right after graph-safe ones (IPC): every peer has finished
// those (whose completion no epoch stamp records) before this one starts, and
// the current epoch's done stamps exist (a graph-first communicator never
// wrote them).
static int eager_after_graph(flux_comm* c, void* const* streams) {
    if (!c->ipc || c->graph_ipc || !c->last_was_graph) return FLUX_OK;
    FLUX_TRY(rank_barrier(c, streams, c->epoch + 1));
    FLUX_TRY(mark_op_done(c, streams, c->epoch));
    c->last_was_graph = false;
    return FLUX_OK;
}

static int ag_gemm_ex_body(flux_comm* c, const flux_problem* p, const flux_tile* tile, int rpct, int transfer,
                           int swizzle_on, const flux_opts* opts, void* const* streams, const flux_operands* operands) {
    flux_opts o;
    FLUX_TRY(graph_opts(c, p, opts, transfer, &o));
    if (!o.graph_safe) return ag_gemm_impl(c, p, tile, rpct, transfer, swizzle_on, &o, streams, operands);
    FLUX_TRY(validate_tiling(p, tile));
    FLUX_TRY(check_heap(c, p));
    if (c->ipc)
        return graph_ipc_op(c, p, streams,
                            [&] { return ag_gemm_impl(c, p, tile, rpct, transfer, swizzle_on, &o, streams, operands); });
    FLUX_TRY(graph_zero(c, p, streams));
    return ag_gemm_impl(c, p, tile, rpct, transfer, swizzle_on, &o, streams, operands);
}

static int gemm_rs_ex_body(flux_comm* c, const flux_problem* p, const flux_tile* tile, int write_mode, int swizzle_on,
                           const flux_opts* opts, void* const* streams, const flux_operands* operands) {
    flux_opts o;
    FLUX_TRY(graph_opts(c, p, opts, -1, &o));
    if (!o.graph_safe) return gemm_rs_impl(c, p, tile, write_mode, swizzle_on, &o, streams, operands);
    if (write_mode == FLUX_FUSED_REDUCE && !o.deterministic_reduce)
        return fail(FLUX_ERR_CONFIG, "graph_safe is not available with the arrival-order FusedReduce");
    FLUX_TRY(validate_tiling(p, tile));
    FLUX_TRY(check_heap(c, p));
    if (c->ipc)
        return graph_ipc_op(c, p, streams,
                            [&] { return gemm_rs_impl(c, p, tile, write_mode, swizzle_on, &o, streams, operands); });
    FLUX_TRY(graph_zero(c, p, streams));
    return gemm_rs_impl(c, p, tile, write_mode, swizzle_on, &o, streams, operands);
}

static int local_gemm_body(flux_comm* c, const flux_problem* p, const flux_opts* opts, void* const* streams) {
    flux_opts o;
    FLUX_TRY(graph_opts(c, p, opts, -1, &o));
    if (!o.graph_safe) return local_gemm_impl(c, p, &o, streams);
    FLUX_TRY(validate_problem(p));
    FLUX_TRY(check_heap(c, p));
    FLUX_TRY(graph_zero(c, p, streams));
    return local_gemm_impl(c, p, &o, streams);
}

int flux_ag_gemm(flux_comm* c, const flux_problem* p, const flux_tile* tile, int rpct, int transfer, int swizzle_on,
                 const flux_opts* opts, void* const* streams) {
    return flux_ag_gemm_ex(c, p, tile, rpct, transfer, swizzle_on, opts, streams, nullptr);
}

static int ag_gemm_impl(flux_comm* c, const flux_problem* p, const flux_tile* tile, int rpct, int transfer,
                        int swizzle_on, const flux_opts* opts, void* const* streams, const flux_operands* operands,
                        const std::vector<std::vector<Desc>>* custom) {
    FLUX_TRY(check_comm(c));
    if (p && p->pattern != FLUX_ALLGATHER_GEMM)
        return fail(FLUX_ERR_CONFIG, "run_fused_allgather_gemm requires AllGatherGemm pattern");
    FLUX_TRY(validate_tiling(p, tile));
    FLUX_TRY(check_heap(c, p));
    FLUX_TRY(check_activation(c, p, opts, operands));
    FLUX_TRY(check_b_layout(c, p, opts, operands));
    FLUX_TRY(eager_after_graph(c, streams));
    const int tp = p->tp, rpr = rows_per_rank(p);
    if (rpct <= 0) rpct = rpr;
    if (p->m / rpct > static_cast<int>(kAgFlagCap)) return fail(FLUX_ERR_CONFIG, "too many comm tiles");
    // Comm specs: the reference's (make_comm_specs) or the caller's orders for
    // the ranks this process drives (run_fused_allgather_gemm's comm_specs,
    // engine.hpp:107-111; the transfer agent walks them, engine.cpp:367-423).
    std::vector<std::vector<Desc>> specs, pull_specs;
    FLUX_TRY(default_specs(p, rpct, transfer, specs));
    std::vector<int> mine;
    local_ranks_only(c, mine);
    if (custom) {
        for (int r : mine) {
            const std::vector<Desc>& o = (*custom)[r];
            FLUX_TRY(validate_comm_spec(p, r, rpct, transfer, o));
            for (const Desc& d : o) {  // what the reference's copy_rows would reject at run time
                const int owner = d.row_begin / rpr;
                if (d.peer < 0 || d.peer >= tp || d.peer == r || (transfer == FLUX_PULL && d.peer != owner))
                    return fail(FLUX_ERR_BOUNDS, "transfer descriptor peer " + S(d.peer) + " rows [" + S(d.row_begin) +
                                                     ",+" + S(d.rows) + ") not served by that peer (rank " + S(r) + ")");
            }
            specs[r] = o;
        }
    }
    if (transfer == FLUX_PULL) pull_specs = specs;
    else FLUX_TRY(default_specs(p, rpct, FLUX_PULL, pull_specs));
    // Directory check: every peer this rank touches must be mapped (workspace.cpp:56-65).
    for (int r : mine)
        for (int q = 0; q < tp; ++q) FLUX_TRY(check_directory(c, r, q));
    OpCommon oc = common_opts(opts);
    oc.ops = operands;
    const Layout L = layout_for(p);
    c->last_launches = 0;
    c->kernel_events_used = 0;
    const uint32_t e = ++c->epoch;
    const size_t rowbytes = static_cast<size_t>(L.a_agg.ld) * 2;
    const int lk = local_k(p);

    // ---- NVLS: warp 3 of the GEMM pushes each rank's own comm tiles into every
    // rank's a_agg with multicast stores and stamps their flags on every rank;
    // the tiles wait on the flags (Alg. 2) ----
    if (oc.o.nvls != FLUX_NVLS_OFF) {
        FLUX_TRY(nvls_check(c, p, oc.o));
        if (lk % 8 != 0) return fail(FLUX_ERR_CONFIG, "NVLS AllGather needs k % 8 == 0 (16-byte multicast stores)");
        if (custom) return fail(FLUX_ERR_CONFIG, "NVLS pushes each rank's own rows to every rank at once; caller comm orders apply to the copy-engine and in-kernel transfers");
        const int cg = choose_cg(p, oc.o);
        std::vector<std::vector<uint32_t>> seq(tp);
        for (int r : mine) {
            const std::vector<int> blocks = ag_block_order(p, r, FLUX_PULL, true, pull_specs);
            seq[r] = device_sequence(p->m, local_cols(p), rpr, swizzle_on ? blocks : std::vector<int>{}, kBM * cg,
                                     group_blocks(rpr, kBM * cg, /*ag=*/true));
        }
        FLUX_TRY(nvls_war(c, mine, streams, e));
        auto extra = [&](const std::vector<int>& g, GemmParams& prm) -> int {
            nvls_fill(c, p, oc.o, prm);
            prm.sm_transfer = 0;
            prm.row_bytes = lk * 2;
            for (size_t li = 0; li < g.size(); ++li) {
                const flux_operands* ops = operands_of(c, oc, g[li]);
                prm.ag_flags[li] = prm.nvls_flags[g[li]];
                prm.shard_src[li] = ops && ops->a.ptr ? static_cast<const char*>(ops->a.ptr)
                                                      : c->ranks[g[li]].heap + L.a_shard.off;
                prm.src_ld_l[li] = static_cast<long long>(ops && ops->a.ptr ? ops->a.ld : L.a_shard.ld) * 2;
            }
            return FLUX_OK;
        };
        FLUX_TRY(launch_groups(c, p, kModeAG, oc, streams, seq, rpct, kInterleaveRank, cg, false, -1, 0, extra));
        if (c->ipc) {
            for (int r : mine) {
                FLUX_CUDA(cudaSetDevice(c->ranks[r].device));
                cudaStream_t s = stream_for(c, r, streams);
                FLUX_TRY(write_value(s, c->ranks[r].heap + kCtrlDone, e));
                FLUX_TRY(write_value(s, c->ranks[r].heap + kCtrlKdone, e));
            }
        }
        return FLUX_OK;
    }

    // ---- transfer engine: copy engines (Alg. 3 on a stream) or the GEMM's own
    // SMs (warp 3 of every CTA pulls a_agg pieces with TMA bulk copies) ----
    if (oc.o.ag_engine == 2 && !ag_sm_engine_ok(p, transfer))
        return fail(FLUX_ERR_CONFIG, "in-kernel AllGather transfer needs Pull or Push and k % 8 == 0");
    size_t per_dev = 1;
    for (const auto& dg : device_groups(c)) per_dev = std::max(per_dev, dg.size());
    const bool use_sm = ag_engine_for(p, transfer, oc.o.ag_engine, rpct, static_cast<int>(per_dev)) == 2;
    if (use_sm) {
        const int cg = choose_cg(p, oc.o);
        const int groups = (p->m + kBM - 1) / kBM;
        const size_t ctr_off = oc.o.graph_safe ? kAgCtrGraphOffset : kAgCtrOffset;
        // Piece geometry: whole contiguous rows up to kPieceBytes, or column splits of long rows.
        const int row_bytes = lk * 2;
        int piece_rows = 1, pieces_per_row = (row_bytes + kPieceBytes - 1) / kPieceBytes;
        // (Every rank must reach the same geometry: SPMD callers pass operands of one shape.)
        bool contiguous = L.a_agg.ld == lk;
        for (int r : mine) {
            const flux_operands* ops = operands_of(c, oc, r);
            if ((ops && ops->a.ptr ? ops->a.ld : L.a_shard.ld) != lk) contiguous = false;
        }
        if (row_bytes <= kPieceBytes && contiguous) {
            pieces_per_row = 1;
            while (piece_rows * 2 <= kBM && piece_rows * 2 * row_bytes <= kPieceBytes && rpr % (piece_rows * 2) == 0)
                piece_rows *= 2;
        }
        // Counters only grow: every operator adds the same pieces per group, so
        // operator number `mult` since the last reset waits for mult x target.
        // They are zeroed only when the piece layout changes (no per-op reset).
        const uint64_t sig = (static_cast<uint64_t>(p->m) << 40) ^ (static_cast<uint64_t>(lk) << 16) ^
                             (static_cast<uint64_t>(piece_rows) << 8) ^ static_cast<uint64_t>(pieces_per_row) ^
                             (static_cast<uint64_t>(tp) << 60);
        const bool graph = oc.o.graph_safe != 0;  // own counter set, zeroed by graph_zero: target x1
        const bool reset = !graph && (c->ag_sig != sig || c->ag_mult > (1u << 30) / std::max(1, kBM * pieces_per_row));
        for (int r : mine) {
            RankState& rs = c->ranks[r];
            FLUX_CUDA(cudaSetDevice(rs.device));
            cudaStream_t s = stream_for(c, r, streams);
            // WAR on my a_agg slot and counters: peers of the previous operator are done
            // (in-process peers on other devices by event, other processes by `done`).
            for (int q = 0; q < tp; ++q) {
                if (q == r) continue;
                if (!c->ranks[q].local) {
                    if (!c->graph_ipc) FLUX_TRY(wait_value_geq(s, c->ranks[q].heap + kCtrlDone, e - 1));
                } else if (c->ranks[q].device != rs.device && c->ranks[q].kernel_evt_valid) {
                    FLUX_CUDA(cudaStreamWaitEvent(s, c->ranks[q].kernel_evt, 0));
                }
            }
            if (reset) FLUX_CUDA(cudaMemsetAsync(rs.heap + ctr_off, 0, (static_cast<size_t>(groups) + 1) * 4, s));
        }
        if (reset && c->ipc) {
            // Layout change across processes: nobody may read a peer's counters
            // before that peer has zeroed them (stream-level barrier, rare).
            for (int r : mine) {
                cudaStream_t s = stream_for(c, r, streams);
                FLUX_TRY(write_value(s, c->ranks[r].heap + kCtrlReady, e));
                for (int q = 0; q < tp; ++q)
                    if (!c->ranks[q].local) FLUX_TRY(wait_value_geq(s, c->ranks[q].heap + kCtrlReady, e));
            }
        }
        if (reset) {
            c->ag_sig = sig;
            c->ag_mult = 0;
        }
        const uint32_t mult = graph ? 1u : ++c->ag_mult;
        std::vector<std::vector<uint32_t>> seq(tp);
        std::vector<std::vector<int>> blocks(tp);
        for (int r : mine) {
            // Pieces always move in arrival order (own block first, then the ring);
            // the swizzle only decides the order the tiles consume them.
            blocks[r] = ag_block_order(p, r, FLUX_PULL, true, pull_specs);
            seq[r] = device_sequence(p->m, local_cols(p), rpr, swizzle_on ? blocks[r] : std::vector<int>{}, kBM * cg,
                                     group_blocks(rpr, kBM * cg, /*ag=*/true));
        }
        const bool step_major = oc.o.emulated_order == 1;
        const bool push = transfer == FLUX_PUSH;
        std::vector<std::vector<int>> blocks_all(tp);  // every rank's consumption order (Push tables)
        if (push)
            for (int q = 0; q < tp; ++q) blocks_all[q] = ag_block_order(p, q, FLUX_PULL, true, pull_specs);
        auto extra = [&](const std::vector<int>& g, GemmParams& prm) -> int {
            // Piece table in consumption order: every slot's own block first (peers
            // copy from it), then the others in the order the tiles need them.
            std::vector<uint32_t> jobs;
            auto add_block = [&](int li, int b) {
                for (int row = b * rpr; row < (b + 1) * rpr; row += piece_rows)
                    jobs.push_back((uint32_t(li) << 28) | (uint32_t(b) << 24) | uint32_t(row));
            };
            // Ranks of this launch pull straight from each other's shards, so with
            // every peer local the table can follow the kernel's consumption order
            // exactly (rank-major: each slot's own block, then its peers').
            bool all_local = true;
            for (int q = 0; q < kMaxRanks; ++q) prm.slot_of[q] = -1;
            for (size_t li = 0; li < g.size(); ++li) prm.slot_of[g[li]] = static_cast<int>(li);
            for (int q = 0; q < tp; ++q) all_local = all_local && prm.slot_of[q] >= 0;
            if (push) {
                // Push: each local source copies its own block into every destination.
                auto add_push = [&](int src_rank, int q) {
                    for (int row = src_rank * rpr; row < (src_rank + 1) * rpr; row += piece_rows)
                        jobs.push_back((uint32_t(prm.slot_of[src_rank]) << 28) | (uint32_t(q) << 24) | uint32_t(row));
                };
                if (all_local) {
                    // Every source in this launch: follow the kernel's consumption order
                    // (destinations rank-major, each in its own block order).
                    for (size_t li = 0; li < g.size(); ++li)
                        for (int step = 0; step < tp; ++step) add_push(blocks_all[g[li]][step], g[li]);
                } else {
                    // The ring (reference push order, engine.cpp:86-95): own a_agg first.
                    for (size_t li = 0; li < g.size(); ++li)
                        for (int k2 = 0; k2 < tp; ++k2) add_push(g[li], (g[li] + k2) % tp);
                }
            } else if (step_major || !all_local) {
                for (size_t li = 0; li < g.size(); ++li) add_block(static_cast<int>(li), g[li]);
                if (step_major) {
                    for (int step = 1; step < tp; ++step)
                        for (size_t li = 0; li < g.size(); ++li) add_block(static_cast<int>(li), blocks[g[li]][step]);
                } else {
                    for (size_t li = 0; li < g.size(); ++li)
                        for (int step = 1; step < tp; ++step) add_block(static_cast<int>(li), blocks[g[li]][step]);
                }
            } else {
                for (size_t li = 0; li < g.size(); ++li)
                    for (int step = 0; step < tp; ++step) add_block(static_cast<int>(li), blocks[g[li]][step]);
            }
            uint32_t* jobs_dev = nullptr;
            FLUX_TRY(upload_order(c, c->ranks[g[0]].device, jobs, &jobs_dev, stream_for(c, g[0], streams)));
            prm.sm_transfer = 1;
            prm.ag_push = push ? 1 : 0;
            for (int q = 0; q < tp; ++q) prm.kdone[q] = at<uint32_t>(c->ranks[q], kCtrlKdone);
            prm.jobs = jobs_dev;
            prm.num_jobs = static_cast<int>(jobs.size());
            prm.piece_rows = piece_rows;
            prm.pieces_per_row = pieces_per_row;
            prm.row_bytes = row_bytes;
            prm.ag_slot_index = groups;
            prm.ag_mult = mult;
            prm.slot_pieces = static_cast<uint32_t>((rpr / piece_rows) * (piece_rows > 1 ? 1 : pieces_per_row));
            for (size_t li = 0; li < g.size(); ++li) {
                const flux_operands* ops = operands_of(c, oc, g[li]);
                prm.src_ld_l[li] = static_cast<long long>(ops && ops->a.ptr ? ops->a.ld : L.a_shard.ld) * 2;
            }
            prm.dst_ld_bytes = static_cast<long long>(L.a_agg.ld) * 2;
            for (int q = 0; q < tp; ++q) {
                prm.agg_src[q] = c->ranks[q].heap + L.a_agg.off;
                prm.ag_ctr[q] = at<uint32_t>(c->ranks[q], ctr_off);
            }
            for (size_t li = 0; li < g.size(); ++li) {
                const flux_operands* ops = operands_of(c, oc, g[li]);
                prm.shard_src[li] = ops && ops->a.ptr ? static_cast<const char*>(ops->a.ptr)
                                                      : c->ranks[g[li]].heap + L.a_shard.off;
                prm.a_dst[li] = c->ranks[g[li]].heap + L.a_agg.off;
            }
            return FLUX_OK;
        };
        FLUX_TRY(launch_groups(c, p, kModeAG, oc, streams, seq, rpct, step_major ? kInterleaveStep : kInterleaveRank,
                               cg, false, -1, 0, extra));
        if (c->ipc && !c->graph_ipc) {
            for (int r : mine) {
                FLUX_CUDA(cudaSetDevice(c->ranks[r].device));
                cudaStream_t s = stream_for(c, r, streams);
                FLUX_TRY(write_value(s, c->ranks[r].heap + kCtrlDone, e));  // my pulls of this epoch are done
                FLUX_TRY(write_value(s, c->ranks[r].heap + kCtrlKdone, e));
            }
        }
        return FLUX_OK;
    }

    // One copy-engine stream per device (several blocked stream-wait memops on
    // many streams can starve each other on shared hardware queues). It starts
    // after the caller's prior work (the A shards) and after the previous kernel
    // of every rank it serves (WAR on a_agg).
    auto groups = device_groups(c);
    for (const auto& g : groups) {
        RankState& lead = c->ranks[g[0]];
        FLUX_CUDA(cudaSetDevice(lead.device));
        for (int r : g) {
            RankState& rs = c->ranks[r];
            FLUX_CUDA(cudaEventRecord(rs.start_evt, stream_for(c, r, streams)));
            FLUX_CUDA(cudaStreamWaitEvent(lead.copy_stream, rs.start_evt, 0));
            if (rs.kernel_evt_valid) FLUX_CUDA(cudaStreamWaitEvent(lead.copy_stream, rs.kernel_evt, 0));
        }
    }

    const int cg = choose_cg(p, oc.o);
    // ---- Alg. 2: the fused GEMM, tiles ordered by expected arrival. Launched
    // first so it computes ready (local) tiles while the host enqueues Alg. 3.
    std::vector<std::vector<uint32_t>> seq(tp);
    for (int r : mine)
        seq[r] = device_sequence(p->m, local_cols(p), rpr, ag_block_order(p, r, transfer, swizzle_on != 0, specs),
                                 kBM * cg, group_blocks(rpr, kBM * cg, /*ag=*/true));
    auto launch_kernel = [&]() {
        return launch_groups(c, p, kModeAG, oc, streams, seq, rpct,
                             oc.o.emulated_order == 1 ? kInterleaveStep : kInterleaveRank, cg);
    };
    // FLUX_SERIALIZE_TRANSFERS=1 (profiling / diagnosis only): all transfers
    // complete before the kernel starts, so its flag waits never block (a
    // profiler replaying the kernel alone cannot re-run the copy engines).
    const char* ser_env = std::getenv("FLUX_SERIALIZE_TRANSFERS");
    const bool serialize = ser_env && std::atoi(ser_env) != 0;
    if (!serialize) FLUX_TRY(launch_kernel());

    // ---- Alg. 3: the transfer loop (engine.cpp:367-423) on the copy engines ----
    const size_t shard_pitch = static_cast<size_t>(L.a_shard.ld) * 2;
    auto copy_rows = [&](cudaStream_t cs, char* dst, size_t dpitch, const char* src, size_t spitch, int rows) -> int {
        const size_t width = static_cast<size_t>(lk) * 2;
        if (dpitch == width && spitch == width)
            FLUX_CUDA(cudaMemcpyAsync(dst, src, width * rows, cudaMemcpyDeviceToDevice, cs));
        else
            FLUX_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToDevice, cs));
        return FLUX_OK;
    };
    const int per_peer = rpr / rpct;
    // SignalBoard::set semantics (signal_board.hpp:25-28, engine.cpp:401-403):
    // every comm-tile flag is raised once per operator; a second set is an
    // error (the transfer loop enqueues every flag write, so the host checks).
    // Fault injection drops or doubles one flag write.
    std::vector<std::vector<uint8_t>> raised(tp, std::vector<uint8_t>(static_cast<size_t>(p->m / rpct), 0));
    auto set_flag = [&](cudaStream_t cs, int r, int f) -> int {
        const bool hit = c->act_fault_kind != 0 && c->act_fault_rank == r && c->act_fault_index == f;
        if (hit && c->act_fault_kind == FLUX_FAULT_DROP_SIGNAL) return FLUX_OK;
        for (int rep = 0; rep < (hit ? 2 : 1); ++rep) {
            if (++raised[r][f] > 1 && c->host_error.empty())
                c->host_error = "flag " + S(f) + " on rank " + S(r) + " set twice";
            FLUX_TRY(write_value(cs, at<uint32_t>(c->ranks[r], kAgFlagOffset) + f, e));
        }
        return FLUX_OK;
    };
    std::vector<std::vector<uint8_t>> waited(tp, std::vector<uint8_t>(tp, 0));
    // TransferRecord timing (opts.trace; engine.cpp:395-420): an event after
    // each descriptor's copy and after its flag write on the copy stream,
    // relative to one base event per copy stream (flux_transfer_log).
    const bool log_xfer = oc.o.trace != 0;
    if (log_xfer) {
        c->xfer_log.clear();
        c->xfer_used = 0;
    }
    auto next_event = [&](cudaEvent_t* ev) -> int {
        if (c->xfer_used == c->xfer_events.size()) {
            cudaEvent_t x;
            FLUX_CUDA(cudaEventCreate(&x));
            c->xfer_events.push_back(x);
        }
        *ev = c->xfer_events[c->xfer_used++];
        return FLUX_OK;
    };
    cudaEvent_t xfer_base = nullptr;
    auto log_copy = [&](cudaStream_t cs, int owner, const Desc& d) -> int {
        if (!log_xfer) return FLUX_OK;
        flux_comm::XferEntry x;
        x.rank = owner;
        x.peer = d.peer;
        x.row_begin = d.row_begin;
        x.rows = d.rows;
        x.base = xfer_base;
        FLUX_TRY(next_event(&x.copy_ev));
        FLUX_CUDA(cudaEventRecord(x.copy_ev, cs));
        c->xfer_log.push_back(x);
        return FLUX_OK;
    };
    auto log_flag = [&](cudaStream_t cs) -> int {
        if (!log_xfer) return FLUX_OK;
        FLUX_TRY(next_event(&c->xfer_log.back().flag_ev));
        FLUX_CUDA(cudaEventRecord(c->xfer_log.back().flag_ev, cs));
        return FLUX_OK;
    };
    for (const auto& g : groups) {
        RankState& lead = c->ranks[g[0]];
        FLUX_CUDA(cudaSetDevice(lead.device));
        cudaStream_t cs = lead.copy_stream;
        if (log_xfer) {
            FLUX_TRY(next_event(&xfer_base));
            FLUX_CUDA(cudaEventRecord(xfer_base, cs));
        }
        auto in_group = [&](int q) { return std::find(g.begin(), g.end(), q) != g.end(); };
        // Remote peers finished pulling my previous shard before I overwrite it
        // (ranks sharing this stream are ordered by the stream itself).
        if (transfer == FLUX_PULL)
            for (int r : g)
                for (int q = 0; q < tp; ++q)
                    if (q != r && !in_group(q)) FLUX_TRY(wait_value_geq(cs, c->ranks[q].heap + kCtrlDone, e - 1));
        // A rank's own shard: caller operand or library buffer. Ranks sharing
        // this device (one stream, so no cross-rank hazards) pull straight from
        // each other's shards instead of from the owner's a_agg slot: nothing
        // waits for the owners' local copies, which would otherwise serialise
        // tp local copies ahead of the first remote block.
        auto shard_of = [&](int q, const char*& ptr, size_t& pitch) {
            const flux_operands* ops = operands_of(c, oc, q);
            ptr = ops && ops->a.ptr ? static_cast<const char*>(ops->a.ptr) : c->ranks[q].heap + L.a_shard.off;
            pitch = ops && ops->a.ptr ? static_cast<size_t>(ops->a.ld) * 2 : shard_pitch;
        };
        // Local shard -> own a_agg slot, local flags preset (engine.cpp:469-472).
        auto local_copy = [&](int r) -> int {
            RankState& rs = c->ranks[r];
            const char* shard;
            size_t pitch;
            shard_of(r, shard, pitch);
            FLUX_TRY(copy_rows(cs, rs.heap + L.a_agg.off + static_cast<size_t>(r) * rpr * rowbytes, rowbytes, shard,
                               pitch, rpr));
            FLUX_TRY(write_value(cs, rs.heap + kCtrlReady, e));
            for (int f = r * rpr / rpct; f < (r + 1) * rpr / rpct; ++f) FLUX_TRY(set_flag(cs, r, f));
            return FLUX_OK;
        };
        // Transfers in the order the kernel consumes them: rank-major when the
        // ranks sharing this device run rank by rank (each rank's own block,
        // then its peers' blocks), else every own block then ring step by step.
        std::vector<std::pair<int, int>> jobs;  // (rank, step); step -1 = local copy
        const bool all_here = static_cast<int>(g.size()) == tp && oc.o.emulated_order != 1 && tp > 1;
        if (all_here) {
            // Every rank on this device and stream: Pull and Push move the same
            // rows (source shard -> destination a_agg), so issue them in exactly
            // the order the rank-major kernel consumes blocks (its block order
            // for this transfer mode and swizzle), whoever "owns" the descriptor.
            for (int cr : g) {
                FLUX_TRY(local_copy(cr));
                RankState& rs = c->ranks[cr];
                if (transfer == FLUX_PULL) {
                    // cr's comm spec in its own order (the reference transfer agent,
                    // engine.cpp:378-405; the kernel's block order follows it).
                    for (const Desc& d : specs[cr]) {
                        const char* shard;
                        size_t pitch;
                        shard_of(d.peer, shard, pitch);
                        FLUX_TRY(copy_rows(cs, rs.heap + L.a_agg.off + static_cast<size_t>(d.row_begin) * rowbytes,
                                           rowbytes, shard + static_cast<size_t>(d.row_begin - d.peer * rpr) * pitch,
                                           pitch, d.rows));
                        FLUX_TRY(log_copy(cs, cr, d));
                        FLUX_TRY(set_flag(cs, cr, d.row_begin / rpct));
                        FLUX_TRY(log_flag(cs));
                    }
                    continue;
                }
                const std::vector<int> order = ag_block_order(p, cr, transfer, swizzle_on != 0, specs);
                for (int b : order) {
                    if (b == cr) continue;
                    const std::vector<Desc>& list = transfer == FLUX_PULL ? specs[cr] : specs[b];
                    const int want_peer = transfer == FLUX_PULL ? b : cr;
                    const char* shard;
                    size_t pitch;
                    shard_of(b, shard, pitch);
                    for (const Desc& d : list) {
                        if (d.peer != want_peer) continue;
                        FLUX_TRY(copy_rows(cs, rs.heap + L.a_agg.off + static_cast<size_t>(d.row_begin) * rowbytes,
                                           rowbytes, shard + static_cast<size_t>(d.row_begin - b * rpr) * pitch, pitch,
                                           d.rows));
                        FLUX_TRY(log_copy(cs, transfer == FLUX_PULL ? cr : b, d));
                        FLUX_TRY(set_flag(cs, cr, d.row_begin / rpct));
                        FLUX_TRY(log_flag(cs));
                    }
                }
            }
        }
        const bool rank_major = transfer == FLUX_PULL && oc.o.emulated_order != 1 && g.size() > 1;
        if (all_here) {
            // issued above
        } else if (rank_major) {
            for (int r : g)
                for (int b = -1; b < tp - 1; ++b) jobs.emplace_back(r, b);
        } else {
            for (int r : g) jobs.emplace_back(r, -1);
            for (int a = 0; a < tp - 1; ++a)
                for (int r : g) jobs.emplace_back(r, a);
        }
        for (const auto& job : jobs) {
            const int r = job.first, step = job.second;
            if (step < 0) {
                FLUX_TRY(local_copy(r));
                continue;
            }
            RankState& rs = c->ranks[r];
            for (int i = step * per_peer; i < (step + 1) * per_peer; ++i) {
                const Desc& d = specs[r][i];
                const int q = d.peer;
                const RankState& qs = c->ranks[q];
                const bool first = !waited[r][q];  // first descriptor involving peer q in this operator
                waited[r][q] = true;
                if (transfer == FLUX_PULL) {
                    char* dst = rs.heap + L.a_agg.off + static_cast<size_t>(d.row_begin) * rowbytes;
                    if (in_group(q)) {
                        const char* shard;
                        size_t pitch;
                        shard_of(q, shard, pitch);
                        FLUX_TRY(copy_rows(cs, dst, rowbytes, shard + static_cast<size_t>(d.row_begin - q * rpr) * pitch,
                                           pitch, d.rows));
                    } else {
                        if (first) FLUX_TRY(wait_value_geq(cs, qs.heap + kCtrlReady, e));
                        FLUX_TRY(copy_rows(cs, dst, rowbytes,
                                           qs.heap + L.a_agg.off + static_cast<size_t>(d.row_begin) * rowbytes, rowbytes,
                                           d.rows));
                    }
                    FLUX_TRY(log_copy(cs, r, d));
                    FLUX_TRY(set_flag(cs, r, d.row_begin / rpct));
                    FLUX_TRY(log_flag(cs));
                } else {
                    if (first && !in_group(q)) FLUX_TRY(wait_value_geq(cs, qs.heap + kCtrlKdone, e - 1));
                    // Push reads from my own a_agg slot (already holds my shard).
                    FLUX_TRY(copy_rows(cs, qs.heap + L.a_agg.off + static_cast<size_t>(d.row_begin) * rowbytes,
                                       rowbytes, rs.heap + L.a_agg.off + static_cast<size_t>(d.row_begin) * rowbytes,
                                       rowbytes, d.rows));
                    FLUX_TRY(log_copy(cs, r, d));
                    FLUX_TRY(set_flag(cs, q, d.row_begin / rpct));
                    FLUX_TRY(log_flag(cs));
                }
            }
        }
        for (int r : g) FLUX_TRY(write_value(cs, c->ranks[r].heap + kCtrlDone, e));
        FLUX_CUDA(cudaEventRecord(lead.copy_evt, cs));
    }
    if (serialize) {
        for (const auto& g : groups)
            for (int r : g) {
                FLUX_CUDA(cudaSetDevice(c->ranks[r].device));
                FLUX_CUDA(cudaStreamWaitEvent(stream_for(c, r, streams), c->ranks[g[0]].copy_evt, 0));
            }
        FLUX_TRY(launch_kernel());
    }
    for (const auto& g : groups)
        for (int r : g) {
            FLUX_CUDA(cudaSetDevice(c->ranks[r].device));
            cudaStream_t s = stream_for(c, r, streams);
            FLUX_TRY(write_value(s, c->ranks[r].heap + kCtrlKdone, e));
            // Later work on the caller's stream is ordered after our transfers.
            FLUX_CUDA(cudaStreamWaitEvent(s, c->ranks[g[0]].copy_evt, 0));
        }
    return FLUX_OK;
}

int flux_gemm_rs(flux_comm* c, const flux_problem* p, const flux_tile* tile, int write_mode, int swizzle_on,
                 const flux_opts* opts, void* const* streams) {
    return flux_gemm_rs_ex(c, p, tile, write_mode, swizzle_on, opts, streams, nullptr);
}

static int gemm_rs_impl(flux_comm* c, const flux_problem* p, const flux_tile* tile, int write_mode, int swizzle_on,
                        const flux_opts* opts, void* const* streams, const flux_operands* operands) {
    FLUX_TRY(check_comm(c));
    if (p && p->pattern != FLUX_GEMM_REDUCESCATTER)
        return fail(FLUX_ERR_CONFIG, "run_fused_gemm_reducescatter requires GemmReduceScatter pattern");
    FLUX_TRY(validate_tiling(p, tile));
    FLUX_TRY(check_heap(c, p));
    if (write_mode != FLUX_WRITE_ALLTOALL && write_mode != FLUX_FUSED_REDUCE)
        return fail(FLUX_ERR_CONFIG, "unknown write mode");
    FLUX_TRY(check_activation(c, p, opts, operands));
    FLUX_TRY(check_b_layout(c, p, opts, operands));
    FLUX_TRY(eager_after_graph(c, streams));
    const int tp = p->tp, rpr = rows_per_rank(p);
    const int tiles = ((p->m + kBM - 1) / kBM) * ((p->n + kBN - 1) / kBN);
    if (static_cast<size_t>(tiles) * tp > kRsFlagCap) return fail(FLUX_ERR_CONFIG, "too many output tiles for the flag table");
    std::vector<int> mine;
    local_ranks_only(c, mine);
    for (int r : mine)
        for (int q = 0; q < tp; ++q) FLUX_TRY(check_directory(c, r, q));
    OpCommon oc = common_opts(opts);
    c->last_launches = 0;
    c->kernel_events_used = 0;
    ++c->epoch;
    const int cg = choose_cg(p, oc.o);
    // NVLS: sources keep their partials in their own region, owners read the
    // sum over every source with multimem.ld_reduce (the owners' reduction
    // units, or the streaming kernel's epilogue).
    const bool nvls = oc.o.nvls != FLUX_NVLS_OFF;
    if (nvls) {
        FLUX_TRY(nvls_check(c, p, oc.o));
        if (write_mode != FLUX_WRITE_ALLTOALL)
            return fail(FLUX_ERR_CONFIG, "NVLS GEMM-RS reduces in the switch: use WriteAlltoAll (FusedReduce red.adds into the owner)");
        if (oc.o.rs_partials != FLUX_F32) return fail(FLUX_ERR_CONFIG, "NVLS GEMM-RS carries fp32 partials");
        FLUX_TRY(nvls_war(c, mine, streams, c->epoch));
    }
    // FusedReduce (engine.cpp:304-319, arrival-order accumulation): sources red.add
    // into the owner's fp32 accumulator. Deterministic FusedReduce (rank-ordered
    // gate, :293-303) is served by the source-ordered owner sum, which gives the
    // same result order without serialising the ranks.
    if (write_mode == FLUX_FUSED_REDUCE && !oc.o.deterministic_reduce) {
        oc.fused_reduce = 1;
        const Layout L = layout_for(p);
        const uint32_t e = c->epoch;
        for (int r : mine) {
            RankState& rs = c->ranks[r];
            FLUX_CUDA(cudaSetDevice(rs.device));
            cudaStream_t s = stream_for(c, r, streams);
            FLUX_CUDA(cudaMemsetAsync(rs.heap + L.staging.off + static_cast<size_t>(e & 1u) * L.stage_parity * 4, 0,
                                      static_cast<size_t>(L.stage_plane) * 4, s));
            FLUX_TRY(write_value(s, rs.heap + kCtrlFrReady, e));
        }
    }
    // Tile order: RankShifted (local block last) or Naive (engine.cpp:210-217,256-261).
    std::vector<std::vector<uint32_t>> seq(tp);
    for (int r : mine) {
        std::vector<int> blocks;
        if (swizzle_on) blocks = block_order(FLUX_SWIZZLE_RANK_SHIFTED, r, tp, oc.o.shift_offset, {});
        else for (int i = 0; i < tp; ++i) blocks.push_back(i);
        seq[r] = device_sequence(p->m, p->n, rpr, blocks, kBM * cg, group_blocks(rpr, kBM * cg, /*ag=*/false),
                                 swizzle_on != 0);
    }
    // Deadlock freedom of the single-device multi-rank launch: a tile may only
    // wait on partials scheduled before it. With ownership blocks aligned to
    // device tiles, RankShifted puts each rank's own block last, so rank-major
    // order with those blocks moved to the end qualifies (and keeps each rank's
    // operands L2-resident); otherwise fall back to position-major.
    const bool aligned = swizzle_on && rpr % (kBM * cg) == 0 && oc.o.emulated_order != 1;
    const int tail = aligned ? (rpr / (kBM * cg)) * ((p->n + kBN - 1) / kBN) : 0;
    // Ownership blocks narrower than a device tile (decode-sized M): sources
    // stage whole tiles, owners sum their rows at the end of the kernel.
    const int tiles_n = (p->n + kBN - 1) / kBN;
    oc.rs_units = ((rpr % kBM != 0 || nvls) && !oc.fused_reduce) ? 1 : 0;
    oc.ops = operands;
    if (oc.o.rs_partials != FLUX_F32 && oc.o.rs_partials != FLUX_BF16)
        return fail(FLUX_ERR_CONFIG, "rs_partials must be F32 or BF16");
    if (oc.o.rs_partials == FLUX_BF16 && oc.fused_reduce)
        return fail(FLUX_ERR_CONFIG, "bf16 partials need WriteAlltoAll");
    // Chained partial sums (kernel, RS branch) when every rank runs in this one
    // launch (rank-major order, owners' blocks last); every chain link waits only
    // on an earlier section.
    {
        const auto groups = device_groups(c);
        const char* env = std::getenv("FLUX_RS_CHAIN");
        // Links wait for the previous rank's tile, so each rank's section must
        // span a few waves (else the sections run concurrently and the chain
        // serialises them; measured on decode shapes).
        const long long tiles_per_rank = static_cast<long long>((p->m + kBM * cg - 1) / (kBM * cg)) * tiles_n;
        const int clusters = std::max(1, sm_count(c->ranks[0].device) / cg);
        oc.rs_chain = aligned && !oc.fused_reduce && !oc.rs_units && groups.size() == 1 &&
                              static_cast<int>(groups[0].size()) == tp && tiles_per_rank >= 2LL * clusters &&
                              !(env && std::atoi(env) == 0)
                          ? 1
                          : 0;
    }
    // Whole-tile blocks of a problem smaller than one wave are summed by the
    // owners' reduction units (the decode path) on every SM, the idle ones
    // included, instead of in the owners' tiles (C1: 67 -> 50 us). Larger
    // problems keep the tail / chain (units measured slower there).
    // FLUX_RS_UNITS=0/1 overrides (profiling).
    if (!oc.rs_chain && !oc.fused_reduce && !oc.rs_units) {
        const auto groups = device_groups(c);
        size_t per_dev = 1;
        for (const auto& dg : groups) per_dev = std::max(per_dev, dg.size());
        const long long tiles_launch = static_cast<long long>((p->m + kBM * cg - 1) / (kBM * cg)) * tiles_n *
                                       static_cast<long long>(per_dev);
        const int clusters = std::max(1, sm_count(c->ranks[mine.empty() ? 0 : mine[0]].device) / cg);
        bool units = tiles_launch < clusters;
        if (const char* env = std::getenv("FLUX_RS_UNITS")) units = std::atoi(env) != 0;
        if (units) oc.rs_units = 1;
    }
    const int interleave =
        oc.rs_units ? kInterleaveBlock : (aligned ? kInterleaveRankTail : kInterleaveStep);
    std::function<int(const std::vector<int>&, GemmParams&)> extra = nullptr;
    if (nvls)
        extra = [&](const std::vector<int>&, GemmParams& prm) -> int {
            nvls_fill(c, p, oc.o, prm);
            return FLUX_OK;
        };
    FLUX_TRY(launch_groups(c, p, oc.rs_units ? kModeRSUnits : kModeRS, oc, streams, seq, 0, interleave, cg,
                           false, -1, oc.rs_units ? 0 : tail, extra));
    return mark_op_done(c, streams, c->epoch);
}

static int local_gemm_impl(flux_comm* c, const flux_problem* p, const flux_opts* opts, void* const* streams) {
    FLUX_TRY(check_comm(c));
    FLUX_TRY(validate_problem(p));
    FLUX_TRY(check_heap(c, p));
    FLUX_TRY(check_activation(c, p, opts, nullptr));
    FLUX_TRY(check_b_layout(c, p, opts, nullptr));
    OpCommon oc = common_opts(opts);
    c->last_launches = 0;
    c->kernel_events_used = 0;
    std::vector<int> mine;
    local_ranks_only(c, mine);
    const int cg = choose_cg(p, oc.o);
    std::vector<std::vector<uint32_t>> seq(p->tp);
    for (int r : mine) seq[r] = device_sequence(p->m, local_cols(p), rows_per_rank(p), {}, kBM * cg);
    const int il = oc.o.emulated_order == 1 ? kInterleaveStep : kInterleaveRank;
    if (p->pattern == FLUX_ALLGATHER_GEMM) return launch_groups(c, p, kModePlain, oc, streams, seq, 0, il, cg, true);
    // GEMM-RS: the full [m, n] partial goes to the staging region (parity 0).
    return launch_groups(c, p, kModePlain, oc, streams, seq, 0, il, cg, false,
                         static_cast<long long>(layout_for(p).staging.off));
}

static int nonoverlap_body(flux_comm* c, const flux_problem* p, const flux_opts* opts, void* const* streams) {
    if (opts && opts->graph_safe) return fail(FLUX_ERR_CONFIG, "graph_safe applies to the fused operators and the local GEMM");
    FLUX_TRY(validate_problem(p));
    FLUX_TRY(check_heap(c, p));
    FLUX_TRY(eager_after_graph(c, streams));
    const int tp = p->tp, rpr = rows_per_rank(p), lk = local_k(p);
    std::vector<int> mine;
    local_ranks_only(c, mine);
    for (int r : mine)
        for (int q = 0; q < tp; ++q) FLUX_TRY(check_directory(c, r, q));
    OpCommon oc = common_opts(opts);
    const Layout L = layout_for(p);
    c->last_launches = 0;
    c->kernel_events_used = 0;
    const uint32_t e = ++c->epoch;
    const int cg = choose_cg(p, oc.o);
    std::vector<std::vector<uint32_t>> seq(tp);
    for (int r : mine) seq[r] = device_sequence(p->m, local_cols(p), rpr, {}, kBM * cg);
    if (p->pattern == FLUX_ALLGATHER_GEMM) {
        // Serial AllGather in rank order (engine.cpp:568-571), then the GEMM.
        const size_t rowbytes = static_cast<size_t>(L.a_agg.ld) * 2;
        for (int r : mine) {
            RankState& rs = c->ranks[r];
            FLUX_CUDA(cudaSetDevice(rs.device));
            cudaStream_t s = stream_for(c, r, streams);
            // WAR on my slot: in-process peers are ordered by their previous kernel
            // event, other processes by their epoch-stamped `done` word.
            for (int q = 0; q < tp; ++q) {
                if (c->ranks[q].local) {
                    if (c->ranks[q].kernel_evt_valid) FLUX_CUDA(cudaStreamWaitEvent(s, c->ranks[q].kernel_evt, 0));
                } else if (q != r) {
                    FLUX_TRY(wait_value_geq(s, c->ranks[q].heap + kCtrlDone, e - 1));
                }
            }
            FLUX_CUDA(cudaMemcpy2DAsync(rs.heap + L.a_agg.off + static_cast<size_t>(r) * rpr * rowbytes, rowbytes,
                                        rs.heap + L.a_shard.off, static_cast<size_t>(L.a_shard.ld) * 2, lk * 2, rpr,
                                        cudaMemcpyDeviceToDevice, s));
            FLUX_TRY(write_value(s, rs.heap + kCtrlReady, e));
            FLUX_CUDA(cudaEventRecord(rs.copy_evt, s));
        }
        for (int r : mine) {
            RankState& rs = c->ranks[r];
            FLUX_CUDA(cudaSetDevice(rs.device));
            cudaStream_t s = stream_for(c, r, streams);
            for (int q = 0; q < tp; ++q) {
                if (q == r) continue;
                if (c->ranks[q].local) FLUX_CUDA(cudaStreamWaitEvent(s, c->ranks[q].copy_evt, 0));
                else FLUX_TRY(wait_value_geq(s, c->ranks[q].heap + kCtrlReady, e));
                FLUX_CUDA(cudaMemcpy2DAsync(rs.heap + L.a_agg.off + static_cast<size_t>(q) * rpr * rowbytes, rowbytes,
                                            c->ranks[q].heap + L.a_agg.off + static_cast<size_t>(q) * rpr * rowbytes,
                                            rowbytes, lk * 2, rpr, cudaMemcpyDeviceToDevice, s));
            }
            FLUX_TRY(write_value(s, rs.heap + kCtrlDone, e));
        }
        FLUX_TRY(launch_groups(c, p, kModePlain, oc, streams, seq, 0,
                               oc.o.emulated_order == 1 ? kInterleaveStep : kInterleaveRank, cg, true));
        return mark_op_done(c, streams, e);
    }
    // GEMM-RS: full fp32 partial into this epoch's staging parity, then the
    // serial source-ordered reduce once every rank's GEMM finished.
    const size_t parity_off = L.staging.off + static_cast<size_t>(e & 1u) * L.stage_parity * 4;
    OpCommon oc32 = oc;
    oc32.o.out_dtype = FLUX_F32;  // fp32 partials, reduced in source order below
    FLUX_TRY(launch_groups(c, p, kModePlain, oc32, streams, seq, 0,
                           oc.o.emulated_order == 1 ? kInterleaveStep : kInterleaveRank, cg, false,
                           static_cast<long long>(parity_off)));
    for (int r : mine) {
        RankState& rs = c->ranks[r];
        FLUX_CUDA(cudaSetDevice(rs.device));
        cudaStream_t s = stream_for(c, r, streams);
        FLUX_TRY(write_value(s, rs.heap + kCtrlKdone, e));
    }
    for (int r : mine) {
        RankState& rs = c->ranks[r];
        FLUX_CUDA(cudaSetDevice(rs.device));
        cudaStream_t s = stream_for(c, r, streams);
        for (int q = 0; q < tp; ++q) {
            if (q == r) continue;
            if (c->ranks[q].local) FLUX_CUDA(cudaStreamWaitEvent(s, c->ranks[q].kernel_evt, 0));
            else FLUX_TRY(wait_value_geq(s, c->ranks[q].heap + kCtrlKdone, e));
        }
        RsReduceParams rp;
        std::memset(&rp, 0, sizeof(rp));
        for (int q = 0; q < tp; ++q)
            rp.partials[q] = reinterpret_cast<const float*>(c->ranks[q].heap + parity_off);
        rp.c = rs.heap + L.c32.off;
        rp.ldc = L.c32.ld;
        rp.out_f32 = oc.o.out_dtype == FLUX_F32;
        rp.rows = rpr;
        rp.n = p->n;
        rp.ld_src = L.ld_stage;
        rp.src_row0 = r * rpr;
        rp.dst_row0 = 0;
        rp.tp = tp;
        FLUX_CUDA(launch_rs_reduce(rp, std::max(1, sm_count(rs.device)) * 4, s));
        ++c->last_launches;
        FLUX_CUDA(cudaEventRecord(rs.kernel_evt, s));
    }
    return mark_op_done(c, streams, e);
}

// run_medium_grained (engine.cpp:653-728) on the device: the decomposed (B2)
// baseline. Chunks of m / partitions rows; AG: the copy stream issues every
// chunk's transfers up front (one event per chunk) and each chunk's GEMM — the
// plain kernel over the tiles holding the chunk's rows — waits for its event;
// RS: each chunk's GEMM writes fp32 partials, then the owner's source-ordered
// reduce of those rows runs on the copy stream while the next chunk computes.
static int medium_grained_body(flux_comm* c, const flux_problem* p, const flux_tile* tile, int partitions,
                               const flux_opts* opts, void* const* streams) {
    if (c->ipc) return fail(FLUX_ERR_CONFIG, "the medium-grained baseline runs on single-process communicators");
    if (opts && opts->graph_safe) return fail(FLUX_ERR_CONFIG, "graph_safe applies to the fused operators and the local GEMM");
    FLUX_TRY(validate_tiling(p, tile));
    FLUX_TRY(check_heap(c, p));
    const int tp = p->tp;
    if (!(partitions == tp || partitions == 2 * tp || (tp == 1 && partitions == 1)))
        return fail(FLUX_ERR_CONFIG, "partitions=" + S(partitions) + " must be tp or 2*tp (tp=" + S(tp) + ")");
    if (p->m % partitions != 0) return fail(FLUX_ERR_CONFIG, "m must be divisible by the partition count");
    std::vector<int> mine;
    local_ranks_only(c, mine);
    for (int r : mine)
        for (int q = 0; q < tp; ++q) FLUX_TRY(check_directory(c, r, q));
    OpCommon oc = common_opts(opts);
    const Layout L = layout_for(p);
    c->last_launches = 0;
    c->kernel_events_used = 0;
    const uint32_t e = ++c->epoch;
    const int rpr = rows_per_rank(p), lk = local_k(p), chunk = p->m / partitions;
    const int cg = choose_cg(p, oc.o), tile_m = kBM * cg;
    const int ncols = p->pattern == FLUX_ALLGATHER_GEMM ? local_cols(p) : p->n;
    const int tiles_n = (ncols + kBN - 1) / kBN;
    auto chunk_seq = [&](int cc) {
        std::vector<std::vector<uint32_t>> seq(tp);
        const int t0 = (cc * chunk) / tile_m, t1 = ((cc + 1) * chunk - 1) / tile_m;
        for (int r : mine)
            for (int tn = 0; tn < tiles_n; ++tn)
                for (int tm = t0; tm <= t1; ++tm) seq[r].push_back(pack_tile(0, tm, tn));
        return seq;
    };
    const auto groups = device_groups(c);
    std::vector<std::vector<cudaEvent_t>> ev(groups.size());
    auto cleanup = [&]() {
        for (auto& v : ev)
            for (cudaEvent_t x : v) cudaEventDestroy(x);
    };
    auto fail_clean = [&](int rc) {
        cleanup();
        return rc;
    };
    // The copy stream of every device group starts after the callers' prior work
    // (inputs) and after every kernel of the previous operator (WAR).
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        RankState& lead = c->ranks[groups[gi][0]];
        FLUX_CUDA(cudaSetDevice(lead.device));
        for (int r : groups[gi]) {
            RankState& rs = c->ranks[r];
            FLUX_CUDA(cudaEventRecord(rs.start_evt, stream_for(c, r, streams)));
            FLUX_CUDA(cudaStreamWaitEvent(lead.copy_stream, rs.start_evt, 0));
        }
        for (int q = 0; q < tp; ++q)
            if (c->ranks[q].kernel_evt_valid) FLUX_CUDA(cudaStreamWaitEvent(lead.copy_stream, c->ranks[q].kernel_evt, 0));
        ev[gi].resize(partitions);
        for (auto& x : ev[gi]) FLUX_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
    if (p->pattern == FLUX_ALLGATHER_GEMM) {
        const size_t rowbytes = static_cast<size_t>(L.a_agg.ld) * 2;
        for (size_t gi = 0; gi < groups.size(); ++gi) {
            RankState& lead = c->ranks[groups[gi][0]];
            FLUX_CUDA(cudaSetDevice(lead.device));
            for (int cc = 0; cc < partitions; ++cc) {
                const int o = (cc * chunk) / rpr, lr = cc * chunk - o * rpr;
                for (int r : groups[gi])
                    FLUX_CUDA(cudaMemcpy2DAsync(c->ranks[r].heap + L.a_agg.off + static_cast<size_t>(cc) * chunk * rowbytes,
                                                rowbytes,
                                                c->ranks[o].heap + L.a_shard.off +
                                                    static_cast<size_t>(lr) * L.a_shard.ld * 2,
                                                static_cast<size_t>(L.a_shard.ld) * 2, lk * 2, chunk,
                                                cudaMemcpyDeviceToDevice, lead.copy_stream));
                FLUX_CUDA(cudaEventRecord(ev[gi][cc], lead.copy_stream));
            }
        }
        for (int cc = 0; cc < partitions; ++cc) {
            for (size_t gi = 0; gi < groups.size(); ++gi) {
                FLUX_CUDA(cudaSetDevice(c->ranks[groups[gi][0]].device));
                FLUX_CUDA(cudaStreamWaitEvent(stream_for(c, groups[gi][0], streams), ev[gi][cc], 0));
            }
            const int rc = launch_groups(c, p, kModePlain, oc, streams, chunk_seq(cc), 0, kInterleaveRank, cg, true);
            if (rc != FLUX_OK) return fail_clean(rc);
        }
        cleanup();
        return FLUX_OK;
    }
    const size_t parity_off = L.staging.off + static_cast<size_t>(e & 1u) * L.stage_parity * 4;
    OpCommon oc32 = oc;
    oc32.o.out_dtype = FLUX_F32;  // fp32 partials, reduced in source order
    for (int cc = 0; cc < partitions; ++cc) {
        const int rc = launch_groups(c, p, kModePlain, oc32, streams, chunk_seq(cc), 0, kInterleaveRank, cg, false,
                                     static_cast<long long>(parity_off));
        if (rc != FLUX_OK) return fail_clean(rc);
        const int o = (cc * chunk) / rpr, lr = cc * chunk - o * rpr;
        if (!c->ranks[o].local) continue;
        RankState& rs = c->ranks[o];
        FLUX_CUDA(cudaSetDevice(rs.device));
        for (int q = 0; q < tp; ++q) FLUX_CUDA(cudaStreamWaitEvent(rs.copy_stream, c->ranks[q].kernel_evt, 0));
        RsReduceParams rp;
        std::memset(&rp, 0, sizeof(rp));
        for (int q = 0; q < tp; ++q) rp.partials[q] = reinterpret_cast<const float*>(c->ranks[q].heap + parity_off);
        rp.c = rs.heap + L.c32.off;
        rp.ldc = L.c32.ld;
        rp.out_f32 = oc.o.out_dtype == FLUX_F32;
        rp.rows = chunk;
        rp.n = p->n;
        rp.ld_src = L.ld_stage;
        rp.src_row0 = cc * chunk;
        rp.dst_row0 = lr;
        rp.tp = tp;
        FLUX_CUDA(launch_rs_reduce(rp, std::max(1, sm_count(rs.device)) * 2, rs.copy_stream));
        ++c->last_launches;
    }
    // Every rank's stream continues after its owner's reduces.
    for (int r : mine) {
        RankState& rs = c->ranks[r];
        FLUX_CUDA(cudaSetDevice(rs.device));
        FLUX_CUDA(cudaEventRecord(rs.copy_evt, rs.copy_stream));
        FLUX_CUDA(cudaStreamWaitEvent(stream_for(c, r, streams), rs.copy_evt, 0));
        FLUX_CUDA(cudaEventRecord(rs.kernel_evt, stream_for(c, r, streams)));
    }
    cleanup();
    return FLUX_OK;
}

// ---------------------------------------------------------------------------
// Chained tensor-parallel MLP: AG-GEMM with the activation
// in its epilogue, then GEMM-RS on the intermediate; backward of the input is
// the same pair with the roles interchanged.
// ---------------------------------------------------------------------------
static int mlp_problems(const flux_mlp* mlp, bool backward, flux_problem* ag, flux_problem* rs) {
    if (!mlp) return fail(FLUX_ERR_CONFIG, "null mlp");
    if (mlp->activation < FLUX_ACT_NONE || mlp->activation > FLUX_ACT_SWIGLU)
        return fail(FLUX_ERR_CONFIG, "unknown activation");
    // SWIGLU: the up-projection has 2 ffn columns (gate/up groups); its input
    // gradient is a GEMM-RS over those 2 ffn columns.
    const bool glu = mlp->activation == FLUX_ACT_SWIGLU;
    const int up_cols = glu && !backward ? 2 * mlp->ffn : mlp->ffn;
    const int rs_k = glu && backward ? 2 * mlp->ffn : mlp->ffn;
    *ag = flux_problem{mlp->m, up_cols, mlp->hidden, mlp->tp, FLUX_ALLGATHER_GEMM};
    *rs = flux_problem{mlp->m, mlp->hidden, rs_k, mlp->tp, FLUX_GEMM_REDUCESCATTER};
    FLUX_TRY(validate_problem(ag));
    return validate_problem(rs);
}

size_t flux_mlp_required_heap_bytes(const flux_mlp* mlp) {
    flux_problem ag, rs, bag, brs;
    if (mlp_problems(mlp, false, &ag, &rs) != FLUX_OK) return 0;
    size_t need = std::max(layout_for(&ag).total, layout_for(&rs).total);
    if (mlp_problems(mlp, true, &bag, &brs) == FLUX_OK)
        need = std::max(need, std::max(layout_for(&bag).total, layout_for(&brs).total));
    return need;
}

static int mlp_pair(flux_comm* c, const flux_problem& ag, const flux_problem& rs, const flux_opts* opts,
                    void* const* streams, const std::vector<flux_operands>& ag_ops,
                    const std::vector<flux_operands>& rs_ops, int act, int act_grad) {
    flux_opts o;
    if (opts) o = *opts;
    else flux_default_opts(&o);
    flux_opts o_ag = o, o_rs = o;
    o_ag.activation = act;
    o_ag.activation_grad = act_grad;
    o_ag.out_dtype = FLUX_BF16;  // the intermediate feeds the next GEMM as bf16
    o_rs.activation = o_rs.activation_grad = FLUX_ACT_NONE;
    const flux_tile t_ag{ag.m / ag.tp, ag.n / ag.tp}, t_rs{rs.m / rs.tp, rs.n};
    FLUX_TRY(flux_ag_gemm_ex(c, &ag, &t_ag, ag.m / ag.tp, FLUX_PULL, 1, &o_ag, streams, ag_ops.data()));
    const int launches = c->last_launches;
    FLUX_TRY(flux_gemm_rs_ex(c, &rs, &t_rs, FLUX_WRITE_ALLTOALL, 1, &o_rs, streams, rs_ops.data()));
    c->last_launches += launches;
    return FLUX_OK;
}

int flux_mlp_forward(flux_comm* c, const flux_mlp* mlp, const flux_opts* opts, void* const* streams,
                     const flux_mlp_operands* ops) {
    FLUX_TRY(check_comm(c));
    flux_problem ag, rs;
    FLUX_TRY(mlp_problems(mlp, false, &ag, &rs));
    if (!ops) return fail(FLUX_ERR_CONFIG, "flux_mlp_forward needs caller operands");
    const int n_ops = c->ipc ? 1 : c->tp;
    std::vector<flux_operands> a(n_ops), r(n_ops);
    for (int i = 0; i < n_ops; ++i) {
        const flux_mlp_operands& m = ops[i];
        if (!m.x.ptr || !m.w_up.ptr || !m.w_down.ptr || !m.act.ptr || !m.out.ptr)
            return fail(FLUX_ERR_CONFIG, "flux_mlp_forward: x, w_up, w_down, act and out are required");
        a[i] = flux_operands{m.x, m.w_up, m.act, m.pre};
        r[i] = flux_operands{m.act, m.w_down, m.out, flux_matrix{nullptr, 0}};
    }
    return mlp_pair(c, ag, rs, opts, streams, a, r, mlp->activation, FLUX_ACT_NONE);
}

int flux_mlp_backward_dx(flux_comm* c, const flux_mlp* mlp, const flux_opts* opts, void* const* streams,
                         const flux_mlp_grad_operands* ops) {
    FLUX_TRY(check_comm(c));
    flux_problem ag, rs;
    FLUX_TRY(mlp_problems(mlp, true, &ag, &rs));
    if (!ops) return fail(FLUX_ERR_CONFIG, "flux_mlp_backward_dx needs caller operands");
    const int n_ops = c->ipc ? 1 : c->tp;
    std::vector<flux_operands> a(n_ops), r(n_ops);
    for (int i = 0; i < n_ops; ++i) {
        const flux_mlp_grad_operands& m = ops[i];
        if (!m.dout.ptr || !m.w_down_t.ptr || !m.w_up_t.ptr || !m.dact.ptr || !m.dx.ptr ||
            (mlp->activation != FLUX_ACT_NONE && !m.pre.ptr))
            return fail(FLUX_ERR_CONFIG, "flux_mlp_backward_dx: dout, w_down_t, w_up_t, pre, dact and dx are required");
        a[i] = flux_operands{m.dout, m.w_down_t, m.dact,
                             mlp->activation != FLUX_ACT_NONE ? m.pre : flux_matrix{nullptr, 0}};
        r[i] = flux_operands{m.dact, m.w_up_t, m.dx, flux_matrix{nullptr, 0}};
    }
    return mlp_pair(c, ag, rs, opts, streams, a, r, FLUX_ACT_NONE, mlp->activation);
}

int flux_sync(flux_comm* c) {
    if (!c) return fail(FLUX_ERR_CONFIG, "null communicator");
    std::string deadlock;
    int code = FLUX_ERR_DEADLOCK;
    for (int r = 0; r < c->tp; ++r) {
        RankState& rs = c->ranks[r];
        if (!rs.local) continue;
        FLUX_CUDA(cudaSetDevice(rs.device));
        FLUX_CUDA(cudaStreamSynchronize(rs.copy_stream));
        FLUX_CUDA(cudaDeviceSynchronize());
        uint32_t err[6] = {0, 0, 0, 0, 0, 0};
        FLUX_CUDA(cudaMemcpy(err, rs.heap + kCtrlErr, sizeof(err), cudaMemcpyDeviceToHost));
        if (err[0] != 0) {
            if (deadlock.empty()) {
                deadlock = error_text(err, r);
                code = code_of(err[0]);
            }
            // Clean state for the next operator: the error record and epoch,
            // the launch-scoped work counters a failed launch may have left
            // armed (dynamic tiles, reduction units), the host mirror.
            c->ag_sig = 0;  // a failed in-kernel AllGather may have left its piece counters short
            const uint32_t zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            FLUX_CUDA(cudaMemcpy(rs.heap + kCtrlErr, zero, 24, cudaMemcpyHostToDevice));
            FLUX_CUDA(cudaMemcpy(rs.heap + kCtrlDynCtr, zero, 16, cudaMemcpyHostToDevice));  // + reduction counters
        }
        if (c->err_host) std::memset(c->err_host + 8 * r, 0, 32);
    }
    if (!deadlock.empty()) return fail(code, deadlock);
    return FLUX_OK;
}

int flux_last_launch_count(const flux_comm* c) { return c ? c->last_launches : 0; }

int flux_trace_read(flux_comm* c, int rank, const flux_problem* p, void* out, size_t max_records, size_t* count) {
    FLUX_TRY(check_comm(c));
    FLUX_TRY(validate_problem(p));
    if (rank < 0 || rank >= c->tp || !c->ranks[rank].local)
        return fail(FLUX_ERR_DIRECTORY, "rank " + S(rank) + " is not driven by this process");
    RankState& rs = c->ranks[rank];
    FLUX_CUDA(cudaSetDevice(rs.device));
    FLUX_CUDA(cudaDeviceSynchronize());
    uint32_t n = 0;
    FLUX_CUDA(cudaMemcpy(&n, rs.heap + kCtrlTraceCursor, 4, cudaMemcpyDeviceToHost));
    size_t k = std::min<size_t>(std::min<size_t>(n, kTraceBytes / 16), max_records);
    if (k) FLUX_CUDA(cudaMemcpy(out, rs.heap + layout_for(p).trace_off, k * 16, cudaMemcpyDeviceToHost));
    if (count) *count = k;
    return FLUX_OK;
}

int flux_transfer_log(flux_comm* c, int rank, flux_transfer_record* out, int max, int* count) {
    if (!c) return fail(FLUX_ERR_CONFIG, "null communicator");
    int n = 0;
    for (const auto& x : c->xfer_log) {
        if (x.rank != rank) continue;
        if (n < max && out) {
            FLUX_CUDA(cudaEventSynchronize(x.flag_ev));
            float t_copy = 0.0f, t_flag = 0.0f;
            FLUX_CUDA(cudaEventElapsedTime(&t_copy, x.base, x.copy_ev));
            FLUX_CUDA(cudaEventElapsedTime(&t_flag, x.base, x.flag_ev));
            out[n] = flux_transfer_record{x.peer, x.row_begin, x.rows, static_cast<int64_t>(t_copy * 1e6),
                                          static_cast<int64_t>(t_flag * 1e6)};
        }
        ++n;
    }
    if (count) *count = n;
    return FLUX_OK;
}

int flux_ag_gemm_ordered(flux_comm* c, const flux_problem* p, const flux_tile* tile, int rpct, int transfer,
                         int swizzle_on, const flux_opts* opts, void* const* streams, const flux_operands* operands,
                         const int* order_peer, const int* order_row_begin, const int* order_rows, int count) {
    return run_op(c, [&]() -> int {
        if (!p || count < 0 || (count > 0 && (!order_peer || !order_row_begin || !order_rows)))
            return fail(FLUX_ERR_CONFIG, "null comm order");
        if (opts && opts->graph_safe) return fail(FLUX_ERR_CONFIG, "graph_safe operators use the reference comm order");
        std::vector<std::vector<Desc>> custom(c->tp);
        int slot = 0;
        for (int r = 0; r < c->tp; ++r) {
            if (!c->ranks[r].local) continue;
            for (int j = 0; j < count; ++j) {
                const size_t i = static_cast<size_t>(slot) * count + j;
                custom[r].push_back({order_peer[i], order_row_begin[i], order_rows[i]});
            }
            ++slot;
        }
        return ag_gemm_impl(c, p, tile, rpct, transfer, swizzle_on, opts, streams, operands, &custom);
    });
}

int flux_comm_inject_fault(flux_comm* c, int kind, int rank, int index) {
    if (!c) return fail(FLUX_ERR_CONFIG, "null communicator");
    if (kind < FLUX_FAULT_NONE || kind > FLUX_FAULT_DOUBLE_SIGNAL) return fail(FLUX_ERR_CONFIG, "unknown fault kind");
    if (kind != FLUX_FAULT_NONE && (rank < 0 || rank >= c->tp || index < 0))
        return fail(FLUX_ERR_CONFIG, "fault target out of range");
    c->fault_kind = kind;
    c->fault_rank = rank;
    c->fault_index = index;
    return FLUX_OK;
}

int flux_comm_set_check_double_set(flux_comm* c, int enable) {
    if (!c) return fail(FLUX_ERR_CONFIG, "null communicator");
    c->check_double = enable != 0;
    return FLUX_OK;
}

int flux_comm_set_timing(flux_comm* c, int enable) {
    if (!c) return fail(FLUX_ERR_CONFIG, "null communicator");
    c->timing = enable != 0;
    return FLUX_OK;
}

int flux_last_kernel_ms(flux_comm* c, float* ms) {
    if (!c || !ms) return fail(FLUX_ERR_CONFIG, "null argument");
    float worst = 0.0f;
    for (int i = 0; i < c->kernel_events_used; ++i) {
        FLUX_CUDA(cudaEventSynchronize(c->kernel_events[i].second));
        float t = 0.0f;
        FLUX_CUDA(cudaEventElapsedTime(&t, c->kernel_events[i].first, c->kernel_events[i].second));
        worst = std::max(worst, t);
    }
    *ms = worst;
    return FLUX_OK;
}

}  // extern "C"
