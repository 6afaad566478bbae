// Shared host/device definitions of the B200 fused-operator kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fluxb200 {

// Device GEMM tile (one CTA, cta_group::1): D[128 x 256] fp32 in TMEM,
// A/B staged by TMA in 128B-swizzled K-major shared memory, BK = 64 bf16.
constexpr int kBM = 128;
constexpr int kBN = 256;
constexpr int kBK = 64;
constexpr int kStages = 4;
constexpr int kUmmaK = 16;
constexpr int kThreads = 256;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 spare, w4-7 epilogue
constexpr int kAStageBytes = kBM * kBK * 2;
constexpr int kBStageBytes = kBN * kBK * 2;
constexpr int kTmemCols = 512;  // two 256-column accumulators (epilogue/MMA overlap)
constexpr int kSmemBytes = kStages * (kAStageBytes + kBStageBytes) + 1024 /*align*/ + 256 /*barriers*/;

constexpr int kMaxRanks = 8;   // TP degree supported by one communicator (one NVSwitch node)

// kModeRSUnits: GEMM-RS whose ownership blocks are narrower than a tile (sources stage whole
//   tiles; the owners' rows are summed by reduction units running alongside the GEMM).
enum Activation : int { kActNone = 0, kActGelu = 1, kActRelu = 2, kActSilu = 3, kActSwiGLU = 4 };
enum KernelMode : int { kModePlain = 0, kModeAG = 1, kModeRS = 2, kModeRSUnits = 3 };

// Control block at the start of every rank's symmetric heap. The flags are
// epoch-stamped (monotonic), so nothing needs resetting between operators; the
// two launch-scoped work counters (dynamic tiles, reduction units) are re-armed
// by the last CTA / group of the launch that used them.
constexpr size_t kCtrlErr = 0;          // u32[4]: code, info0, info1, info2
constexpr size_t kCtrlErrEpoch = 16;    // u32: epoch of the operator whose wait recorded the error; +4: failing rank + 1
constexpr size_t kCtrlReady = 64;       // u32: epoch at which this rank's A shard is staged (AG pull source ready)
constexpr size_t kCtrlDone = 68;        // u32: epoch whose peer pulls this rank has finished
constexpr size_t kCtrlKdone = 72;       // u32: epoch whose kernel finished on this rank (push targets)
constexpr size_t kCtrlFrReady = 76;     // u32: epoch whose FusedReduce accumulator is zeroed (RS FusedReduce)
constexpr size_t kCtrlTraceCursor = 80; // u32: records written to this rank's trace ring
constexpr size_t kCtrlDynCtr = 88;      // u32: dynamic tile scheduler — next tile (zeroed by the last cluster out)
constexpr size_t kCtrlDynExit = 92;     // u32: dynamic tile scheduler — clusters finished
constexpr size_t kCtrlRedCtr = 96;      // u32: decode RS reduction — next unit (zeroed by the last group out)
constexpr size_t kCtrlRedExit = 100;    // u32: decode RS reduction — groups finished
// Device-side rank barrier (graph-safe operators of the one-process-per-GPU
// communicator): monotonic, never zeroed (outside every graph_zero range).
constexpr size_t kCtrlBarGen = 104;     // u32: barriers this rank has entered
constexpr size_t kCtrlBarArr = 108;     // u32: arrivals of peers at this rank's barriers
constexpr size_t kTraceBytes = size_t(4) << 20;  // trace ring at the end of the data region (16 B records)
// Trace record kinds (the reference CausalityLog event names, engine.hpp:37-63).
// kEvLaunch (not in the reference schema): a CTA's first (tile_col 0) and last (tile_col 1)
// instruction, for launch-latency profiling.
enum TraceKind : uint32_t { kEvComputeStart = 1, kEvSignalSet = 2, kEvTileWrite = 3, kEvReduce = 4, kEvWait = 5,
                            kEvLaunch = 6 };
__host__ __device__ inline uint64_t trace_word(uint32_t kind, int rank, uint32_t target, int tile_row, int tile_col) {
    return (static_cast<uint64_t>(kind) << 60) | (static_cast<uint64_t>(rank & 0xF) << 56) |
           (static_cast<uint64_t>(target & 0xFFFFFFu) << 32) | (static_cast<uint64_t>(tile_row & 0xFFFF) << 16) |
           static_cast<uint64_t>(tile_col & 0xFFFF);
}
constexpr size_t kAgFlagOffset = 4096;  // u32[kAgFlagCap]: one flag per comm tile (SignalBoard)
constexpr size_t kAgFlagCap = 16384;
// In-kernel AllGather: u32[kAgGroupCap] monotonic piece counters per 128-row
// group of a_agg (+ one own-block counter), +1 per landed piece, zeroed on layout change.
// Tail split (Plain / AG): epoch-tagged arrival counters of the split tail tiles.
constexpr size_t kTailCtrOffset = 72 * 1024;
constexpr int kTailCtrCap = 256;   // per counter set; two sets (slices parked / RS-units slices staged)
constexpr int kTailMaxSplits = 8;
constexpr int kTailWsCtas = 160;  // workspace slots (>= CTAs of one launch): 128 x 256 fp32 each
// Streaming decode kernel: epoch-tagged arrival counters of its split n-tiles.
constexpr size_t kSkCtrOffset = 76 * 1024;
constexpr int kSkCtrCap = 8192;  // u32 (76 KiB .. 108 KiB): arrivals [0, cap/2), RS shares stored [cap/2, cap)
constexpr int kSkMaxSegsHost = 8;  // K-segments per n-tile (flux_stream_kernel kSkMaxSegs)
constexpr int kSkRows = 128;     // weight rows (output columns) per n-tile = MMA M
constexpr int kSkMaxStages = 12;
constexpr int kSkSmemMax = 232448;  // dynamic shared memory opt-in limit (227 KiB)
constexpr size_t kAgCtrOffset = 128 * 1024;
constexpr size_t kAgGroupCap = 16384;  // per counter set
// Graph-safe operators use their own counter set (zeroed by each of them), so
// replays never disturb the eager operators' monotonic counters.
constexpr size_t kAgCtrGraphOffset = kAgCtrOffset + kAgGroupCap * 4;
constexpr int kPieceBytes = 16384;      // one TMA bulk copy (global -> smem -> global)
constexpr size_t kRsFlagOffset = 256 * 1024;  // u32[tile][src]: partial of tile from src landed
constexpr size_t kRsFlagCap = (512 * 1024) / 4;
constexpr size_t kDataOffset = 1 << 20;
// NVLS region (flux_comm_opts.nvls_bytes; one VMM allocation per rank bound to
// one multicast object): AllGather comm-tile flags, then the data area (AG:
// a_agg [m, k] bf16; RS: the source's partial planes, [parity][owner][rpr][n] fp32).
constexpr size_t kNvlsFlagOffset = 0;
constexpr size_t kNvlsDataOffset = 64 * 1024;  // kAgFlagCap u32 flags before it

// Error codes written by device waits into the control block.
constexpr uint32_t kErrAgFlagTimeout = 1;
constexpr uint32_t kErrRsFlagTimeout = 2;
constexpr uint32_t kErrDoubleSet = 3;       // a flag stamped twice in one operator (signal_board.hpp:25-28)
constexpr uint32_t kErrBarrierTimeout = 4;  // a graph-safe operator's rank barrier

// Fault injection (tests: the reference's deadlock / double-set paths,
// acceptance.cpp:121-158, engine.cpp:401-403): armed for one operator.
enum FaultKind : int { kFaultNone = 0, kFaultDropSignal = 1, kFaultDoubleSignal = 2 };

// Tile order entry: local rank (4 bits) | tile row (14 bits) | tile col (14 bits).
__host__ __device__ inline uint32_t pack_tile(int l, int tm, int tn) {
    return (uint32_t(l) << 28) | (uint32_t(tm) << 14) | uint32_t(tn);
}

struct GemmParams {
    CUtensorMap tma_a[kMaxRanks];  // per local rank: A operand [m, k] (AG: a_agg, RS: A shard)
    CUtensorMap tma_b[kMaxRanks];  // per local rank: B operand [n, k] K-major
    void* c[kMaxRanks];            // per local rank: output
    int global_rank[kMaxRanks];    // local slot -> global rank id
    const uint32_t* ag_flags[kMaxRanks];   // per local rank: comm-tile flags
    uint32_t* ctrl[kMaxRanks];             // per local rank: control block (error word)
    float* staging[kMaxRanks];             // per GLOBAL rank: staging planes base (peer pointers)
    uint32_t* rs_flags[kMaxRanks];         // per GLOBAL rank: (tile, src) flags (peer pointers)
    const uint32_t* order;                 // tile schedule (pack_tile entries)
    int num_tiles;
    int m, n, k;                   // per-rank GEMM: A [m, k], B [n, k], C [m, n]
    int ldc;                       // C row pitch (elements) of the library's C buffers (RS peers' C)
    int ldc_l[kMaxRanks];          // per local slot: C row pitch of the C it writes (caller-provided or library)
    int out_f32;                   // C element type
    int tiles_n;                   // ceil(n / kBN)
    int tp, rpr;                   // TP degree, rows per rank
    int rpct;                      // AG rows per comm tile
    int ld_stage;                  // staging row pitch (elements) = n padded
    long long stage_plane;         // elements per (src) plane = rpr * ld_stage
    long long stage_parity;        // elements per parity set = tp * stage_plane
    uint32_t epoch;
    unsigned long long timeout_ns;
    unsigned long long jitter_seed;
    int fused_reduce;              // RS: 1 = red.add into the owner accumulator (arrival order)
    // AG in-kernel transfer (warp 3 of every CTA pulls a_agg pieces with TMA bulk copies)
    int sm_transfer;
    // NVLS (opts.nvls): 1 multicast through the NVSwitch (multimem.*), 2 the same
    // protocol with unicast loops over every rank's region (tests on one GPU).
    int nvls;
    char* nvls_data[kMaxRanks];        // per GLOBAL rank: data area (unicast)
    uint32_t* nvls_flags[kMaxRanks];   // per GLOBAL rank: AG comm-tile flags (unicast)
    char* nvls_data_mc;                // nvls = 1: multicast address of the data area
    uint32_t* nvls_flags_mc;           // nvls = 1: multicast address of the flags
    long long nvls_ld_bytes;           // AG: row pitch of a_agg in the data area
    int ag_direct;                 // AG with tp = 1: A is read from the rank's own shard (the gathered A), no waits
    const uint32_t* jobs;          // (slot << 28) | (src rank << 24) | first row of the piece chunk
    int num_jobs;
    int piece_rows;                // rows per piece chunk (contiguous rows), >= 1
    int pieces_per_row;            // column splits of one row (row bytes > kPieceBytes)
    int row_bytes;                 // k * 2
    long long dst_ld_bytes;        // a_agg row pitch in bytes
    long long src_ld_l[kMaxRanks]; // per local slot: A shard row pitch in bytes
    const char* agg_src[kMaxRanks];    // per GLOBAL rank: its a_agg (peer pointers; pull source)
    const char* shard_src[kMaxRanks];  // per local slot: its own A shard (local piece source)
    int slot_of[kMaxRanks];        // per GLOBAL rank: its local slot in this launch (same device), else -1
    int all_local;                 // every rank runs in this launch: flag producers are on this GPU
    char* a_dst[kMaxRanks];            // per local slot: its a_agg
    uint32_t* ag_ctr[kMaxRanks];   // per GLOBAL rank: monotonic piece counters (peer pointers)
    int ag_slot_index;             // counter index of "own block copied" (after the group counters)
    uint32_t slot_pieces;          // pieces of one rank's own block
    uint32_t ag_mult;              // operators run on these counters since their last reset (targets scale by it)
    // Push (engine.cpp:406-419 on the SMs): jobs carry (source slot, DESTINATION rank,
    // rows); a source copies its own block into every destination's a_agg and
    // bumps the destination's counter. A destination in another process is
    // written only after its previous operator's kernel finished (kdone).
    int ag_push;
    const uint32_t* kdone[kMaxRanks];  // per GLOBAL rank: kernel-done epoch word (peer pointers)
    // RS with ownership blocks narrower than a tile: owners reduce during the GEMM
    int rs_units;
    int red_rows;                  // owner rows per reduction unit (8 or 16)
    int red_warm;                  // reduction units: one dry pass over the first unit before its wait
    uint32_t* red_ctr;             // reduction unit counter (lead rank's control block)
    uint32_t* red_exit;
    // Device event trace (reference CausalityLog, engine.hpp:37-63): 16-byte records
    unsigned long long* trace[kMaxRanks];  // per local slot: ring (nullptr = tracing off)
    uint32_t* trace_cursor[kMaxRanks];     // per local slot: next record index
    uint32_t trace_cap;
    float* fr_acc[kMaxRanks];      // per GLOBAL rank: FusedReduce fp32 accumulator [rpr, ld_stage] (this parity)
    const uint32_t* fr_ready[kMaxRanks];  // per GLOBAL rank: control word, accumulator zeroed at epoch
    // Epilogue activation (Plain / AG): act = flux_activation applied to the
    // accumulator; act_grad = C is acc * act'(aux) (aux = saved pre-activation);
    // aux_save = also store the pre-activation into aux (forward of a chain).
    int act, act_grad, aux_save;
    void* aux[kMaxRanks];          // per local slot: bf16 [m, n] pre-activation
    int ld_aux[kMaxRanks];
    int rs_chain;                  // RS, every rank in this launch: chained partial sums (see kernel)
    // Dynamic tile scheduler: the pair leader's producer fetches tiles from a
    // global counter (tail-split units stay statically one per cluster) and
    // hands them to its pair through a shared-memory queue.
    uint32_t* dyn_ctr;             // nullptr: static stride
    uint32_t* dyn_exit;
    int b_mn;                      // B operand given as [k, n] row-major (MN-major), else [n, k]
    int part_bf16;                 // RS staging partials stored as bf16 (opts.rs_partials)
    // Tail split (Plain / AG): the last (num tiles mod clusters) tiles run as
    // tail_splits K-slices each; the last arriving slice sums them in order.
    int tail_base, tail_splits;    // order[tail_base..] are split; tail_splits <= 1: off
    uint32_t tail_seq;             // per-launch tag of the tail counters
    float* tail_ws;                // [tail tile][split][cta of pair][128 x 256] fp32
    uint32_t* tail_ctr;            // [tail tile][cta of pair]: (tail_seq << 8) | arrivals
    int dbg;                       // profiling ablations (FLUX_DEBUG): 1 skip RS remote stores, 2 skip RS owner reduce
    // Error reporting: a timed-out wait also writes its record into this
    // host-mapped mirror ([global rank][4] u32), which the host reads at the
    // start of the next operator without synchronising (nullptr: off).
    uint32_t* err_host;
    // Fault injection (one operator): drop / double the signal `fault_index` of
    // rank `fault_rank`'s flag table (AG in-kernel: 128-row group counter;
    // RS: tile * tp + source).
    int fault_kind, fault_rank, fault_index;
    int check_double;              // RS flags: exchange-and-check instead of store (double-set detector)
    // Streaming decode kernel (flux_stream_kernel, decode-sized M): weights on the
    // MMA M side (128-row n-tiles), tokens on N; the (slot, n-tile, k-block)
    // space is split evenly over sk_ctas CTAs (stream-K); the K-segments of an
    // n-tile are summed in segment order by the last CTA to arrive (tail_ws
    // holds [cta][first/last segment][sk_mp x 128] fp32 partials).
    int sk_mp;                     // tokens padded to a multiple of 16 (MMA N)
    int sk_stages;                 // smem ring depth
    int sk_pref;                   // AG: weight stages loaded ahead of the gathered token rows
    int sk_nt, sk_kb;              // n-tiles (128 weight rows) per slot, k-blocks
    long long sk_work;             // slots x n-tiles x k-blocks
    int sk_ctas;                   // CTAs with GEMM work (<= grid)
    int sk_acc_cols;               // TMEM columns per accumulator (two accumulators)
    int sk_cluster;                // > 1: clusters of this many CTAs split each n-tile's K; the
                                   // partial accumulators meet in the leader's shared memory (DSMEM)
    int sk_red_ring;               // 1: one tile per cluster; the leader's drained stage ring is the
                                   // reduction buffer (no dedicated one, so more stages fit)
    uint32_t* sk_ctr;              // per (slot, n-tile): (tail_seq << 8) | arrivals
};

struct RsReduceParams {
    const float* partials[kMaxRanks];  // per source rank: full [m, n] fp32 partial (peer pointers)
    void* c;
    int ldc, out_f32, rows, n, ld_src, tp;
    int src_row0;  // first partial row summed (global row)
    int dst_row0;  // its row in C (the owner's local row)
};

// Host launchers (flux_kernels.cu).
// cg: CTAs per MMA tile (1 = 128x256 tiles, 2 = CTA pairs with 256x256 tiles).
cudaError_t launch_gemm(int mode, int cg, const GemmParams& p, int grid, cudaStream_t stream);
int gemm_tile_rows(int cg);
cudaError_t launch_rs_reduce(const RsReduceParams& p, int grid, cudaStream_t stream);
// Streaming decode kernel (modes Plain, AG, RSUnits); smem from stream_smem_bytes.
cudaError_t launch_stream(int mode, const GemmParams& p, int grid, int smem, cudaStream_t stream);
int stream_smem_bytes(int mode, int mp, int stages, int cluster = 1);
int stream_max_clusters(int mode, const GemmParams& p, int cluster, int smem);

// Graph-safe operators: zero byte ranges (4-byte multiples) of several heaps,
// one CTA per heap.
constexpr int kZeroMaxRanges = 8;
struct ZeroParams {
    char* heap[kMaxRanks];
    uint32_t off[kZeroMaxRanges];
    uint32_t bytes[kZeroMaxRanges];
    int nranges;
};
cudaError_t launch_zero_ranges(const ZeroParams& p, int nheaps, cudaStream_t stream);
// One-thread barrier across the ranks of a multi-process communicator: enter
// (gen += 1), arrive at every peer (arr += 1, release, system scope), wait until
// this rank's arrivals reach gen x (tp - 1) (acquire), bounded by timeout_ns
// (the error word gets kErrBarrierTimeout).
struct BarrierParams {
    uint32_t* gen;
    uint32_t* arr;
    uint32_t* peer_arr[kMaxRanks];
    uint32_t* err;       // this rank's control block (error record)
    uint32_t* err_host;  // host-mapped mirror [rank][8]
    int tp, me;
    uint32_t epoch;
    uint64_t timeout_ns;
};
cudaError_t launch_rank_barrier(const BarrierParams& p, cudaStream_t stream);

}  // namespace fluxb200
