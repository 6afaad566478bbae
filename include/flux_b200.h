/*
 * flux_b200.h — C ABI of the B200-native fused tensor-parallel operators
 * (AllGather-GEMM and GEMM-ReduceScatter, Flux arXiv 2406.06858).
 *
 * This is the drop-in boundary for the reference's hot path. Every entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj). Plain C types only: pointers, ints, sizes. All device
 * work is asynchronous on the caller's streams; flux_sync() joins it and
 * surfaces device-side failures (e.g. a signal wait that timed out) as
 * FLUX_ERR_DEADLOCK, mirroring overlap::DeadlockError.
 *
 * Data model (reference workspace.hpp:12-19, problem.hpp:14-38):
 *   AllGatherGemm     rank r: A shard [m/tp, k] bf16, B shard [n/tp, k] bf16
 *                     (weight stored [out, in] = K-major, i.e. the transpose of
 *                     the reference's b_shard [k, n/tp]), gathered A a_agg
 *                     [m, k], output C [m, n/tp].
 *   GemmReduceScatter rank r: A shard [m, k/tp], B shard [n, k/tp] (K-major),
 *                     output C [m/tp, n] = rows owned by r of the rank-ordered
 *                     sum of all partial products.
 * The library owns these buffers inside a per-rank symmetric heap (the
 * reference ShardedWorkspace + its peer directory, workspace.cpp:5-29,56-65);
 * callers address them through flux_buffer().
 */
#ifndef FLUX_B200_H_
#define FLUX_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FLUX_ABI_VERSION 8

/* Return codes. The reference raises C++ exceptions (errors.hpp:9-31); each
 * maps to one code. The C++ shim (include/flux/overlap.hpp) rethrows them. */
typedef enum {
    FLUX_OK = 0,
    FLUX_ERR_CONFIG = 1,    /* overlap::ConfigError   */
    FLUX_ERR_SHAPE = 2,     /* overlap::ShapeError    */
    FLUX_ERR_DIRECTORY = 3, /* overlap::DirectoryError (peer mapping missing) */
    FLUX_ERR_DEADLOCK = 4,  /* overlap::DeadlockError (device wait timed out) */
    FLUX_ERR_BOUNDS = 5,    /* overlap::BoundsError   */
    FLUX_ERR_CUDA = 6,      /* CUDA runtime / driver failure */
    FLUX_ERR_RUNTIME = 7    /* std::runtime_error: a signal flag set twice in one operator
                               (SignalBoard::set -> false, engine.cpp:401-403) */
} flux_status;

/* overlap::Pattern (problem.hpp:10) */
typedef enum { FLUX_ALLGATHER_GEMM = 0, FLUX_GEMM_REDUCESCATTER = 1 } flux_pattern;
/* overlap::TransferMode (engine.hpp:16) */
typedef enum { FLUX_PULL = 0, FLUX_PUSH = 1 } flux_transfer_mode;
/* overlap::WriteMode (engine.hpp:17) */
typedef enum { FLUX_WRITE_ALLTOALL = 0, FLUX_FUSED_REDUCE = 1 } flux_write_mode;
/* overlap::SwizzleKind (swizzle.hpp:10) */
typedef enum { FLUX_SWIZZLE_NAIVE = 0, FLUX_SWIZZLE_RANK_SHIFTED = 1, FLUX_SWIZZLE_ARRIVAL_ALIGNED = 2 } flux_swizzle_kind;
typedef enum { FLUX_BF16 = 0, FLUX_F32 = 1 } flux_dtype;

/* Buffers of one rank (overlap::RankBuffers, workspace.hpp:12-19). */
typedef enum {
    FLUX_BUF_A_SHARD = 0,
    FLUX_BUF_B_SHARD = 1,
    FLUX_BUF_A_AGG = 2,
    FLUX_BUF_C_OUT = 3,
    FLUX_BUF_STAGING = 4
} flux_buffer_kind;

/* overlap::ProblemSpec (problem.hpp:22-38) */
typedef struct {
    int m, n, k, tp;
    int pattern; /* flux_pattern */
} flux_problem;

/* overlap::TileShape (problem.hpp:40-43): ownership / comm granularity. The
 * device MMA tile is fixed by the kernel (128x256); (tm, tn) keeps the
 * reference's divisibility contract and error messages. */
typedef struct {
    int tm, tn;
} flux_tile;

/* overlap::EngineOptions (engine.hpp:65-72) plus the B200 knobs. */
typedef struct {
    int workers_per_rank;      /* accepted for API parity; the device uses every SM */
    int deterministic_reduce;  /* 1: fixed-order sum (other sources ascending, then the owner's own) */
    long long poll_budget;     /* accepted for API parity (device waits are time-bounded) */
    double wall_budget_s;      /* device spin-wait timeout (default 10 s, engine.hpp:69) */
    uint64_t interleave_seed;  /* nonzero: device jitter (nanosleep) before tiles, race testing */
    int shift_offset;          /* RankShifted offset (swizzle.hpp:27), default 1 */
    int out_dtype;             /* flux_dtype of C (default BF16) */
    int emulated_order;        /* several ranks on one device: 0 locality-first (rank-major,
                                  RS own blocks last), 1 position-major across ranks */
    int cta_group;             /* 0 auto, 1 = 128x256 tiles per CTA, 2 = CTA pairs (256x256, cta_group::2) */
    int ag_engine;             /* AllGather transfers: 0 auto, 1 copy engines (stream memcpy + flag
                                  writes), 2 in-kernel (TMA bulk copies by the GEMM's SMs, Pull or Push) */
    int trace;                 /* 1: record the device event trace of the next operators (flux_trace_read) */
    int activation;            /* flux_activation fused into the AllGather-GEMM / local GEMM epilogue */
    int activation_grad;       /* flux_activation whose derivative scales C: C = acc * act'(aux) */
    int rs_partials;           /* flux_dtype of the GEMM-RS cross-rank partials: F32 (default) or BF16
                                  (half the NVLink bytes; one bf16 rounding per partial / chain link;
                                  WriteAlltoAll only) */
    int b_layout;              /* flux_b_layout of caller-provided B (operands.b): NK = [n/tp or n, k]
                                  (nn.Linear.weight, default) or KN = [k, n] row-major (the reference's
                                  b_shard; no transposed copy needed, e.g. for the backward pass) */
    int graph_safe;            /* 1: the operator may be captured in a CUDA graph and replayed: it
                                  zeroes the flags / counters it uses before its kernel (one small
                                  kernel) and runs the in-kernel AllGather on its own counter set,
                                  so every replay starts from a clean state. Single-process
                                  communicators; AllGather uses the in-kernel transfer engine (no
                                  host stream memops); not with the arrival-order FusedReduce. */
    int decode_kernel;         /* flux_decode_kernel: GEMMs of at most 128 rows (decode) run on the
                                  streaming kernel (weights on the MMA M side, tokens on N, stream-K
                                  over the weight shard) unless FLUX_DECODE_TILE */
    int nvls;                  /* flux_nvls: NVLink SHARP multicast through the NVSwitch (north_star:
                                  "reduce through NVLS multicast where the host exposes it").
                                  AllGather-GEMM: every rank pushes its own A rows once with
                                  multimem.st into all ranks' a_agg and stamps each comm tile's
                                  flag on all ranks with one multicast store. GEMM-RS: every
                                  source writes its partial into its own region; each owner
                                  reads the sum over all sources with multimem.ld_reduce
                                  (reduced in the switch; fp32 partials, WriteAlltoAll).
                                  FLUX_NVLS_MULTICAST needs a communicator created with
                                  nvls_bytes > 0; FLUX_NVLS_EMULATED runs the same protocol
                                  with unicast loops over the ranks' regions (tests on one GPU). */
} flux_opts;

typedef enum { FLUX_DECODE_AUTO = 0, FLUX_DECODE_TILE = 1, FLUX_DECODE_STREAM = 2 } flux_decode_kernel;

typedef enum { FLUX_NVLS_OFF = 0, FLUX_NVLS_MULTICAST = 1, FLUX_NVLS_EMULATED = 2 } flux_nvls;

typedef enum { FLUX_B_NK = 0, FLUX_B_KN = 1 } flux_b_layout;

/* Epilogue activations (chained MLP; paper Fig. 2). GELU is
 * the erf form. SWIGLU: the local N columns come in 256-column groups of 128
 * gate then 128 up columns; C receives silu(gate) * up (N/2 columns) and aux,
 * if given, the N pre-activation columns. activation_grad = SWIGLU: C (2N
 * columns, same grouping) receives dgate, dup from the GEMM's dz and aux. */
typedef enum {
    FLUX_ACT_NONE = 0,
    FLUX_ACT_GELU = 1,
    FLUX_ACT_RELU = 2,
    FLUX_ACT_SILU = 3,
    FLUX_ACT_SWIGLU = 4
} flux_activation;

typedef struct {
    size_t heap_bytes;         /* per-rank symmetric heap size (0 = 1 GiB) */
    size_t nvls_bytes;         /* > 0: also create an NVLS multicast region of this many bytes per
                                  rank (VMM memory bound to one cuMulticast object over every
                                  rank's GPU; single-process communicators over distinct GPUs).
                                  Creation fails with FLUX_ERR_CUDA naming the step when the host
                                  does not expose multicast (flux_nvls_probe tells beforehand). */
} flux_comm_opts;

typedef struct flux_comm flux_comm;

/* Device view of one buffer: element (i, j) is at ptr + (i*ld + j)*elem_size. */
typedef struct {
    void* ptr;
    int rows, cols, ld;
    int dtype; /* flux_dtype */
} flux_buffer_desc;

/* ---- diagnostics ---------------------------------------------------------- */
const char* flux_last_error(void);          /* thread-local message of the last failure */
int flux_abi_version(void);
int flux_device_sm_count(int device);       /* 0 without a GPU */
void flux_default_opts(flux_opts* opts);    /* EngineOptions{} defaults */

/* ---- problem / tiling (problem.cpp:15-47) ---------------------------------- */
/* ProblemSpec::validate + validate_tiling; same rules and messages. */
int flux_problem_validate(const flux_problem* problem, const flux_tile* tile);
/* grid_for (problem.cpp:40-47) */
int flux_grid_for(const flux_problem* problem, const flux_tile* tile, int* tile_rows,
                  int* tile_cols, int* row_blocks);

/* ---- schedules (swizzle.cpp:23-80, topology.cpp:46-178) -------------------- */
/* tile_order(SwizzlePolicy{kind, rank, tp, shift_offset, arrival_blocks}, grid_for(problem, tile))
 * writes grid.tiles() coordinates. n_arrival == 0 means the default ring order. */
int flux_tile_order(const flux_problem* problem, const flux_tile* tile, int kind, int rank,
                    int shift_offset, const int* arrival_blocks, int n_arrival, int* out_rows,
                    int* out_cols);
/* map_tile(SwizzlePolicy{kind, rank, tp, shift_offset, arrival_blocks}, i, GridDims{tile_rows,
 * tile_cols, row_blocks}) (swizzle.cpp:51-73): the single implementation of the tile bijection
 * (flux_tile_order and the C++ shim use it). BoundsError for i outside the grid. */
int flux_map_tile(int kind, int rank, int tp, int shift_offset, const int* arrival_blocks, int n_arrival,
                  int tile_rows, int tile_cols, int row_blocks, int index, int* out_row, int* out_col);
/* comm_order(Topology{NVLinkRing}, rank, tp, rows_per_rank, rpct): descriptors
 * (peer, row_begin, rows). *count receives the number written (<= max). */
int flux_comm_order(int rank, int tp, int rows_per_rank, int rows_per_comm_tile, int* out_peer,
                    int* out_row_begin, int* out_rows, int max, int* count);
/* make_comm_specs(problem, Topology{}, rpct, mode) (engine.cpp:77-99) for one
 * rank, including CommTileSpec::validate (engine.cpp:40-75). */
int flux_make_comm_spec(const flux_problem* problem, int rank, int rows_per_comm_tile,
                        int transfer, int* out_peer, int* out_row_begin, int* out_rows, int max,
                        int* count);

/* CommTileSpec::validate (engine.cpp:40-75) of one rank's descriptor list. */
int flux_validate_comm_spec(const flux_problem* problem, int rank, int rows_per_comm_tile, int transfer,
                            const int* peer, const int* row_begin, const int* rows, int count);

/* ---- communicator = symmetric heap + peer directory (workspace.hpp:22-43) --- */
size_t flux_required_heap_bytes(const flux_problem* problem);
/* Single process: rank r lives on devices[r]. Devices may repeat (several ranks
 * emulated on one GPU, the reference's threads-as-ranks model, engine.cpp:172-191);
 * distinct devices get peer access over NVLink. */
int flux_comm_create(int tp, const int* devices, const flux_comm_opts* opts, flux_comm** out);
/* One process per GPU (torchrun): create, export a handle blob, all-gather the
 * blobs out of band (torch.distributed), connect. */
int flux_comm_create_ipc(int rank, int tp, int device, const flux_comm_opts* opts,
                         flux_comm** out);
size_t flux_comm_ipc_blob_bytes(void);
int flux_comm_ipc_handle(flux_comm* comm, void* blob);
int flux_comm_ipc_connect(flux_comm* comm, const void* blobs /* tp * blob_bytes, rank order */);
/* Host-only validation of a gathered blob set (magic, ranks, tp, heap size). */
int flux_ipc_blobs_check(const void* blobs, int tp, size_t heap_bytes);
int flux_comm_destroy(flux_comm* comm);
int flux_comm_tp(const flux_comm* comm);
int flux_comm_rank(const flux_comm* comm); /* IPC: own rank; single process: -1 */
/* Simulates an incomplete init-phase exchange (workspace.cpp:67-69, tests only). */
int flux_comm_drop_peer(flux_comm* comm, int from_rank, int peer_rank);

/* NVLS capability probe: 1 if a multicast object can be created over `devices`
 * (n >= 1 distinct GPUs) and bound to memory on each, else 0 with the failing
 * step in `why` (e.g. "cuMulticastCreate: invalid argument"). No GPU: 0. */
int flux_nvls_probe(int n, const int* devices, char* why, int why_len);
/* Bytes of the NVLS region a problem needs (flux_comm_opts.nvls_bytes). */
size_t flux_nvls_required_bytes(const flux_problem* problem);
/* 1 if the communicator owns an NVLS multicast region. */
int flux_comm_nvls(const flux_comm* comm);
/* NVLS for one process per GPU, after flux_comm_ipc_connect. The multicast
 * handle is a POSIX file descriptor the caller hands from rank 0 to the others
 * (a Unix socket with SCM_RIGHTS; comm.py does it): rank 0 _export()s it, the
 * others _import() it (the fd is consumed), every rank _add_device()s its GPU,
 * and once all have (caller's barrier) every rank _bind()s its memory; a second
 * barrier before the first NVLS operator (peers' regions zeroed). Errors name
 * the failing step ("NVLS unavailable: cuMulticastCreate: ..."). */
int flux_comm_nvls_ipc_export(flux_comm* comm, size_t nvls_bytes, int* fd_out);
int flux_comm_nvls_ipc_import(flux_comm* comm, size_t nvls_bytes, int fd);
int flux_comm_nvls_ipc_add_device(flux_comm* comm);
int flux_comm_nvls_ipc_bind(flux_comm* comm);
/* Buffer of `rank` for `problem` (any rank in single-process mode; own rank in IPC mode). */
int flux_buffer(flux_comm* comm, int rank, int kind, const flux_problem* problem,
                flux_buffer_desc* out);
/* Copy a dense host matrix (rows x cols, row pitch host_ld elements, dtype of
 * the buffer) into / out of a buffer, asynchronously on `stream` (NULL = the
 * rank's default stream). Host memory should be pinned for async behaviour. */
int flux_copy_in(flux_comm* comm, int rank, int kind, const flux_problem* problem,
                 const void* host, int host_ld, void* stream);
int flux_copy_out(flux_comm* comm, int rank, int kind, const flux_problem* problem, void* host,
                  int host_ld, void* stream);

/* ---- the fused operators -------------------------------------------------- */
/* run_fused_allgather_gemm (engine.hpp:107-111, engine.cpp:443-556; paper Alg. 2+3).
 * streams: one per rank in single-process mode (NULL = library streams), one in
 * IPC mode. Comm tiles move on copy engines (Alg. 3) and raise per-comm-tile
 * flags; the tcgen05 GEMM's TMA producer waits on them (Alg. 2). */
int flux_ag_gemm(flux_comm* comm, const flux_problem* problem, const flux_tile* tile,
                 int rows_per_comm_tile, int transfer, int swizzle_on, const flux_opts* opts,
                 void* const* streams);
/* run_fused_gemm_reducescatter (engine.hpp:101-103, engine.cpp:221-352; paper Alg. 1).
 * The epilogue stores each partial tile into the owner's staging plane over
 * NVLink and raises a per-(tile, source) flag; the owner reduces in a fixed
 * order (the other sources ascending, then its own partial) inside its
 * local-tile epilogue (deterministic). When all ranks share one launch the
 * sources chain the sum in that order instead (each adds its partial to the
 * running sum its predecessor left), and the owner reads one plane. */
int flux_gemm_rs(flux_comm* comm, const flux_problem* problem, const flux_tile* tile,
                 int write_mode, int swizzle_on, const flux_opts* opts, void* const* streams);
/* The AllGather transfer engine flux_ag_gemm uses for this problem: 1 copy
 * engines, 2 in-kernel (opts.ag_engine, or the automatic choice when 0). */
int flux_ag_engine(const flux_problem* problem, int transfer, const flux_opts* opts);
/* Local GEMM only (tp ranks each compute their own C = A_agg B^T / A B^T with no
 * communication): T_gemm_nonsplit of Eq. 1 and the TP=1 path. */
int flux_local_gemm(flux_comm* comm, const flux_problem* problem, const flux_opts* opts,
                    void* const* streams);
/* run_nonoverlap (engine.hpp:125-126, engine.cpp:558-605): serial copy-engine
 * collective then the same GEMM kernel (or GEMM then serial reduce). */
int flux_nonoverlap(flux_comm* comm, const flux_problem* problem, const flux_opts* opts,
                    void* const* streams);
/* run_medium_grained (engine.hpp:144-145, schedule engine.cpp:607-651): the
 * decomposed (B2) baseline — m split into `partitions` (tp or 2*tp; 1 at tp=1)
 * row chunks; AG: every chunk's copy-engine transfers are issued up front and
 * each chunk's GEMM (this library's kernel) waits for its chunk; RS: chunk
 * GEMMs into fp32 partials, each chunk's source-ordered reduce on a side
 * stream overlapping the next chunk's GEMM. Single-process communicators. */
int flux_medium_grained(flux_comm* comm, const flux_problem* problem, const flux_tile* tile, int partitions,
                        const flux_opts* opts, void* const* streams);
/* Caller-owned operands (e.g. PyTorch tensors): per rank (tp entries in
 * single-process mode, 1 in IPC mode); NULL ptr fields use the library's
 * buffers. A = the rank's A shard, B = its weight shard [out, in] (K-major),
 * C = its output; element (i, j) at ptr + (i*ld + j)*elem_size, ld in elements,
 * rows 16-byte aligned. Only the symmetric state (a_agg, staging, flags) must
 * live in the library heap. For GEMM-RS a caller C needs m/tp % 128 == 0. */
typedef struct {
    void* ptr;
    int ld;
} flux_matrix;
typedef struct {
    flux_matrix a, b, c;
    flux_matrix aux; /* AG epilogue: pre-activation [m, n/tp] bf16 — written when
                        opts.activation is set (optional), read when opts.activation_grad is */
} flux_operands;
int flux_ag_gemm_ex(flux_comm* comm, const flux_problem* problem, const flux_tile* tile,
                    int rows_per_comm_tile, int transfer, int swizzle_on, const flux_opts* opts,
                    void* const* streams, const flux_operands* operands);
int flux_gemm_rs_ex(flux_comm* comm, const flux_problem* problem, const flux_tile* tile,
                    int write_mode, int swizzle_on, const flux_opts* opts, void* const* streams,
                    const flux_operands* operands);
/* run_fused_allgather_gemm with the caller's comm specs (engine.hpp:107-111
 * `comm_specs`): for every rank this process drives (in rank order; one in
 * IPC mode) `count` descriptors (peer, row_begin, rows) at [slot * count + j],
 * validated like CommTileSpec::validate (ConfigError / BoundsError). The
 * copy-engine transfer loop walks them in the given order (engine.cpp:367-423)
 * and the tiles follow the arrival order they imply (arrival_aligned_policy,
 * swizzle.cpp:23-29 / the Push arrival sort, engine.cpp:480-501). */
int flux_ag_gemm_ordered(flux_comm* comm, const flux_problem* problem, const flux_tile* tile,
                         int rows_per_comm_tile, int transfer, int swizzle_on, const flux_opts* opts,
                         void* const* streams, const flux_operands* operands, const int* order_peer,
                         const int* order_row_begin, const int* order_rows, int count);
/* TransferRecord of the last AllGather run with opts.trace on the copy-engine
 * transfer engine (engine.hpp:79-85): per descriptor of `rank`'s comm spec, in
 * issue order, the device times (ns, CUDA events on the copy stream relative to
 * its first transfer) at which its copy completed and its flag was raised;
 * copy_done_ns <= flag_set_ns (test_engine.cpp:102-115). */
typedef struct {
    int peer, row_begin, rows;
    int64_t copy_done_ns, flag_set_ns;
} flux_transfer_record;
int flux_transfer_log(flux_comm* comm, int rank, flux_transfer_record* out, int max, int* count);

/* ---- chained tensor-parallel MLP (paper Fig. 2, §3) ------
 * Forward: act = activation(AllGather(x) W_up^T) on every rank (AG-GEMM with
 * the activation in its epilogue), then out = ReduceScatter(act W_down^T)
 * (GEMM-RS). Per rank (tp entries single-process, 1 in IPC mode), bf16,
 * row-major, ld in elements:
 *   x [m/tp, hidden]; w_up [ffn/tp (x2 for SWIGLU), hidden]; w_down [hidden, ffn/tp];
 *   pre [m, ffn/tp] (optional: saved pre-activation, not with SWIGLU);
 *   act [m, ffn/tp] (the intermediate); out [m/tp, hidden] (needs m/tp % 128 == 0).
 * Backward of the input (the AG <-> RS interchange): dact =
 * (AllGather(dout) W_down) * act'(pre) (AG-GEMM, derivative in the epilogue),
 * then dx = ReduceScatter(dact W_up) (GEMM-RS), with the transposed weights
 * w_down_t [ffn/tp, hidden] and w_up_t [hidden, ffn/tp]. SWIGLU: pre and dact
 * are [m, 2 ffn/tp] in the gate/up grouping (dgate, dup) and w_up_t is
 * [hidden, 2 ffn/tp]. With opts.b_layout = KN the *_t fields take the forward
 * weights untransposed (w_down [hidden, ffn/tp], w_up [ffn/tp, hidden]). */
typedef struct {
    int m, hidden, ffn, tp;
    int activation; /* flux_activation */
} flux_mlp;
typedef struct {
    flux_matrix x, w_up, w_down, pre, act, out;
} flux_mlp_operands;
typedef struct {
    flux_matrix dout, w_down_t, w_up_t, pre, dact, dx;
} flux_mlp_grad_operands;
int flux_mlp_forward(flux_comm* comm, const flux_mlp* mlp, const flux_opts* opts, void* const* streams,
                     const flux_mlp_operands* operands);
int flux_mlp_backward_dx(flux_comm* comm, const flux_mlp* mlp, const flux_opts* opts, void* const* streams,
                         const flux_mlp_grad_operands* operands);
/* Heap bytes per rank the MLP calls need (the larger of their two operators). */
size_t flux_mlp_required_heap_bytes(const flux_mlp* mlp);

/* Joins all work of the last operator; returns FLUX_ERR_DEADLOCK if a device
 * wait timed out (message names the flag, as spin_wait does, engine.cpp:149-162). */
int flux_sync(flux_comm* comm);
/* Number of this library's kernels launched by the last operator call. */
int flux_last_launch_count(const flux_comm* comm);
/* Measurement hooks: when enabled, every fused launch is bracketed by CUDA
 * events on its launching stream; flux_last_kernel_ms returns the longest
 * launch of the last operator (waits for it). */
int flux_comm_set_timing(flux_comm* comm, int enable);
/* Device event trace of the last traced operator on `rank` (reference
 * CausalityLog, engine.hpp:37-63): 16-byte records {u64 %globaltimer ns;
 * u64 kind<<60 | rank<<56 | target<<32 | tile_row<<16 | tile_col}, kinds
 * 1 compute_start, 2 signal_set, 3 tile_write, 4 reduce. Waits for the device. */
int flux_trace_read(flux_comm* comm, int rank, const flux_problem* problem, void* out,
                    size_t max_records, size_t* count);
int flux_last_kernel_ms(flux_comm* comm, float* ms);

/* ---- fault injection and checking (tests; reference acceptance.cpp:121-158,
 * spin_wait engine.cpp:149-162, SignalBoard signal_board.hpp:25-28) ---------
 * Arms a fault for the NEXT operator only: DROP_SIGNAL never raises signal
 * `index` of rank `rank`'s flag table, so the waiter times out after
 * opts.wall_budget_s and flux_sync returns FLUX_ERR_DEADLOCK naming the flag;
 * DOUBLE_SIGNAL raises it twice. Signal index per table: AllGather copy-engine
 * flags: comm tile (row / rows_per_comm_tile); AllGather in-kernel transfer:
 * 128-row group of a_agg; GEMM-RS: output tile * tp + source rank (tile =
 * 128-row tile row * ceil(n / 256) + 256-column tile). A device failure is also
 * reported by the next operator call (FLUX_ERR_DEADLOCK / FLUX_ERR_RUNTIME,
 * without synchronising) until flux_sync clears it. */
typedef enum { FLUX_FAULT_NONE = 0, FLUX_FAULT_DROP_SIGNAL = 1, FLUX_FAULT_DOUBLE_SIGNAL = 2 } flux_fault_kind;
int flux_comm_inject_fault(flux_comm* comm, int kind, int rank, int index);
/* Double-set detector for the device-stamped GEMM-RS flags (an exchange that
 * checks the previous stamp instead of a plain store): a second stamp in one
 * operator makes flux_sync return FLUX_ERR_RUNTIME "flag i on rank r set
 * twice". Copy-engine AllGather flags are always checked on the host (the
 * operator call itself returns FLUX_ERR_RUNTIME). */
int flux_comm_set_check_double_set(flux_comm* comm, int enable);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* FLUX_B200_H_ */
