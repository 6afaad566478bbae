// Fused tensor-parallel GEMM kernels for sm_100a (B200).
//
// One persistent, warp-specialised tcgen05 GEMM serves every role
// (KernelMode):
//   Plain  — C = A B^T, no communication (TP=1 and the Eq. 1 "non-split GEMM").
//   AG     — paper Alg. 2 (reference engine.cpp:516-547): before the TMA
//            producer loads the A rows of a tile it spins on the per-comm-tile
//            flags covering those rows (reference spin_wait on SignalBoard,
//            engine.cpp:529-539); flags are raised by the copy-engine transfer
//            loop (Alg. 3, engine.cpp:367-423) on a side stream, or by warp 3
//            of every CTA pulling a_agg pieces with TMA bulk copies.
//   RS     — paper Alg. 1 (reference engine.cpp:265-341): the epilogue routes
//            every accumulator row to its owner (owner_of_row, problem.hpp:37)
//            as tile-major partials (WriteAlltoAll, engine.cpp:285-292) or
//            red.add (FusedReduce, :304-319) and raises a per-(tile, source)
//            flag; the owner reduces its rows inside its local-tile epilogue
//            in a fixed order, replacing the reference's reduce agent
//            (engine.cpp:324-341); with every rank in one launch the partials
//            are chained instead (each source adds to its predecessor's sum).
//   RSUnits — RS with ownership blocks narrower than a tile (decode) or a
//            problem smaller than one wave: sources stage whole tiles and stamp
//            per-(tile, source) flags; the owners' rows are summed by reduction
//            units on warps 2-3 during the GEMM (and the epilogue warps after).
// Epilogue options: activations (GELU / ReLU / SiLU / SwiGLU), pre-activation
// save, derivative scaling (MLP backward); tail split of the last wave
// (Plain / AG); B operand K-major or MN-major; bf16 RS partials (PB).
//
// Roles: warp 0 = TMA producer (one lane), warp 1 = MMA issuer (one lane),
// warp 2 = TMEM allocator, warp 3 = in-kernel AllGather transfer (AG),
// warps 2-3 = reduction units (RSUnits), warps 4..7 = epilogue (TMEM lane
// quadrants 0..3). Pipelines: a smem ring (TMA -> MMA), two TMEM accumulators
// (MMA -> epilogue). The tile schedule is a host-built table (reference
// tile_order, swizzle.cpp:75-80) walked with a static stride of the cluster
// count (or fetched from a counter: FLUX_DYN_SCHED, ablation).
#include <cuda_bf16.h>

#include <atomic>

#include "flux_internal.hpp"

namespace fluxb200 {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier -----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- TMA ------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// ---- tcgen05 ----------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                 : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, bf16 in, fp32 accumulate.
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
// 32 lanes x 32 consecutive fp32 columns: thread i receives row (lane base + i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- clusters / CTA pairs (cta_group::2) --------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of the same shared variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load whose completion is signalled to the pair leader's mbarrier.
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
// D[256 x N] across the pair: A rows 0-127 / 128-255 and B rows (N) halves
// come from each CTA's shared memory at the same offsets.
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on the same barrier in both CTAs of the pair once the MMAs retire.
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAITC:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONEC;\n\t"
        "bra LAB_WAITC;\n"
        "DONEC:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void st_shared_cluster_s32(uint32_t cluster_addr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

// Shared-memory matrix descriptor: K-major, 128B swizzle, 8-row core groups
// 1024 B apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
    const uint64_t addr = smem_u32(p);
    return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}
// MN-major 128B-swizzled operand (B given as [k, n] row-major): 64-element MN
// atoms of 8 K-rows x 128 B; K groups of 8 rows 1 KiB apart (SBO), MN atoms
// (one 64 x 64 TMA box each) 8 KiB apart (LBO).
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(const void* p) {
    const uint64_t addr = smem_u32(p);
    return ((addr >> 4) & 0x3FFFull) | (uint64_t(8192 >> 4) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}
constexpr int kMnBoxBytes = 64 * kBK * 2;  // one 64 (N) x 64 (K) bf16 TMA box

// Instruction descriptor: D f32, A/B bf16, both K-major, M x N.
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// ---- cross-rank signalling (system scope: peers are other GPUs) -------------------
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ float4 ld_cg_f4(const float* p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
// Cross-rank partials (RS staging): 4 consecutive elements at element offset e
// of a plane base, fp32 or (opts.rs_partials = BF16) bf16 — half the bytes over
// NVLink / HBM, one rounding per stored partial.
template <int PB>
__device__ __forceinline__ float4 ld_part4(const float* base, long long e) {
    if (!PB) return ld_cg_f4(base + e);
    // Plain (non-volatile) load so the compiler can batch several before the
    // unpacking that consumes them.
    const uint2 w = __ldcg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(base) + e));
    return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u), __uint_as_float(w.y << 16),
                       __uint_as_float(w.y & 0xFFFF0000u));
}
template <int PB>
__device__ __forceinline__ void st_part4(float* base, long long e, const float4& v) {
    if (!PB) {
        *reinterpret_cast<float4*>(base + e) = v;
        return;
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&lo);
    w.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(base) + e) = w;
}

// ---- NVLS: multimem through the NVSwitch (opts.nvls) --------------------------------
// nvls = 1: one access to the multicast address reaches every rank's copy (the
// switch replicates stores and reduces loads); nvls = 2: the same protocol as
// unicast loops over the ranks' regions (tests on one GPU). Regular accesses to
// the same memory use the unicast addresses: fence.proxy.alias orders the two.
__device__ __forceinline__ void nvls_st16(const GemmParams& p, long long off, const uint4& v) {
    if (p.nvls == 1) {
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p.nvls_data_mc + off),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
    } else {
#pragma unroll
        for (int r = 0; r < kMaxRanks; ++r)
            if (r < p.tp) *reinterpret_cast<uint4*>(p.nvls_data[r] + off) = v;
    }
}
// AllGather comm-tile flag f stamped with the operator's epoch on every rank
// (release, system scope: after the tile's rows, which every lane of the warp
// stored before the caller's __syncwarp).
__device__ __forceinline__ void nvls_flag_set(const GemmParams& p, int f) {
    asm volatile("fence.proxy.alias;" ::: "memory");
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (p.nvls == 1) {
        asm volatile("multimem.st.release.sys.global.u32 [%0], %1;" ::"l"(p.nvls_flags_mc + f), "r"(p.epoch) : "memory");
    } else {
#pragma unroll
        for (int r = 0; r < kMaxRanks; ++r)
            if (r < p.tp) st_release_sys(p.nvls_flags[r] + f, p.epoch);
    }
}
// Sum over every rank of the 4 fp32 at element offset e of the data areas (the
// owner's rows of all sources' partials): reduced in the switch (nvls = 1), or
// in rank order (nvls = 2).
__device__ __forceinline__ float4 nvls_ld_reduce4(const GemmParams& p, long long e) {
    float4 v;
    if (p.nvls == 1) {
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(reinterpret_cast<const float*>(p.nvls_data_mc) + e)
                     : "memory");
        return v;
    }
    float4 w[kMaxRanks];
#pragma unroll
    for (int r = 0; r < kMaxRanks; ++r)
        if (r < p.tp) w[r] = ld_cg_f4(reinterpret_cast<const float*>(p.nvls_data[r]) + e);
    v = w[0];
#pragma unroll
    for (int r = 1; r < kMaxRanks; ++r)
        if (r < p.tp) {
            v.x += w[r].x;
            v.y += w[r].y;
            v.z += w[r].z;
            v.w += w[r].w;
        }
    return v;
}
// GEMM-RS partial of source `me` for owner o's rows: with NVLS the source keeps
// it in its own region (plane o; the owner reduces over the sources through the
// multicast address), else it goes to the owner's staging region (plane me).
__device__ __forceinline__ float* rs_plane_base(const GemmParams& p, int o, int me, long long& plane_off) {
    if (p.nvls) {
        plane_off = static_cast<long long>(o) * p.stage_plane;
        return reinterpret_cast<float*>(p.nvls_data[me]);
    }
    plane_off = static_cast<long long>(me) * p.stage_plane;
    return p.staging[o];
}

// ---- bulk copies (in-kernel AllGather transfer) -----------------------------------
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_group() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_f4(float* p, float a, float b, float c, float d) {
    asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
// Callers reach it after lane-divergent code (one lane spinning on a flag while
// its warp-mates wait here): __syncwarp reconverges the warp first, so the
// .aligned barrier (bar.sync) is well defined. (The non-.aligned barrier.sync
// measured up to 30 % slower on the decode RS epilogues.)
__device__ __forceinline__ void named_bar_sync(int id, int n) {
    __syncwarp();
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Bounded spin (reference spin_wait, engine.cpp:149-162): epoch-stamped flag
// reaches `target`, or the timeout records an error naming the flag.
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Every producer of this launch's flags on this GPU (all ranks in one launch):
// gpu-scope acquires suffice.
__device__ __forceinline__ uint32_t ld_acquire_flag(const GemmParams& p, const uint32_t* f) {
    return p.all_local && !(p.dbg & 512) ? ld_acquire_gpu(f) : ld_acquire_sys(f);
}
// First failure of an operator: the error record {code, info0, info1, info2,
// epoch, failing rank + 1} goes into the launch's lead slot's control block
// (slot 0: the first failure of the whole launch, which the sibling waits of
// every slot watch, so one missing signal does not cascade into timeouts of
// tiles stalled behind it) and into the failing slot's own; flux_sync reads
// them. The host-mapped mirror ([global rank][8] u32) carries the same
// records so the next operator call can report the failure without a sync.
__device__ __noinline__ void record_error(const GemmParams& p, int l, uint32_t code, uint32_t info0, uint32_t info1,
                             uint32_t info2) {
    const uint32_t who = static_cast<uint32_t>(p.global_rank[l]) + 1u;
    for (int s = 0; s < (l == 0 ? 1 : 2); ++s) {
        const int slot = s == 0 ? 0 : l;
        uint32_t* ctrl = p.ctrl[slot];
        if (atomicCAS(ctrl + 0, 0u, code) != 0u) continue;
        ctrl[1] = info0;
        ctrl[2] = info1;
        ctrl[3] = info2;
        ctrl[kCtrlErrEpoch / 4] = p.epoch;
        ctrl[kCtrlErrEpoch / 4 + 1] = who;
        if (p.err_host != nullptr) {
            volatile uint32_t* h = p.err_host + 8 * p.global_rank[slot];
            h[1] = info0;
            h[2] = info1;
            h[3] = info2;
            h[5] = who;
            __threadfence_system();
            h[0] = code;
        }
    }
    __threadfence_system();
}

// Bounded spin of local slot l on an epoch-stamped flag / monotonic counter.
// Waits of this operator abort early once a sibling wait of the SAME operator
// failed (the error record carries its epoch); an error left over from an
// earlier operator does not short-circuit later waits.
__device__ bool wait_flag(const uint32_t* flag, uint32_t target, const GemmParams& p, int l, uint32_t code,
                          uint32_t info0, uint32_t info1) {
    if (static_cast<int32_t>(ld_acquire_flag(p, flag) - target) >= 0) return true;
    const uint64_t t0 = globaltimer();
    uint32_t ns = 32;
    const volatile uint32_t* ctrl = p.ctrl[0];  // the launch's first failure (record_error)
    for (;;) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
        if (static_cast<int32_t>(ld_acquire_flag(p, flag) - target) >= 0) return true;
        if (globaltimer() - t0 > p.timeout_ns) {
            record_error(p, l, code, info0, info1, target);
            return false;
        }
        if (ctrl[0] != 0u && ctrl[kCtrlErrEpoch / 4] == p.epoch) return false;  // sibling failed
    }
}

__device__ __forceinline__ bool fault_hit(const GemmParams& p, int rank, int index) {
    return p.fault_kind != kFaultNone && p.fault_rank == rank && p.fault_index == index;
}

// Stamp RS flag (tile, src) of owner o with this operator's epoch (local slot l
// sets it): gpu scope when the owner runs in this launch, system scope for a
// peer GPU. With the double-set detector on, the stamp is an exchange and a
// previous stamp of the same epoch is an error (SignalBoard::set returning
// false, signal_board.hpp:25-28 / engine.cpp:401-403).
__device__ void rs_flag_set(const GemmParams& p, int l, int o, int tile_id, int src) {
    if (p.nvls) asm volatile("fence.proxy.alias;" ::: "memory");  // the partial (unicast) before the flag
    const int idx = tile_id * p.tp + src;
    uint32_t* f = p.rs_flags[o] + idx;
    const bool hit = fault_hit(p, o, idx);
    if (hit && p.fault_kind == kFaultDropSignal) return;
    const bool gpu = p.slot_of[o] >= 0 && !(p.dbg & 512);  // dbg 512: ablation, always sys
    for (int rep = 0; rep < (hit ? 2 : 1); ++rep) {
        if (p.check_double) {
            uint32_t old;
            if (gpu)
                asm volatile("atom.release.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(old) : "l"(f), "r"(p.epoch) : "memory");
            else
                asm volatile("atom.release.sys.global.exch.b32 %0, [%1], %2;" : "=r"(old) : "l"(f), "r"(p.epoch) : "memory");
            if (old == p.epoch)
                record_error(p, l, kErrDoubleSet, static_cast<uint32_t>(idx), static_cast<uint32_t>(o),
                             static_cast<uint32_t>(tile_id));
        } else if (gpu) {
            st_release_gpu(f, p.epoch);
        } else {
            st_release_sys(f, p.epoch);
        }
    }
}

// Pieces that fill 128-row group g of a_agg (in-kernel AllGather transfer).
__device__ __forceinline__ uint32_t ag_group_target(const GemmParams& p, int g) {
    const int rows = min(kBM, p.m - g * kBM);
    return p.piece_rows > 1 ? static_cast<uint32_t>(rows / p.piece_rows)
                            : static_cast<uint32_t>(rows * p.pieces_per_row);
}

// One 16-byte record of the device event trace: %globaltimer, then
// kind(4) | rank(4) | target(24) | tile_row(16) | tile_col(16).
__device__ __forceinline__ void trace_event(const GemmParams& p, int l, uint32_t kind, int rank, int tile_row,
                                            int tile_col, uint32_t target) {
    if (p.trace[l] == nullptr) return;
    const uint64_t ts = globaltimer();
    const uint32_t i = atomicAdd(p.trace_cursor[l], 1u);
    if (i >= p.trace_cap) return;
    unsigned long long* rec = p.trace[l] + 2ull * i;
    rec[0] = ts;
    rec[1] = trace_word(kind, rank, target, tile_row, tile_col);
}

// Publish one landed AG piece (trace timestamp taken before the release).
__device__ __forceinline__ void ag_signal(const GemmParams& p, uint32_t* ctr, int meta) {
    const int l = meta >> 16, g = meta & 0xFFFF;
    const bool hit = fault_hit(p, p.global_rank[l], g);
    if (hit && p.fault_kind == kFaultDropSignal) return;
    trace_event(p, l, kEvSignalSet, p.global_rank[l], g, 0, static_cast<uint32_t>(g));
    red_release_gpu_add(ctr, hit ? 2u : 1u);
}

__device__ __forceinline__ void decode(uint32_t e, int& l, int& tm, int& tn) {
    l = static_cast<int>(e >> 28);
    tm = static_cast<int>((e >> 14) & 0x3FFFu);
    tn = static_cast<int>(e & 0x3FFFu);
}

__device__ __forceinline__ uint32_t pack_bf16x2(uint32_t lo, uint32_t hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
    return *reinterpret_cast<uint32_t*>(&v);
}

// Store 32 fp32 accumulators of one row (cols [col, col+32)) to C.
// Store W fp32 accumulators of one row (cols [col, col+W)) to C as bf16 or fp32.
template <int W>
__device__ __forceinline__ void store_row(void* c, long long off, int col, int n, int out_f32, const float (&v)[W]) {
    if (out_f32) {
        float* dst = static_cast<float*>(c) + off;
        if (col + W <= n) {
#pragma unroll
            for (int j = 0; j < W; j += 4)
                *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (col + j < n) dst[j] = v[j];
        }
    } else {
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(c) + off;
        if (W == 4 && col + W <= n) {
            uint2 w;
            w.x = pack_bf16x2(__float_as_uint(v[0]), __float_as_uint(v[1]));
            w.y = pack_bf16x2(__float_as_uint(v[2 % W]), __float_as_uint(v[3 % W]));
            *reinterpret_cast<uint2*>(dst) = w;
        } else if (col + W <= n) {
#pragma unroll
            for (int j = 0; j + 7 < W; j += 8) {
                uint4 w;
                w.x = pack_bf16x2(__float_as_uint(v[j + 0]), __float_as_uint(v[j + 1]));
                w.y = pack_bf16x2(__float_as_uint(v[j + 2]), __float_as_uint(v[j + 3]));
                w.z = pack_bf16x2(__float_as_uint(v[j + 4]), __float_as_uint(v[j + 5]));
                w.w = pack_bf16x2(__float_as_uint(v[j + 6]), __float_as_uint(v[j + 7]));
                *reinterpret_cast<uint4*>(dst + j) = w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (col + j < n) dst[j] = __float2bfloat16_rn(v[j]);
        }
    }
}

// Work unit t of the schedule: a whole tile, or (tail split) K-slice `split`
// of tail tile order[tail_base + (t - tail_base) / tail_splits].
__device__ __forceinline__ void tile_unit(const GemmParams& p, int t, int k_blocks, uint32_t& entry, int& kb0, int& kb1,
                                          int& split) {
    if (p.tail_splits <= 1 || t < p.tail_base) {
        entry = p.order[t];
        kb0 = 0;
        kb1 = k_blocks;
        split = -1;
        return;
    }
    const int u = t - p.tail_base, S = p.tail_splits;
    entry = p.order[p.tail_base + u / S];
    split = u % S;
    kb0 = split * k_blocks / S;
    kb1 = (split + 1) * k_blocks / S;
}

// Arrival on a tail counter tagged with this launch's sequence number; returns
// the arrival count (the first arrival of a launch restarts it). acq_rel at gpu
// scope: orders this CTA's workspace stores (after a CTA barrier) before it.
__device__ __forceinline__ uint32_t tail_arrive(uint32_t* ctr, uint32_t seq) {
    const uint32_t tag = seq & 0xFFFFFFu;
    uint32_t old = *reinterpret_cast<volatile uint32_t*>(ctr);
    for (;;) {
        const uint32_t nv = (old >> 8) == tag ? old + 1u : ((tag << 8) | 1u);
        uint32_t prev;
        asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;"
                     : "=r"(prev) : "l"(ctr), "r"(old), "r"(nv) : "memory");
        if (prev == old) return nv & 0xFFu;
        old = prev;
    }
}

// Epilogue activations (erf GELU, ReLU, SiLU) and their derivatives.
__device__ __forceinline__ float act_fwd(int a, float x) {
    switch (a) {
        case kActGelu: return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
        case kActRelu: return fmaxf(x, 0.0f);
        case kActSilu: return x / (1.0f + __expf(-x));
        default: return x;
    }
}
__device__ __forceinline__ float act_bwd(int a, float x) {
    switch (a) {
        case kActGelu:
            return 0.5f * (1.0f + erff(x * 0.70710678118654752f)) + x * 0.3989422804014327f * __expf(-0.5f * x * x);
        case kActRelu: return x > 0.0f ? 1.0f : 0.0f;
        case kActSilu: {
            const float sg = 1.0f / (1.0f + __expf(-x));
            return sg * (1.0f + x * (1.0f - sg));
        }
        default: return 1.0f;
    }
}
// W bf16 values of one row (cols [col, col+W)) as floats; 0 past n.
template <int W>
__device__ __forceinline__ void load_row_bf16(const void* base, long long off, int col, int n, float (&x)[W]) {
    const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(base) + off;
    if (col + W <= n && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
#pragma unroll
        for (int j = 0; j < W; j += 8) {
            const uint4 w = *reinterpret_cast<const uint4*>(src + j);
            const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                x[j + 2 * t] = __uint_as_float(u[t] << 16);
                x[j + 2 * t + 1] = __uint_as_float(u[t] & 0xFFFF0000u);
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < W; ++j) x[j] = col + j < n ? __bfloat162float(src[j]) : 0.0f;
    }
}

// acc = w (first term, so no 0 + x rounding or -0 sign flip) or acc += w.
__device__ __forceinline__ void sum_into(float (&acc)[4], const float4& w, bool& first) {
    if (first) {
        acc[0] = w.x;
        acc[1] = w.y;
        acc[2] = w.z;
        acc[3] = w.w;
        first = false;
    } else {
        acc[0] += w.x;
        acc[1] += w.y;
        acc[2] += w.z;
        acc[3] += w.w;
    }
}

// Decode-sized RS, owner side. The rows each local rank owns are cut into
// units of p.red_rows rows x one column tile (TW = 256 or 128 columns),
// ordered column tile first (the order in which the schedule completes them).
// Two otherwise idle warps of every CTA (2 and 3) take units from a
// launch-wide counter while the GEMM runs; the epilogue warps (then the
// producer / MMA warps) join once their GEMM work is done; the last group out
// re-arms the counter for the next launch. A unit waits for the tp flags (tile,
// source) of the tile(s) its rows lie in, then each thread keeps kU positions x
// tp sources in flight (consecutive threads on consecutive 4-column groups of
// a row, coalesced) and sums them in the canonical order (other sources
// ascending, then the owner) into the owner's C. The GEMM never waits on a
// reduction, so these waits cannot deadlock.
// TW: columns per unit = the RS flag column tile (TW for the tile kernel,
// kSkRows for the streaming decode kernel); compile-time so positions split
// into (row, 4-column group) with shifts. kU: positions per thread in flight.
template <int PB, int TW, int kU = 4>
__device__ __noinline__ void owner_reduce(const GemmParams& p, int tid, int nthr, int bar_id, int* slot, bool warm) {
    const int tp = p.tp, tiles_n = p.tiles_n, rpr = p.rpr, n = p.n, out_f32 = p.out_f32;
    const long long ld_stage = p.ld_stage, stage_plane = p.stage_plane;
    const uint32_t epoch = p.epoch, parity = p.epoch & 1u;
    const bool no_wait = (p.dbg & 32) != 0;  // dbg 32: profiling ablation, no waits
    const int red_rows = p.red_rows;
    const int nch = (rpr + red_rows - 1) / red_rows;
    int nl = 0;
    while (nl < kMaxRanks && p.c[nl] != nullptr) ++nl;
    const int per_tn = nl * nch;
    const int units = per_tn * tiles_n;
    for (;;) {
        if (tid == 0) *slot = static_cast<int>(atomicAdd(p.red_ctr, 1u));
        named_bar_sync(bar_id, nthr);
        const int u = *slot;
        if (u >= units) break;
        const int tn = u / per_tn, rem = u % per_tn;
        const int l = rem / nch;
        const int me = p.global_rank[l];
        const int r0 = me * rpr + (rem % nch) * red_rows, r1 = min(r0 + red_rows, (me + 1) * rpr);
        const int tm0 = r0 / kBM, tm1 = (r1 - 1) / kBM;
        const int npos = (r1 - r0) * (TW / 4);
        const float* const sbase = p.staging[me];  // element offsets below (fp32 or bf16 elements, PB)
        const long long e0 = parity * p.stage_parity + static_cast<long long>(r0 - me * rpr) * ld_stage;
        void* const cl = p.c[l];
        const long long ldc = p.ldc_l[l];
        // warm: a group that starts with the kernel runs its first unit's body
        // once dry (loads issued, stores off) before it waits, so the body's
        // instructions and the unit's staging lines are cached by the time the
        // partials land (the body otherwise runs on a cold instruction cache,
        // fetched from DRAM after an L2 flush: ~10 us at decode sizes).
        for (int pass = warm ? 0 : 1; pass < 2; ++pass) {
        if (pass == 1) {
            if (tid < (tm1 - tm0 + 1) * tp && !no_wait) {
                const int tile_id = (tm0 + tid / tp) * tiles_n + tn;
                wait_flag(p.rs_flags[me] + tile_id * tp + tid % tp, epoch, p, l, kErrRsFlagTimeout,
                          static_cast<uint32_t>(tile_id), static_cast<uint32_t>(tid % tp));
                if (tid == 0) trace_event(p, l, kEvReduce, me, tm0, tn, static_cast<uint32_t>(me));
            }
            named_bar_sync(bar_id, nthr);  // flags acquired; everyone has read *slot
            if (p.nvls) asm volatile("fence.proxy.alias;" ::: "memory");
        }
        for (int b = tid; b < npos; b += nthr * kU) {
            float4 v[kU][kMaxRanks];
#pragma unroll
            for (int i = 0; i < kU; ++i) {
                const int pos = b + i * nthr;
                const int col = tn * TW + (pos % (TW / 4)) * 4;
                if (pos < npos && col < n) {
                    const long long e = e0 + (pos / (TW / 4)) * ld_stage + col;
                    if (p.nvls) {
                        v[i][0] = nvls_ld_reduce4(p, e + me * stage_plane);  // every source, summed in the switch
                    } else {
#pragma unroll
                        for (int s = 0; s < kMaxRanks; ++s)
                            if (s < tp) v[i][s] = ld_part4<PB>(sbase, e + s * stage_plane);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < kU; ++i) {
                const int pos = b + i * nthr;
                const int col = tn * TW + (pos % (TW / 4)) * 4;
                if (pos < npos && col < n) {
                    float acc[4];
                    bool first = true;
                    if (p.nvls) {
                        sum_into(acc, v[i][0], first);
                    } else {
#pragma unroll
                        for (int s = 0; s < kMaxRanks; ++s)
                            if (s < tp && s != me) sum_into(acc, v[i][s], first);
#pragma unroll
                        for (int s = 0; s < kMaxRanks; ++s)
                            if (s == me) sum_into(acc, v[i][s], first);
                    }
                    const long long lr = r0 - me * rpr + pos / (TW / 4);
                    if (pass == 1) store_row<4>(cl, lr * ldc + col, col, n, out_f32, acc);
                }
            }
        }
        }
        warm = false;
        if (tid == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 13, static_cast<uint32_t>(u));  // unit summed (profiling)
    }
    if (tid == 0) {
        trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 17 + bar_id, 0);  // group out of units (profiling)
        __threadfence();
        if (atomicAdd(p.red_exit, 1u) == 3u * gridDim.x - 1u) {  // three groups per CTA
            atomicExch(p.red_ctr, 0u);
            atomicExch(p.red_exit, 0u);
        }
    }
}

// In-kernel AllGather transfer (Alg. 3 on the SMs), one lane of warp 3 of
// every CTA: walks this CTA's share of the piece table — TMA bulk copy global
// -> smem -> global through two buffers, then a release increment of the
// destination group's counter. Two loads are in flight: piece i+1 is loaded
// while piece i is stored (a buffer is reloaded once the store that used it
// has read it), and a piece is published once its store has completed. Remote
// pieces first wait until the source rank's own slot of a_agg is complete.
// (Inlined: as a called function its Piece arrays live in local memory, and the
// decode AllGathers measured 8-20 us slower.)
__device__ __forceinline__ void ag_transfer(const GemmParams& p, uint8_t* sComm, uint64_t* cbar) {
    struct Piece {
        const char* src;
        char* dst;
        uint32_t bytes;
        uint32_t* ctr;
        uint32_t* slot_ctr;
        int meta;  // (slot << 16) | group, for the trace
        int dest;  // Push: the destination rank (the reference's signal_set target)
        int buf;
    };
    uint32_t phase[2] = {0u, 0u};
    Piece ld[2] = {};  // loads in flight, oldest first
    int nld = 0;
    Piece st[2] = {};  // stored, awaiting completion + publication, oldest first
    int nst = 0;
    int nb = 0;   // buffer of the next load
    auto publish = [&](const Piece& P) {
        if (P.ctr) {
            if (p.ag_push) {  // the destination's counter, possibly on another GPU
                const bool hit = fault_hit(p, P.dest, P.meta & 0xFFFF);
                if (hit && p.fault_kind == kFaultDropSignal) {
                    // dropped (fault injection)
                } else {
                    trace_event(p, P.meta >> 16, kEvSignalSet, p.global_rank[P.meta >> 16], P.meta & 0xFFFF,
                                0, static_cast<uint32_t>(P.dest));
                    if (p.slot_of[P.dest] >= 0) red_release_gpu_add(P.ctr, hit ? 2u : 1u);
                    else red_release_sys_add(P.ctr, hit ? 2u : 1u);
                }
            } else {
                ag_signal(p, P.ctr, P.meta);
            }
        }
        if (P.slot_ctr) red_release_gpu_add(P.slot_ctr, 1u);
    };
    auto store_oldest = [&]() {  // wait for the oldest load, store it
        const Piece P = ld[0];
        mbar_wait(&cbar[P.buf], phase[P.buf]);
        phase[P.buf] ^= 1u;
        trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 10, 0);  // piece loaded (launch profiling)
        bulk_store(P.dst, sComm + P.buf * kPieceBytes, P.bytes);
        ld[0] = ld[1];
        --nld;
        if (nst == 2) {  // keep at most two stores outstanding: publish the older
            bulk_wait_group<1>();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            publish(st[0]);
            st[0] = st[1];
            nst = 1;
        }
        st[nst++] = P;
    };
    auto drain = [&]() {  // everything in flight stored, completed and published
        while (nld > 0) store_oldest();
        bulk_wait_group<0>();
        trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 11, 0);  // stores complete (launch profiling)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        for (int i = 0; i < nst; ++i) publish(st[i]);
        nst = 0;
    };
    int checked_src = -1;
    if (static_cast<int>(blockIdx.x) < p.num_jobs) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 12, 0);
    for (int j = blockIdx.x; j < p.num_jobs; j += gridDim.x) {
        const uint32_t e = p.jobs[j];
        const int l = static_cast<int>(e >> 28), q = static_cast<int>((e >> 24) & 0xFu);
        const int row0 = static_cast<int>(e & 0xFFFFFFu);
        const int me = p.global_rank[l];
        const int g = row0 / kBM;
        const char* src;
        char* dst;
        uint32_t* ctr;
        uint32_t* slot_ctr = nullptr;
        if (p.ag_push) {
            // q = destination: my own rows go to its a_agg and count there.
            if (p.slot_of[q] < 0 && q != checked_src) {
                drain();  // (no wait may hold a signal)
                wait_flag(p.kdone[q], p.epoch - 1u, p, l, kErrAgFlagTimeout,
                          static_cast<uint32_t>(p.ag_slot_index), 0xFFFE0000u | static_cast<uint32_t>(q));
                checked_src = q;
            }
            src = p.shard_src[l] + static_cast<long long>(row0 - me * p.rpr) * p.src_ld_l[l];
            dst = const_cast<char*>(p.agg_src[q]) + static_cast<long long>(row0) * p.dst_ld_bytes;
            ctr = p.ag_ctr[q] + g;
            // Keep the own-slot counter in step with Pull operators' targets.
            if (q == me) slot_ctr = p.ag_ctr[me] + p.ag_slot_index;
        } else {
        dst = p.a_dst[l] + static_cast<long long>(row0) * p.dst_ld_bytes;
        ctr = p.ag_ctr[me] + g;
        slot_ctr = q == me ? p.ag_ctr[me] + p.ag_slot_index : nullptr;
        if (q == me) {
            src = p.shard_src[l] + static_cast<long long>(row0 - me * p.rpr) * p.src_ld_l[l];
        } else if (p.slot_of[q] >= 0) {
            // A rank on this device (same launch): pull straight from its shard.
            const int sl = p.slot_of[q];
            src = p.shard_src[sl] + static_cast<long long>(row0 - q * p.rpr) * p.src_ld_l[sl];
        } else {
            if (q != checked_src) {
                // Publish everything in flight before blocking: another CTA may be
                // waiting for our own-block pieces (no wait may hold a signal).
                drain();
                // The source's own slot (its shard copied into its a_agg) is complete.
                wait_flag(p.ag_ctr[q] + p.ag_slot_index, p.ag_mult * p.slot_pieces, p, l,
                          kErrAgFlagTimeout, static_cast<uint32_t>(p.ag_slot_index),
                          0xFFFF0000u | static_cast<uint32_t>(q));
                asm volatile("fence.proxy.async.global;" ::: "memory");
                checked_src = q;
            }
            src = p.agg_src[q] + static_cast<long long>(row0) * p.dst_ld_bytes;
        }
        }  // pull
        const int npieces = p.piece_rows > 1 ? 1 : p.pieces_per_row;
        for (int c = 0; c < npieces; ++c) {
            const int off = c * kPieceBytes;
            Piece P;
            P.src = src + off;
            P.dst = dst + off;
            P.bytes = p.piece_rows > 1 ? static_cast<uint32_t>(p.piece_rows * p.row_bytes)
                                       : static_cast<uint32_t>(min(kPieceBytes, p.row_bytes - off));
            P.ctr = ctr;
            P.slot_ctr = slot_ctr;
            P.meta = (l << 16) | g;
            P.dest = q;
            P.buf = nb;
            if (nld == 2) store_oldest();  // frees nothing yet: its buffer is read by the store
            // The last store that used this buffer has read it.
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            mbar_expect_tx(&cbar[nb], P.bytes);
            bulk_load(sComm + nb * kPieceBytes, P.src, P.bytes, &cbar[nb]);
            ld[nld++] = P;
            nb ^= 1;
        }
    }
    drain();
}

// NVLS AllGather push (warp 3, every lane): each local slot's own comm tiles
// (rpct rows of its block, the reference's Push descriptors of that rank,
// engine.cpp:406-419, with every peer as destination at once) go to every
// rank's a_agg with one multicast store per 16 bytes, then the tile's flag is
// stamped on every rank. The consumers wait on those flags exactly as for the
// copy-engine transfer (Alg. 2). Peers finished reading their a_agg for the
// previous operator before this launch (host stream waits).
__device__ void ag_push_nvls(const GemmParams& p, int lane) {
    int nl = 0;
    while (nl < kMaxRanks && p.c[nl] != nullptr) ++nl;
    const int tpr = p.rpr / p.rpct;  // comm tiles per rank block
    const int n16 = p.row_bytes / 16;
    const int total = p.rpct * n16;
    constexpr int kU = 4;
    for (int j = blockIdx.x; j < nl * tpr; j += gridDim.x) {
        const int l = j / tpr, me = p.global_rank[l];
        const int f = me * tpr + j % tpr;
        const int row0 = f * p.rpct;
        const char* src = p.shard_src[l] + static_cast<long long>(row0 - me * p.rpr) * p.src_ld_l[l];
        const long long dst = static_cast<long long>(row0) * p.nvls_ld_bytes;
        for (int c0 = lane; c0 < total; c0 += 32 * kU) {
            uint4 v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int idx = c0 + u * 32;
                if (idx < total)
                    v[u] = __ldg(reinterpret_cast<const uint4*>(src + static_cast<long long>(idx / n16) * p.src_ld_l[l]) +
                                 idx % n16);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int idx = c0 + u * 32;
                if (idx < total) nvls_st16(p, dst + static_cast<long long>(idx / n16) * p.nvls_ld_bytes + 16ll * (idx % n16), v[u]);
            }
        }
        __syncwarp();
        if (lane == 0) {
            const bool hit = fault_hit(p, me, f);
            if (!(hit && p.fault_kind == kFaultDropSignal)) {
                trace_event(p, l, kEvSignalSet, me, f, 0, static_cast<uint32_t>(f));
                nvls_flag_set(p, f);
            }
        }
        __syncwarp();
    }
}

// Epilogue staging through shared memory. Warp q owns a 32-row x 32-column
// fp32 window (4 KiB) whose 16-byte granules are XOR-swizzled by row, so both
// the row-per-thread writes (TMEM layout) and the row-contiguous reads are
// bank-conflict free; the reads turn the epilogue's global traffic from 32 rows
// x 16 B per warp instruction into 4 rows x 128 B (coalesced).
constexpr int kEpiWarpBytes = 32 * 32 * 4;
#ifndef FLUX_EPI_U
#define FLUX_EPI_U 4
#endif
constexpr int kEpiU = FLUX_EPI_U;  // coalesced positions per thread per step (x tp loads in flight)
__device__ __forceinline__ void epi_stage(uint8_t* wbuf, int lane, const uint32_t (&r)[32]) {
    __syncwarp();  // the previous chunk's reads of this window are done
    const uint32_t base = smem_u32(wbuf) + static_cast<uint32_t>(lane) * 128u;
#pragma unroll
    for (int g = 0; g < 8; ++g)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + ((static_cast<uint32_t>(g ^ (lane & 7))) << 4)),
                     "r"(r[4 * g]), "r"(r[4 * g + 1]), "r"(r[4 * g + 2]), "r"(r[4 * g + 3])
                     : "memory");
    __syncwarp();
}
// Tile-major WriteAlltoAll staging: float offset of the 128 x 256 partial of
// output tile (local row lr0 of the owner's block, column tile tn) in a plane.
__device__ __forceinline__ long long stage_tile_off(long long lr0, int tn, int tiles_n) {
    return ((lr0 / kBM) * tiles_n + tn) * static_cast<long long>(kBM * kBN);
}
__device__ __forceinline__ float4 epi_read(const uint8_t* wbuf, int i, int g) {
    // ld.shared (a plain dereference compiled to a generic LD here)
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(smem_u32(wbuf + i * 128 + ((g ^ (i & 7)) << 4))));
    return v;
}

}  // namespace

// Per-variant geometry. CG = CTAs cooperating on one MMA tile: 1 (cta_group::1,
// 128 x 256 tile per CTA) or 2 (cta_group::2 CTA pair, 256 x 256 tile; each CTA
// stages half of A (128 rows) and half of B (128 of the 256 N rows)).
constexpr int kBarRegion = 512;  // mbarriers + TMEM slot + tile queue
template <int CG, int MODE = kModePlain>
struct Geo {
    static constexpr int kTileM = kBM * CG;                 // rows of one scheduled tile
    static constexpr int kBRows = kBN / CG;                 // B rows (N) staged per CTA
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kBBytes = kBRows * kBK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStagesN = CG == 2 ? 6 : 4;
    static constexpr int kCommBytes = MODE == kModeAG ? 2 * kPieceBytes : 0;  // in-kernel AG staging
    static constexpr int kEpiBytes = MODE == kModeRS || MODE == kModeRSUnits ? 4 * kEpiWarpBytes : 0;  // RS epilogue windows
    static constexpr int kSmem = kStagesN * kStageBytes + kCommBytes + kEpiBytes + 1024 + kBarRegion;
    static constexpr uint32_t kIdescV = make_idesc(kTileM, kBN);
};

constexpr int kTileQ = 4;  // dynamic scheduler: tile-queue depth

// The sequence of work units a CTA processes. Static: cluster_id, +clusters,
// ... Dynamic: the pair leader's producer fetches from a global counter (tiles
// below `dyn_end`, then at most one statically assigned tail-split unit per
// cluster, so all slices of a tail tile stay co-resident) and publishes each
// unit in a kTileQ-slot queue to the other roles of both CTAs; -1 ends it.
struct TileSeq {
    const GemmParams* p;
    int cluster_id, num_clusters, cta_rank, qi = 0;
    uint32_t qph = 0;
    bool fetcher, dyn_done = false, tail_done = false;
    int t = -1;       // static cursor
    int pend = -1;    // dynamic: the next fetch, issued one unit ahead so its latency hides
    __device__ int fetch() {
        const int dyn_end = p->tail_splits > 1 ? p->tail_base : p->num_tiles;
        if (!dyn_done) {
            const int v = pend < 0 ? static_cast<int>(atomicAdd(p->dyn_ctr, 1u)) : pend;
            if (v < dyn_end) {
                pend = static_cast<int>(atomicAdd(p->dyn_ctr, 1u));
                return v;
            }
            dyn_done = true;
        }
        if (!tail_done) {
            tail_done = true;
            const int u = dyn_end + cluster_id;
            if (p->tail_splits > 1 && u < p->num_tiles) return u;
        }
        return -1;
    }
    // Next unit; the fetcher also publishes it (producer warp of the pair leader).
    template <int CG>
    __device__ int next(uint64_t* qfull, uint64_t* qempty, int* qtile) {
        if (p->dyn_ctr == nullptr) {
            t = t < 0 ? cluster_id : t + num_clusters;
            return t < p->num_tiles ? t : -1;
        }
        int v;
        if (fetcher) {
            v = fetch();
            mbar_wait_acq_cluster(&qempty[qi], qph ^ 1u);
            qtile[qi] = v;
            if (CG == 2) st_shared_cluster_s32(mapa(smem_u32(&qtile[qi]), 1), v);
            mbar_arrive(&qfull[qi]);
            if (CG == 2) mbar_arrive_cluster(mapa(smem_u32(&qfull[qi]), 1));
        } else {
            mbar_wait_acq_cluster(&qfull[qi], qph);
            v = qtile[qi];
        }
        return v;
    }
    // Consumers release the slot they read (lane 0 of each consuming warp).
    template <int CG>
    __device__ void release(uint64_t* qempty, bool arrive) {
        if (p->dyn_ctr == nullptr) return;
        __syncwarp(__activemask());  // every lane's read of the slot precedes lane 0's release
        if (!fetcher && arrive) {
            if (CG == 2 && cta_rank != 0) mbar_arrive_cluster(mapa(smem_u32(&qempty[qi]), 0));
            else mbar_arrive(&qempty[qi]);
        }
        if (++qi == kTileQ) {
            qi = 0;
            qph ^= 1u;
        }
    }
};

// PB: RS cross-rank partials stored as bf16 (1) or fp32 (0) — a template
// parameter so the owner's batched loads stay branch-free.
// EPI: Plain / AG epilogue with activations / saved pre-activation /
// derivative scaling (1), or the plain store (0) — a template parameter so the
// common path carries none of that code (the kernels are latency-bound on cold
// instruction fetch at decode sizes).
template <int MODE, int CG, int PB = 0, int EPI = 0>
__global__ void __launch_bounds__(kThreads, 1) flux_gemm_kernel(const __grid_constant__ GemmParams p) {
    using G = Geo<CG, MODE>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + G::kStagesN * G::kABytes;
    uint8_t* sComm = sB + G::kStagesN * G::kBBytes;  // 2 x kPieceBytes (AG only)
    uint8_t* sEpi = sComm + G::kCommBytes;           // 4 x 4 KiB epilogue windows (RS only)
    uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + G::kEpiBytes);
    uint64_t* empty = full + G::kStagesN;
    uint64_t* tfull = empty + G::kStagesN;
    uint64_t* tempty = tfull + 2;
    uint64_t* cbar = tempty + 2;  // 2 comm-piece barriers (AG)
    uint64_t* qfull = cbar + 2;    // dynamic scheduler: tile queue slots full / empty
    uint64_t* qempty = qfull + kTileQ;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qempty + kTileQ);
    int* qtile = reinterpret_cast<int*>(tmem_slot + 2);
    int* red_slot = qtile + kTileQ;  // decode RS reduction: unit broadcast per group
    static_assert((2 * G::kStagesN + 6 + 2 * kTileQ) * 8 + 8 + 4 * kTileQ + 16 <= kBarRegion, "barrier region");

    constexpr int TWU = kBN;  // owner reduction units: 256-column tiles
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t cta_rank = CG == 2 ? cluster_ctarank() : 0u;
    const bool leader = cta_rank == 0;
    const int cluster_id = blockIdx.x / CG;
    const int num_clusters = gridDim.x / CG;

    if (warp == 0 && lane == 0) {
        trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 0, 0);
        for (int l = 0; l < kMaxRanks; ++l) {
            if (p.c[l] == nullptr) break;
            tma_prefetch(&p.tma_a[l]);
            tma_prefetch(&p.tma_b[l]);
        }
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < G::kStagesN; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * CG);  // every epilogue warp of the pair drains it
            mbar_init(&cbar[a], 1);
        }
        for (int i = 0; i < kTileQ; ++i) {
            mbar_init(&qfull[i], 1);
            // leader: MMA lane + its 4 epilogue warps (+ the peer's producer and 4 epilogue warps)
            mbar_init(&qempty[i], CG == 2 ? 10 : 5);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        if (CG == 2) tmem_alloc_pair(tmem_slot, kTmemCols);
        else tmem_alloc(tmem_slot, kTmemCols);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp == 0 && lane == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 30, 0);  // prologue done (profiling)

    const int k_blocks = (p.k + kBK - 1) / kBK;

    if (warp == 0) {
        // ===== TMA producer (both CTAs of a pair load their halves) =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            uint64_t jit = p.jitter_seed ? p.jitter_seed * 0x9e3779b97f4a7c15ull + blockIdx.x : 0;
            TileSeq seq{&p, cluster_id, num_clusters, static_cast<int>(cta_rank)};
            seq.fetcher = leader;
            for (int t = seq.next<CG>(qfull, qempty, qtile); t >= 0; t = seq.next<CG>(qfull, qempty, qtile)) {
                seq.release<CG>(qempty, true);
                int l, tm, tn, kb0, kb1, split;
                uint32_t entry;
                tile_unit(p, t, k_blocks, entry, kb0, kb1, split);
                decode(entry, l, tm, tn);
                const int row0 = tm * G::kTileM + static_cast<int>(cta_rank) * kBM;
                const int bcol0 = tn * kBN + static_cast<int>(cta_rank) * G::kBRows;
                if (jit) {  // reference Jitter (engine.cpp:116-128): perturb interleavings
                    jit ^= jit >> 12; jit ^= jit << 25; jit ^= jit >> 27;
                    const uint32_t r = static_cast<uint32_t>((jit * 0x2545F4914F6CDD1Dull) >> 40);
                    if ((r & 15u) == 0u) __nanosleep(r & 0xFFFFu);
                }
                if (MODE == kModeAG && row0 < p.m && !p.ag_direct) {
                    if (p.sm_transfer) {
                        // In-kernel transfer: every piece of this 128-row group landed.
                        const int g = row0 / kBM;
                        wait_flag(p.ag_ctr[p.global_rank[l]] + g, p.ag_mult * ag_group_target(p, g), p,
                                  l, kErrAgFlagTimeout, static_cast<uint32_t>(g),
                                  static_cast<uint32_t>(tm * 65536 + tn));
                    } else {
                        // Alg. 2: wait for every comm tile covering this CTA's A rows.
                        const int rlast = min(row0 + kBM, p.m) - 1;
                        const int f0 = row0 / p.rpct, f1 = rlast / p.rpct;
                        for (int f = f0; f <= f1; ++f)
                            wait_flag(p.ag_flags[l] + f, p.epoch, p, l, kErrAgFlagTimeout,
                                      static_cast<uint32_t>(f), static_cast<uint32_t>(tm * 65536 + tn));
                    }
                    // Flag acquire (generic proxy) before TMA reads (async proxy).
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    if (split <= 0)
                        trace_event(p, l, kEvComputeStart, p.global_rank[l], row0 / kBM, tn,
                                    static_cast<uint32_t>(p.sm_transfer ? row0 / kBM : row0 / p.rpct));
                }
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    if (CG == 2) {
                        if (leader) mbar_expect_tx(&full[stage], 2 * G::kStageBytes);
                        tma_load_2d_pair(sA + stage * G::kABytes, &p.tma_a[l], &full[stage], kb * kBK, row0);
                        if (p.b_mn) {  // [k, n] weights: kBRows / 64 boxes of 64 (N) x 64 (K)
                            for (int j = 0; j < G::kBRows / 64; ++j)
                                tma_load_2d_pair(sB + stage * G::kBBytes + j * kMnBoxBytes, &p.tma_b[l], &full[stage],
                                                 bcol0 + j * 64, kb * kBK);
                        } else {
                            tma_load_2d_pair(sB + stage * G::kBBytes, &p.tma_b[l], &full[stage], kb * kBK, bcol0);
                        }
                    } else {
                        mbar_expect_tx(&full[stage], G::kStageBytes);
                        tma_load_2d(sA + stage * G::kABytes, &p.tma_a[l], &full[stage], kb * kBK, row0);
                        if (p.b_mn) {
                            for (int j = 0; j < G::kBRows / 64; ++j)
                                tma_load_2d(sB + stage * G::kBBytes + j * kMnBoxBytes, &p.tma_b[l], &full[stage],
                                            bcol0 + j * 64, kb * kBK);
                        } else {
                            tma_load_2d(sB + stage * G::kBBytes, &p.tma_b[l], &full[stage], kb * kBK, bcol0);
                        }
                    }
                    if (++stage == G::kStagesN) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
            if (p.dyn_ctr != nullptr && leader) {
                // Every fetch of this cluster precedes its exit count; the last
                // cluster out re-arms the counter for the next launch.
                __threadfence();
                if (atomicAdd(p.dyn_exit, 1u) == static_cast<uint32_t>(num_clusters - 1)) {
                    atomicExch(p.dyn_ctr, 0u);
                    atomicExch(p.dyn_exit, 0u);
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (the pair leader issues for both CTAs) =====
        if (lane == 0 && leader) {
            int stage = 0;
            uint32_t phase = 0;
            int as = 0;
            uint32_t aphase = 0;
            bool first_mma = true;
            TileSeq seq{&p, cluster_id, num_clusters, static_cast<int>(cta_rank)};
            seq.fetcher = false;
            for (int t = seq.next<CG>(qfull, qempty, qtile); t >= 0; t = seq.next<CG>(qfull, qempty, qtile)) {
                seq.release<CG>(qempty, true);
                int kb0, kb1, split;
                uint32_t entry;
                tile_unit(p, t, k_blocks, entry, kb0, kb1, split);
                mbar_wait(&tempty[as], aphase ^ 1u);
                tc_fence_after();
                const uint32_t d = tmem_base + static_cast<uint32_t>(as * kBN);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (kb == kb0 && first_mma) {  // first stage landed (launch profiling)
                        trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 32, 0);
                        first_mma = false;
                    }
                    const uint64_t adesc = smem_desc_sw128(sA + stage * G::kABytes);
                    const uint64_t bdesc = p.b_mn ? smem_desc_mn_sw128(sB + stage * G::kBBytes)
                                                  : smem_desc_sw128(sB + stage * G::kBBytes);
                    // K-major: +32 B along K inside the 128B atom = +2 in the >>4 address
                    // field; MN-major: +16 K-rows = +2 KiB = +128.
                    const uint64_t bstep = p.b_mn ? 128ull : 2ull;
                    const uint32_t idesc = G::kIdescV | (p.b_mn ? (1u << 16) : 0u);
#pragma unroll
                    for (int kk = 0; kk < kBK / kUmmaK; ++kk) {
                        if (CG == 2)
                            umma_bf16_pair(d, adesc + 2ull * kk, bdesc + bstep * kk, idesc, (kb > kb0 || kk != 0) ? 1u : 0u);
                        else
                            umma_bf16(d, adesc + 2ull * kk, bdesc + bstep * kk, idesc, (kb > kb0 || kk != 0) ? 1u : 0u);
                    }
                    // Frees the smem slot (in both CTAs) when these MMAs retire.
                    if (CG == 2) umma_commit_pair(&empty[stage]);
                    else umma_commit(&empty[stage]);
                    if (++stage == G::kStagesN) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                if (CG == 2) umma_commit_pair(&tfull[as]);  // accumulator ready for both epilogues
                else umma_commit(&tfull[as]);
                if (++as == 2) {
                    as = 0;
                    aphase ^= 1u;
                }
            }
        }
    } else if (MODE == kModeRSUnits && (warp == 2 || warp == 3)) {
        // ===== decode RS: owners' reduction, concurrent with the GEMM =====
        owner_reduce<PB, TWU>(p, threadIdx.x - 64, 64, 3, &red_slot[0], p.red_warm != 0);
    } else if (warp == 3) {
        // ===== in-kernel AllGather transfer (Alg. 3 on the SMs) =====
        if (MODE == kModeAG && p.nvls) ag_push_nvls(p, lane);
        else if (MODE == kModeAG && p.sm_transfer && lane == 0) ag_transfer(p, sComm, cbar);
    } else if (warp >= 4) {
        // ===== epilogue: each CTA drains its own 128 TMEM lanes (rows) =====
        const int q = warp - 4;            // TMEM lane quadrant (warp % 4)
        const int et = threadIdx.x - 128;  // epilogue thread 0..127
        uint8_t* wbuf = sEpi + q * kEpiWarpBytes;
        const uint32_t tempty_leader = CG == 2 ? mapa(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);
        int as = 0;
        uint32_t aphase = 0;
        bool first_epi = true;
        TileSeq seq{&p, cluster_id, num_clusters, static_cast<int>(cta_rank)};
        seq.fetcher = false;
        for (int t = seq.next<CG>(qfull, qempty, qtile); t >= 0; t = seq.next<CG>(qfull, qempty, qtile)) {
            seq.release<CG>(qempty, lane == 0);
            int l, tmp, tn, kb0, kb1, split;
            uint32_t entry;
            tile_unit(p, t, k_blocks, entry, kb0, kb1, split);
            decode(entry, l, tmp, tn);
            const int tm = tmp * CG + static_cast<int>(cta_rank);  // 128-row tile index
            const int row0 = tm * kBM;
            const int col0 = tn * kBN;
            const int row = row0 + q * 32 + lane;
            const bool valid = row < p.m;
            bool released = false;
            mbar_wait(&tfull[as], aphase);
            tc_fence_after();
            if (et == 0 && first_epi) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 33, 0);  // first accumulator ready
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                   static_cast<uint32_t>(as * kBN);
            // Tail split (K-slices of one tile in the last wave): park this slice's
            // accumulator, hand TMEM back to the MMA warp, wait until every slice
            // of the tile has parked; returns this thread's row in slice 0's slot
            // (slots are [column][row] fp32, slice s at + s * CG * 128 * 256).
            auto park_tail_slice = [&]() -> const float* {
                const int ti = (t - p.tail_base) / p.tail_splits;
                const long long slot_stride = static_cast<long long>(kBM) * kBN;
                // Slot layout [column][row] (row fastest): a warp's 32 rows of one
                // column are 128 contiguous bytes, so these stores and the summing
                // loads are coalesced without a shared-memory transpose.
                float* mine = p.tail_ws + (static_cast<long long>(ti * p.tail_splits + split) * CG + cta_rank) *
                                              slot_stride + q * 32 + lane;
                for (int c = 0; c < kBN / 32; ++c) {
                    if (col0 + c * 32 >= p.n) break;  // warp-uniform
                    uint32_t r[32];
                    tmem_ld32(tbase + c * 32, r);
                    tmem_ld_wait();
                    if (valid) {  // rows past m (decode-sized M) are never read back
#pragma unroll
                        for (int j = 0; j < 32; ++j) mine[(c * 32 + j) * kBM] = __uint_as_float(r[j]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2) mbar_arrive_cluster(tempty_leader + static_cast<uint32_t>(as * 8));
                    else mbar_arrive(&tempty[as]);
                }
                released = true;
                // All slices of this tile run in the same (last) wave: wait for
                // every one of them, then each slice sums and stores its share
                // of the 32-column chunks (c % slices == slice), so the
                // reduction is spread over the slices' CTAs.
                named_bar_sync(1, 128);
                if (et == 0) {
                    uint32_t* ctr = p.tail_ctr + ti * CG + cta_rank;
                    const uint32_t done = ((p.tail_seq & 0xFFFFFFu) << 8) | static_cast<uint32_t>(p.tail_splits);
                    if (tail_arrive(ctr, p.tail_seq) != static_cast<uint32_t>(p.tail_splits)) {
                        const uint64_t t0 = globaltimer();
                        for (;;) {
                            uint32_t v;
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                            if (v == done) break;
                            if (globaltimer() - t0 > p.timeout_ns) {
                                record_error(p, l, kErrAgFlagTimeout, static_cast<uint32_t>(ti),
                                             0xFFFE0000u | static_cast<uint32_t>(split), done);
                                break;
                            }
                            __nanosleep(64);
                        }
                    }
                }
                named_bar_sync(1, 128);
                return p.tail_ws + (static_cast<long long>(ti * p.tail_splits) * CG + cta_rank) * slot_stride + q * 32 +
                       lane;
            };
            if (row0 >= p.m) {
                // Fully out-of-range half of a pair tile: nothing to store or signal.
            } else if (MODE != kModeRS && MODE != kModeRSUnits) {
                if (EPI && p.act == kActSwiGLU) {
                    // Gated MLP: each 256-column tile holds 128 gate then 128 up
                    // columns; C gets silu(gate) * up, 128 columns per tile.
                    for (int c = 0; c < kBN / 64; ++c) {
                        const int col = col0 + c * 32;
                        if (col >= p.n) break;  // warp-uniform
                        uint32_t rg[32], ru[32];
                        tmem_ld32(tbase + c * 32, rg);
                        tmem_ld32(tbase + (c + kBN / 64) * 32, ru);
                        tmem_ld_wait();
                        if (valid && p.aux_save) {  // pre-activation (gate and up) for the backward pass
                            float g[32], u[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                g[j] = __uint_as_float(rg[j]);
                                u[j] = __uint_as_float(ru[j]);
                            }
                            const long long aoff = static_cast<long long>(row) * p.ld_aux[l];
                            store_row<32>(p.aux[l], aoff + col, col, p.n, 0, g);
                            store_row<32>(p.aux[l], aoff + col + kBN / 2, col + kBN / 2, p.n, 0, u);
                        }
                        if (valid) {
                            float v[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                v[j] = act_fwd(kActSilu, __uint_as_float(rg[j])) * __uint_as_float(ru[j]);
                            const int ocol = tn * (kBN / 2) + c * 32;
                            store_row<32>(p.c[l], static_cast<long long>(row) * p.ldc_l[l] + ocol, ocol, p.n / 2,
                                          p.out_f32, v);
                        }
                    }
                } else {
                    // Tail split: park this K-slice's accumulator, the last slice to
                    // arrive sums all of them in slice order and runs the epilogue.
                    bool do_store = true;
                    const float* tail_src = nullptr;
                    if (split >= 0) tail_src = park_tail_slice();
                    for (int c = 0; do_store && c < kBN / 32; ++c) {
                        const int col = col0 + c * 32;
                        if (col >= p.n) break;  // warp-uniform
                        if (tail_src && c % p.tail_splits != split) continue;
                        uint32_t r[32];
                        if (!tail_src) {
                            tmem_ld32(tbase + c * 32, r);
                            tmem_ld_wait();
                        }
                        if (valid) {
                            float v[32];
                            if (tail_src) {
                                const long long slot_stride = static_cast<long long>(CG) * kBM * kBN;
#pragma unroll
                                for (int j = 0; j < 32; ++j) v[j] = __ldcg(tail_src + (c * 32 + j) * kBM);
                                for (int x = 1; x < p.tail_splits; ++x) {
                                    float w[32];
#pragma unroll
                                    for (int j = 0; j < 32; ++j) w[j] = __ldcg(tail_src + x * slot_stride + (c * 32 + j) * kBM);
#pragma unroll
                                    for (int j = 0; j < 32; ++j) v[j] += w[j];
                                }
                            } else {
#pragma unroll
                                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                            }
                            if (EPI && p.act_grad == kActSwiGLU) {
                                // Backward of the gated MLP: v = dz for output columns
                                // [col, col+32) of group col/128; the saved pre-activation
                                // holds that group's gate and up columns (256-wide groups),
                                // and C (2n columns, same grouping) receives dgate, dup.
                                const int gcol = (col / (kBN / 2)) * kBN + col % (kBN / 2), ucol = gcol + kBN / 2;
                                const long long abase = static_cast<long long>(row) * p.ld_aux[l];
                                float xg[32], xu[32], dg[32];
                                load_row_bf16<32>(p.aux[l], abase + gcol, gcol, 2 * p.n, xg);
                                load_row_bf16<32>(p.aux[l], abase + ucol, ucol, 2 * p.n, xu);
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    const float sg = 1.0f / (1.0f + __expf(-xg[j]));
                                    dg[j] = v[j] * xu[j] * sg * (1.0f + xg[j] * (1.0f - sg));
                                    v[j] = v[j] * xg[j] * sg;  // dup = dz * silu(gate)
                                }
                                const long long cbase = static_cast<long long>(row) * p.ldc_l[l];
                                store_row<32>(p.c[l], cbase + gcol, gcol, 2 * p.n, p.out_f32, dg);
                                store_row<32>(p.c[l], cbase + ucol, ucol, 2 * p.n, p.out_f32, v);
                                continue;
                            }
                            if (EPI && (p.act_grad || p.act || p.aux_save)) {
                                const long long aoff = static_cast<long long>(row) * p.ld_aux[l] + col;
                                if (p.aux_save) store_row<32>(p.aux[l], aoff, col, p.n, 0, v);
                                if (p.act_grad) {
                                    float x[32];
                                    load_row_bf16<32>(p.aux[l], aoff, col, p.n, x);
#pragma unroll
                                    for (int j = 0; j < 32; ++j) v[j] *= act_bwd(p.act_grad, x[j]);
                                } else if (p.act) {
#pragma unroll
                                    for (int j = 0; j < 32; ++j) v[j] = act_fwd(p.act, v[j]);
                                }
                            }
                            store_row<32>(p.c[l], static_cast<long long>(row) * p.ldc_l[l] + col, col, p.n,
                                          p.out_f32, v);
                        }
                    }
                }
            } else if (MODE == kModeRSUnits) {
                // Ownership blocks narrower than a tile (decode-sized M): every source
                // stores its whole partial tile into the owners' staging planes and
                // stamps flag (tile, source) of each owner in the tile. The owners
                // sum their rows after their own GEMM work (owner_reduce_phase).
                // Through the warp's smem window, so each store instruction writes
                // 4 rows x 128 contiguous bytes.
                const int me = p.global_rank[l];
                const uint32_t parity = p.epoch & 1u;
                const int tile_id = tm * p.tiles_n + tn;
                const int rpr = p.rpr;
                const long long ld_stage = p.ld_stage;
                if (split >= 0) {
                    // Split-K (fewer tiles than SMs, e.g. one GPU's decode share): the
                    // slices of the tile park their accumulators, each slice sums its
                    // share of the 32-column chunks in slice order (deterministic) and
                    // stores them into the owners' staging planes (row per thread, 128
                    // contiguous bytes); the last slice to finish stamps the flags.
                    const float* src = park_tail_slice();
                    const long long slot_stride = static_cast<long long>(CG) * kBM * kBN;
                    const int o = valid ? row / rpr : 0;
                    for (int c = split; c < kBN / 32; c += p.tail_splits) {
                        const int colc = col0 + c * 32;
                        if (colc >= p.n) break;  // warp-uniform
                        if (!valid || (p.dbg & 8)) continue;
                        float v[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = __ldcg(src + (c * 32 + j) * kBM);
                        for (int x = 1; x < p.tail_splits; ++x) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) v[j] += __ldcg(src + x * slot_stride + (c * 32 + j) * kBM);
                        }
                        long long pl;
                        float* const dst = rs_plane_base(p, o, me, pl);
                        const long long e = parity * p.stage_parity + pl +
                                            (row - static_cast<long long>(o) * rpr) * ld_stage + colc;
                        if (colc + 32 <= p.n) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                st_part4<PB>(dst, e + j, make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                        } else {
                            for (int j = 0; j < 32 && colc + j < p.n; j += 4)  // ld_stage pads to 256 columns
                                st_part4<PB>(dst, e + j, make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                        }
                    }
                    // Every slice's stores precede its arrival; the last arrival
                    // (acquire) stamps the owners' flags (release, cumulative).
                    named_bar_sync(1, 128);
                    if (et == 0) {
                        __threadfence_system();
                        const int ti = (t - p.tail_base) / p.tail_splits;
                        uint32_t* ctr2 = p.tail_ctr + kTailCtrCap + ti * CG + cta_rank;
                        if (tail_arrive(ctr2, p.tail_seq) == static_cast<uint32_t>(p.tail_splits)) {
                            const int o0 = row0 / rpr, o1 = (min(row0 + kBM, p.m) - 1) / rpr;
                            trace_event(p, l, kEvTileWrite, me, tm, tn, static_cast<uint32_t>(o0));
                            for (int oo = o0; oo <= o1; ++oo) rs_flag_set(p, l, oo, tile_id, me);
                        }
                    }
                } else {
                // Staging address of each of the 8 rows this lane writes through the
                // smem window (row it * 4 + lane / 8 of the warp's 32), computed once
                // per tile: the chunk loop only adds the column (the per-store owner
                // division and 64-bit plane arithmetic dominated it: C1 1.45 us per
                // 32-column chunk).
                char* rowp[8];
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int grow = row0 + q * 32 + it * 4 + (lane >> 3);
                    rowp[it] = nullptr;
                    if (grow < p.m) {
                        const int o = grow / rpr;
                        long long pl;
                        float* const dst = rs_plane_base(p, o, me, pl);
                        const long long e = parity * p.stage_parity + pl + (grow - static_cast<long long>(o) * rpr) * ld_stage;
                        rowp[it] = reinterpret_cast<char*>(dst) + e * (PB ? 2 : 4);
                    }
                }
                for (int c = 0; c < kBN / 32; ++c) {
                    const int colc = col0 + c * 32;
                    if (colc >= p.n) break;  // warp-uniform
                    if (et == 0 && first_epi && (c == 1 || c == 4)) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 34 + c, 0);  // chunk c of the first tile (profiling)
                    uint32_t r[32];
                    tmem_ld32(tbase + c * 32, r);
                    tmem_ld_wait();
                    if (p.dbg & 8) continue;  // dbg 8: profiling ablation, no staging stores
                    if (row0 + q * 32 >= p.m) continue;  // no rows of this warp in range
                    // A partly valid warp (decode M) stores its rows directly.
                    if (row0 + q * 32 + 32 > p.m || (p.dbg & 64)) {  // dbg 64: ablation, always direct
                        if (valid) {
                            const int o = row / rpr;
                            long long pl;
                            float* const dst = rs_plane_base(p, o, me, pl);
                            const long long e = parity * p.stage_parity + pl +
                                                (row - static_cast<long long>(o) * rpr) * ld_stage + colc;
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                st_part4<PB>(dst, e + j,
                                             make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                         __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
                        }
                        continue;
                    }
                    epi_stage(wbuf, lane, r);
                    const int col = colc + (lane & 7) * 4;
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        if (rowp[it] == nullptr || col >= p.n) continue;
                        st_part4<PB>(reinterpret_cast<float*>(rowp[it]), col, epi_read(wbuf, it * 4 + (lane >> 3), lane & 7));
                    }
                }
                // The accumulator is in staging now: hand TMEM back to the MMA warp.
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2) mbar_arrive_cluster(tempty_leader + static_cast<uint32_t>(as * 8));
                    else mbar_arrive(&tempty[as]);
                }
                released = true;
                named_bar_sync(1, 128);
                const int o0 = row0 / p.rpr, o1 = (min(row0 + kBM, p.m) - 1) / p.rpr;
                if (et == 0) trace_event(p, l, kEvTileWrite, me, tm, tn, static_cast<uint32_t>(o0));
                for (int o = o0 + et; o <= o1; o += 128)
                    rs_flag_set(p, l, o, tile_id, me);
                }  // whole-tile staging
            } else {
                const int me = p.global_rank[l];
                const uint32_t parity = p.epoch & 1u;
                const int owner = valid ? row / p.rpr : -1;
                const bool remote = valid && owner != me;
                const int tile_id = tm * p.tiles_n + tn;
                const int rlast = min(row0 + kBM, p.m) - 1;
                const int o0 = row0 / p.rpr, o1 = rlast / p.rpr;
                if (p.rs_chain) {
                    // Chained partial sums (every rank in this launch, rank-major
                    // schedule with every owner's block moved behind all other tiles,
                    // ownership blocks aligned to tiles). The partials of a tile are
                    // summed in the canonical order — the other sources ascending,
                    // then the owner — as a chain through the owner's staging plane:
                    // each source adds its accumulator to the running sum its
                    // predecessor left (flag (tile, predecessor)) and writes it back;
                    // the owner adds its own accumulator to that one plane instead of
                    // reading tp-1 partials. Every wait targets an earlier section.
                    // (A variant where the last source closes each chain, so the owner
                    // blocks need no tail, measured no faster: it trades the tail's
                    // weight re-stream for staging the owners' partials.)
                    const int o = o0, tp = p.tp;
                    const int last = o == tp - 1 ? tp - 2 : tp - 1;
                    const bool own_tile = me == o;
                    const bool closes = own_tile;
                    const int pred = own_tile ? last : (me - 1 == o ? me - 2 : me - 1);
                    const long long lr0 = row0 - static_cast<long long>(o) * p.rpr;
                    float* const sbase = p.staging[o];  // plane 0 of the owner, element offsets below
                    const long long e0 = parity * p.stage_parity + stage_tile_off(lr0, tn, p.tiles_n) + q * 1024;
                    if (et == 0) {
                        if (pred >= 0)
                            wait_flag(p.rs_flags[o] + tile_id * tp + pred, p.epoch, p, l, kErrRsFlagTimeout,
                                      static_cast<uint32_t>(tile_id), static_cast<uint32_t>(pred));
                        if (closes) trace_event(p, l, kEvReduce, me, tm, tn, static_cast<uint32_t>(o));
                    }
                    named_bar_sync(1, 128);
                    const int os = p.slot_of[o];
                    void* cdst = closes ? p.c[os] : nullptr;
                    const int ldc_o = closes ? p.ldc_l[os] : 0;
                    for (int c = 0; c < kBN / 32; ++c) {
                        const int colc = col0 + c * 32;
                        if (colc >= p.n) break;  // warp-uniform
                        float4 sum[8];
                        if (pred >= 0) {  // running sum, loaded before the TMEM round trip
#pragma unroll
                            for (int it = 0; it < 8; ++it)
                                sum[it] = ld_part4<PB>(sbase, e0 + c * 4096 + it * 128 + lane * 4);
                        }
                        uint32_t r[32];
                        tmem_ld32(tbase + c * 32, r);
                        tmem_ld_wait();
                        epi_stage(wbuf, lane, r);
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            const int i = it * 4 + (lane >> 3), g = lane & 7;
                            const int col = colc + g * 4;
                            if (col >= p.n) continue;
                            float4 v = epi_read(wbuf, i, g);
                            if (pred >= 0) {
                                v.x = sum[it].x + v.x;
                                v.y = sum[it].y + v.y;
                                v.z = sum[it].z + v.z;
                                v.w = sum[it].w + v.w;
                            }
                            if (closes) {
                                float acc[4] = {v.x, v.y, v.z, v.w};
                                store_row<4>(cdst, (lr0 + q * 32 + i) * ldc_o + col, col, p.n, p.out_f32, acc);
                            } else {
                                st_part4<PB>(sbase, e0 + c * 4096 + it * 128 + lane * 4, v);
                            }
                        }
                    }
                    named_bar_sync(1, 128);
                    if (!closes && et == 0) {
                        trace_event(p, l, kEvTileWrite, me, tm, tn, static_cast<uint32_t>(o));
                        rs_flag_set(p, l, o, tile_id, me);
                    }
                } else {
                if (p.fused_reduce) {
                    // FusedReduce: each owner zeroes this parity's accumulator on its
                    // stream before the launch and stamps fr_ready; wait for that once.
                    if (et <= o1 - o0 && o0 + et != me)
                        wait_flag(p.fr_ready[o0 + et], p.epoch, p, l, kErrRsFlagTimeout,
                                  static_cast<uint32_t>(tile_id), static_cast<uint32_t>(o0 + et));
                    named_bar_sync(1, 128);
                }
                // Phase 1: ship remote rows to their owners (Alg. 1 line 5): plain stores
                // into the owner's staging plane for this source (WriteAlltoAll), or
                // vector red.add into the owner's fp32 accumulator (FusedReduce).
                // Each 32-column chunk goes TMEM -> registers -> this warp's smem
                // window -> coalesced global stores (4 rows x 128 B per instruction).
                if (__any_sync(0xffffffffu, remote) && !(p.dbg & 1)) {
                    // RS mode: ownership blocks are whole 128-row tiles, so the owner is
                    // uniform over this CTA's rows. WriteAlltoAll staging is tile-major:
                    // each (tile, source) partial is one contiguous 128 KiB run in the
                    // order the owner reads it back (DRAM-page and NVLink friendly).
                    // FusedReduce also runs with blocks narrower than a tile: its owner
                    // is per row.
                    const long long lr0 = row0 - static_cast<long long>(o0) * p.rpr;
                    float* const wbase = p.staging[o0];
                    const long long we0 = parity * p.stage_parity + me * p.stage_plane +
                                          stage_tile_off(lr0, tn, p.tiles_n) + q * 1024;
                    for (int c = 0; c < kBN / 32; ++c) {
                        const int colc = col0 + c * 32;
                        if (colc >= p.n) break;  // warp-uniform
                        uint32_t r[32];
                        tmem_ld32(tbase + c * 32, r);
                        tmem_ld_wait();
                        epi_stage(wbuf, lane, r);
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            const int i = it * 4 + (lane >> 3), g = lane & 7;
                            const int col = colc + g * 4;
                            const int grow = row0 + q * 32 + i;
                            if (grow >= p.m || col >= p.n) continue;
                            const float4 v = epi_read(wbuf, i, g);
                            if (p.fused_reduce) {
                                const int o = grow / p.rpr;
                                if (o != me)
                                    red_add_f4(p.fr_acc[o] + (grow - static_cast<long long>(o) * p.rpr) * p.ld_stage + col,
                                               v.x, v.y, v.z, v.w);
                            } else {
                                st_part4<PB>(wbase, we0 + c * 4096 + it * 128 + lane * 4, v);
                            }
                        }
                    }
                    // No per-thread system fence: the named barrier below orders these stores
                    // before the signalling thread's st.release.sys (release is cumulative).
                }
                named_bar_sync(1, 128);
                // Signal each owner in this tile that our partial landed.
                if (et <= o1 - o0) {
                    const int o = o0 + et;
                    if (o != me) {
                        trace_event(p, l, kEvTileWrite, me, tm, tn, static_cast<uint32_t>(o));
                        rs_flag_set(p, l, o, tile_id, me);
                    }
                }
                // Phase 2: owned rows = sum of all partials in the canonical order.
                const bool mine_in_tile = (me >= o0 && me <= o1);
                if (mine_in_tile && (p.dbg & 2)) {
                    // Ablation: the owner stores only its own accumulator (no waits, no reduce).
                    const bool owned = valid && owner == me;
                    for (int c = 0; c < kBN / 32; ++c) {
                        const int col = col0 + c * 32;
                        if (col >= p.n) break;
                        uint32_t r[32];
                        tmem_ld32(tbase + c * 32, r);
                        tmem_ld_wait();
                        if (owned) {
                            float v[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                            store_row<32>(p.c[l], static_cast<long long>(row - me * p.rpr) * p.ldc_l[l] + col, col,
                                          p.n, p.out_f32, v);
                        }
                    }
                } else if (mine_in_tile) {
                    if (et == 0) {
                        for (int s = 0; s < p.tp; ++s)
                            if (s != me)
                                wait_flag(p.rs_flags[me] + tile_id * p.tp + s, p.epoch, p, l, kErrRsFlagTimeout,
                                          static_cast<uint32_t>(tile_id), static_cast<uint32_t>(s));
                        trace_event(p, l, kEvReduce, me, tm, tn, static_cast<uint32_t>(me));
                    }
                    named_bar_sync(1, 128);
                    // Coalesced fixed-order sum: the own accumulator chunk is staged
                    // in this warp's smem window; lanes then walk 4 rows x 32 columns
                    // per step, loading every source's float4 before adding in the
                    // canonical order (deterministic; FusedReduce: the accumulator of
                    // the others + own).
                    const long long lr0 = row0 - static_cast<long long>(me) * p.rpr;  // tile's first owned row
                    const float* src0 = p.fused_reduce ? p.fr_acc[me] : p.staging[me];
                    const long long se0 = parity * p.stage_parity + stage_tile_off(lr0, tn, p.tiles_n) + q * 1024;
                    for (int c = 0; c < kBN / 32; ++c) {
                        const int colc = col0 + c * 32;
                        if (colc >= p.n) break;  // warp-uniform
                        uint32_t r[32];
                        tmem_ld32(tbase + c * 32, r);
                        tmem_ld_wait();
                        epi_stage(wbuf, lane, r);
#pragma unroll
                        for (int it0 = 0; it0 < 8; it0 += kEpiU) {
                            float4 v[kEpiU][kMaxRanks];
                            bool ok[kEpiU];
#pragma unroll
                            for (int u = 0; u < kEpiU; ++u) {
                                const int i = (it0 + u) * 4 + (lane >> 3), g = lane & 7;
                                const int col = colc + g * 4;
                                const long long lr = lr0 + q * 32 + i;  // row within my block
                                ok[u] = row0 + q * 32 + i < p.m && col < p.n && lr >= 0 && lr < p.rpr;
                                if (ok[u]) {
                                    if (p.fused_reduce) {
                                        v[u][0] = ld_cg_f4(src0 + lr * p.ld_stage + col);
                                    } else {
                                        const long long e = se0 + c * 4096 + (it0 + u) * 128 + lane * 4;
#pragma unroll
                                        for (int s2 = 0; s2 < kMaxRanks; ++s2)
                                            if (s2 < p.tp && s2 != me)
                                                v[u][s2] = ld_part4<PB>(src0, e + s2 * p.stage_plane);
                                    }
                                }
                            }
#pragma unroll
                            for (int u = 0; u < kEpiU; ++u) {
                                if (!ok[u]) continue;
                                const int i = (it0 + u) * 4 + (lane >> 3), g = lane & 7;
                                const float4 own = epi_read(wbuf, i, g);
                                float acc[4];
                                if (p.fused_reduce) {  // arrival-order sum of the others + own
                                    acc[0] = v[u][0].x + own.x;
                                    acc[1] = v[u][0].y + own.y;
                                    acc[2] = v[u][0].z + own.z;
                                    acc[3] = v[u][0].w + own.w;
                                } else {
                                    // The canonical deterministic order (same as the chain and
                                    // the decode owner units): the other sources ascending, then
                                    // the owner's own partial.
                                    bool first = true;
#pragma unroll
                                    for (int s2 = 0; s2 < kMaxRanks; ++s2) {
                                        if (s2 >= p.tp) break;
                                        if (s2 == me) continue;
                                        sum_into(acc, v[u][s2], first);
                                    }
                                    sum_into(acc, own, first);
                                }
                                const int col = colc + g * 4;
                                store_row<4>(p.c[l], (lr0 + q * 32 + i) * p.ldc_l[l] + col, col, p.n, p.out_f32, acc);
                            }
                        }
                    }
                }
                }  // !rs_chain
            }
            if (!released) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2) mbar_arrive_cluster(tempty_leader + static_cast<uint32_t>(as * 8));
                    else mbar_arrive(&tempty[as]);
                }
            }
            if (et == 0 && first_epi) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 34, 0);  // first tile stored
            first_epi = false;
            if (++as == 2) {
                as = 0;
                aphase ^= 1u;
            }
        }
        if (MODE == kModeRSUnits) owner_reduce<PB, TWU>(p, et, 128, 4, &red_slot[1], false);
    }
    if (MODE == kModeRSUnits && warp < 2) {
        // The producer and MMA warps are done with the GEMM: a third group of
        // reduction units (shortens the last block's exposed sums).
        __syncwarp();
        owner_reduce<PB, TWU>(p, threadIdx.x, 64, 5, &red_slot[2], false);
    }

    if (CG == 2) cluster_sync();
    else __syncthreads();
    if (warp == 0 && lane == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 1, 0);  // CTA done
    if (warp == 2) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_pair(tmem_base, kTmemCols);
        else tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ===========================================================================
// Streaming decode kernel (decode-sized M: one GPU's share of a decode step).
//
// With M <= 128 tokens the tile kernel's 128 x 256 output tiles are too few to
// occupy 148 SMs (one GPU's Llama-2-70B up-proj share, N/TP = 3584: 14 tiles)
// and each tile wastes 7/8 of its MMA rows; the op is a stream of the weight
// shard through HBM. Here the weights are the MMA's M operand (128-row
// n-tiles, K-major, TMA) and the tokens its N operand (sk_mp = M padded to 16):
// D[128 x sk_mp] += W[128 x 64] . T[sk_mp x 64]^T per k-block, fp32 in TMEM.
// The (slot, n-tile, k-block) space is split evenly over the CTAs (stream-K),
// so every SM streams the same number of weight bytes; an n-tile cut between
// CTAs is summed by the last of them to arrive, in segment (K) order, so the
// result does not depend on arrival order. A deep smem ring (up to 12 stages of
// 16 KiB weights) keeps ~150 KiB per SM in flight.
//   Plain / AG: C[m, n] (+ activation). AG: the producer streams weight stages
//     before it waits for the gathered token rows (in-kernel transfer counters or
//     copy-engine comm-tile flags), so the AllGather hides under the weight
//     stream; warp 3 runs the in-kernel transfer (ag_transfer).
//   RSUnits: every finished n-tile's partial goes to its owners' staging planes
//     with flag (n-tile, source); the CTA that finishes the n-tile then sums its
//     own rank's rows of it over every source (after their flags) into C, so
//     the reduction runs in the epilogue that just produced the tile (no
//     separate reduction pass, no cold code after the weight stream).
// ===========================================================================
constexpr int kSkWBytes = kSkRows * kBK * 2;  // 16 KiB weight stage
constexpr int kSkMaxSegs = 8;                 // K-segments per n-tile (the host sizes the grid to keep it)
constexpr int kSkBarBytes = 512;

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// First work unit of CTA c, and the CTA whose range holds unit x (sk_work >= sk_ctas,
// so the range starts strictly increase).
// (32-bit: the host keeps sk_work * (sk_ctas + 1) below 2^31; 64-bit divisions
// inline ~100 instructions at every call site.)
__device__ __forceinline__ long long sk_start(const GemmParams& p, int c) {
    return static_cast<long long>(static_cast<uint32_t>(c) * static_cast<uint32_t>(p.sk_work) /
                                  static_cast<uint32_t>(p.sk_ctas));
}
__device__ __forceinline__ int sk_cta_of(const GemmParams& p, long long x) {
    const uint32_t w = static_cast<uint32_t>(p.sk_work);
    return static_cast<int>((static_cast<uint32_t>(x + 1) * static_cast<uint32_t>(p.sk_ctas) + w - 1) / w) - 1;
}
// Walks one CTA's range as segments (tile tt = slot * sk_nt + n-tile, k-blocks [kb0, kb1)).
struct SkIter {
    long long cur, end;
    int kb;
    int cl = 1, c = 0, t = 0, nq = 0, ntiles = 0;  // cluster split-K: tiles t, t + nq, ...; K-segment c of cl
    __device__ bool next(int& tt, int& kb0, int& kb1) {
        if (cl > 1) {
            if (t >= ntiles) return false;
            tt = t;
            kb0 = c * kb / cl;
            kb1 = (c + 1) * kb / cl;
            t += nq;
            return true;
        }
        if (cur >= end) return false;
        tt = static_cast<int>(cur / kb);
        kb0 = static_cast<int>(cur % kb);
        kb1 = static_cast<int>(min(static_cast<long long>(kb), kb0 + (end - cur)));
        cur += kb1 - kb0;
        return true;
    }
};
__device__ __forceinline__ SkIter sk_iter(const GemmParams& p, long long r0, long long r1) {
    SkIter it{r0, r1, p.sk_kb};
    if (p.sk_cluster > 1) {
        it.cl = p.sk_cluster;
        it.c = static_cast<int>(blockIdx.x) % it.cl;
        it.t = static_cast<int>(blockIdx.x) / it.cl;
        it.nq = p.sk_ctas / it.cl;
        it.ntiles = static_cast<int>(p.sk_work / p.sk_kb);
    }
    return it;
}
__device__ __forceinline__ void st_shared_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

// Slot of the segment of tile tt held by CTA c: 2c when the tile holds the
// CTA's first unit, else 2c + 1 (the CTA's last segment). Indexes the fp32
// partials parked in tail_ws; sk_ctr[tt] counts the tile's parked segments
// (tagged with the launch sequence number, tail_arrive).
__device__ __forceinline__ int sk_slot_index(const GemmParams& p, int c, int tt) {
    return 2 * c + (sk_start(p, c) >= static_cast<long long>(tt) * p.sk_kb ? 0 : 1);
}
__device__ __forceinline__ float* sk_slot(const GemmParams& p, int c, int tt) {
    return p.tail_ws + static_cast<long long>(sk_slot_index(p, c, tt)) * kSkRows * p.sk_mp;
}
// Final values of 16 tokens (m0..m0+15) of output column `col` of slot l.
template <int MODE, int PB, int ACT>
__device__ __forceinline__ void sk_store(const GemmParams& p, int l, int col, int m0, int mv, const float (&v)[16]) {
    if (col >= p.n) return;
    if (MODE == kModeRSUnits) {
        const int me = p.global_rank[l], rpr = p.rpr;
        const long long base = static_cast<long long>(p.epoch & 1u) * p.stage_parity + col;
        // Owner and row within its block advance with the row (one division per
        // 16 rows, not one per store).
        int o = m0 / rpr, lr = m0 - o * rpr;
        long long pl;
        float* dst = rs_plane_base(p, o, me, pl);
        long long e = base + pl + static_cast<long long>(lr) * p.ld_stage;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (m0 + i >= mv) break;
            if (lr == rpr) {
                ++o;
                lr = 0;
                dst = rs_plane_base(p, o, me, pl);
                e = base + pl;
            }
            if (PB) reinterpret_cast<__nv_bfloat16*>(dst)[e] = __float2bfloat16_rn(v[i]);
            else dst[e] = v[i];
            ++lr;
            e += p.ld_stage;
        }
    } else {
        const long long ldc = p.ldc_l[l];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int m = m0 + i;
            if (m >= mv) break;
            const float x = ACT ? act_fwd(p.act, v[i]) : v[i];
            if (p.out_f32) static_cast<float*>(p.c[l])[m * ldc + col] = x;
            else static_cast<__nv_bfloat16*>(p.c[l])[m * ldc + col] = __float2bfloat16_rn(x);
        }
    }
}

// The canonical-order sum of this rank's rows of n-tile j (other sources
// ascending, then this rank) into C, KB float4 groups per thread in flight with
// their sources (RMAX >= tp; NVLS loads one reduced group). Epilogue warps (128 threads).
template <int PB, int KB, int RMAX>
__device__ __forceinline__ void sk_rs_sum(const GemmParams& p, int l, int j, int F, int me, int tp, long long e0,
                                          const float* sbase, int et) {
    for (int f0 = et; f0 < F; f0 += 128 * KB) {
        float4 w[KB][RMAX];
#pragma unroll
        for (int u = 0; u < KB; ++u) {
            const int f = f0 + u * 128;
            const int lr = f / (kSkRows / 4), c2 = j * kSkRows + (f % (kSkRows / 4)) * 4;
            if (f >= F || c2 >= p.n) continue;
            const long long e = e0 + static_cast<long long>(lr) * p.ld_stage + c2;
            if (p.nvls) {
                asm volatile("fence.proxy.alias;" ::: "memory");
                w[u][0] = nvls_ld_reduce4(p, e + me * p.stage_plane);
            } else {
#pragma unroll
                for (int s2 = 0; s2 < RMAX; ++s2)
                    if (s2 < tp) w[u][s2] = ld_part4<PB>(sbase, e + s2 * p.stage_plane);
            }
        }
#pragma unroll
        for (int u = 0; u < KB; ++u) {
            const int f = f0 + u * 128;
            const int lr = f / (kSkRows / 4), c2 = j * kSkRows + (f % (kSkRows / 4)) * 4;
            if (f >= F || c2 >= p.n) continue;
            float acc[4];
            bool first = true;
            if (p.nvls) {
                sum_into(acc, w[u][0], first);
            } else {
#pragma unroll
                for (int s2 = 0; s2 < RMAX; ++s2)
                    if (s2 < tp && s2 != me) sum_into(acc, w[u][s2], first);
#pragma unroll
                for (int s2 = 0; s2 < RMAX; ++s2)
                    if (s2 == me) sum_into(acc, w[u][s2], first);
            }
            store_row<4>(p.c[l], static_cast<long long>(lr) * p.ldc_l[l] + c2, c2, p.n, p.out_f32, acc);
        }
    }
}

// GEMM-RS in the streaming kernel, once n-tile j of slot l is complete in this
// CTA and its partial rows are in every owner's plane (this rank's own rows
// included): stamp the peers' flags, then finish this rank's own rows here —
// wait for the other sources' partials of the tile and sum the planes in the
// canonical order (other sources ascending, then this rank) into C. Every CTA
// publishes a tile before it waits on that tile, and CTAs walk their tiles in
// order, so the waits cannot form a cycle. Epilogue warps (128 threads).
template <int PB>
__device__ __forceinline__ void sk_rs_finish(const GemmParams& p, int l, int j, int mv, int et) {
    if (p.nvls) asm volatile("fence.proxy.alias;" ::: "memory");  // own rows: unicast stores, multicast reads
    named_bar_sync(1, 128);
    const int me = p.global_rank[l], tp = p.tp, rpr = p.rpr;
    if (et == 0) trace_event(p, l, kEvTileWrite, me, 0, j, 0u);
    if (et < tp && et != me) rs_flag_set(p, l, et, j, me);
    if (et < tp && et != me)
        wait_flag(p.rs_flags[me] + j * tp + et, p.epoch, p, l, kErrRsFlagTimeout,
                  static_cast<uint32_t>(j), static_cast<uint32_t>(et));
    named_bar_sync(1, 128);
    if (et == 0) trace_event(p, l, kEvReduce, me, 0, j, static_cast<uint32_t>(me));
    const float* const sbase = p.staging[me];
    const long long e0 = static_cast<long long>(p.epoch & 1u) * p.stage_parity;
    const int F = min(rpr, mv - me * rpr) * (kSkRows / 4);  // float4 groups of my rows
    // One source (one rank per owner, or NVLS summing in the switch): four groups
    // per thread in flight; the rows are otherwise a chain of dependent DRAM
    // round trips (M=64 at tp=1: 16 per thread). More sources: one group at a
    // time with every source's load (this code runs once per launch on a cold
    // instruction cache, where a longer body measured slower).
    if (p.nvls || tp == 1) sk_rs_sum<PB, 4, 1>(p, l, j, F, me, tp, e0, sbase, et);
    else sk_rs_sum<PB, 1, kMaxRanks>(p, l, j, F, me, tp, e0, sbase, et);
}

template <int MODE, int PB = 0, int ACT = 0>
__global__ void __launch_bounds__(kThreads, 1) flux_stream_kernel(const __grid_constant__ GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int mp = p.sk_mp, ns = p.sk_stages, kbn = p.sk_kb;
    const int tbytes = mp * kBK * 2;  // token stage: mp rows x 128 B (multiple of 2 KiB)
    uint8_t* sW = smem;
    uint8_t* sT = sW + ns * kSkWBytes;
    uint8_t* sComm = sT + ns * tbytes;  // AG: 2 x kPieceBytes
    // Cluster split-K: the leader's reduction buffer, one [128 columns][mp + 4]
    // fp32 slot per non-leader segment (padded rows: conflict-free v4 stores).
    const int cl = p.sk_cluster, ldr = mp + 4;
    const bool ring = cl > 1 && p.sk_red_ring;  // one tile per cluster: the drained ring holds the slots
    // Ring mode with more than one 16-row chunk (GEMM-RS excepted: its owner finish
    // needs the whole tile from one CTA): every CTA sums and stores the chunks
    // q == its rank (mod cl), so the slices spread over the cluster instead of
    // converging on the leader.
    const bool dist = ring && MODE != kModeRSUnits && min(p.m, mp) > 16;
    // Distributed slots hold only the receiver's chunks: chunk q at row (q / cl) * 16
    // of a [128 columns][16 * ceil(chunks / cl) + 4] slot (same conflict-free padding).
    const int ldd = 16 * (((min(p.m, mp) + 15) / 16 + cl - 1) / max(cl, 1)) + 4;
    float* sRed = ring ? reinterpret_cast<float*>(sW) : reinterpret_cast<float*>(sComm + (MODE == kModeAG ? 2 * kPieceBytes : 0));
    const int red_bytes = cl > 1 && !ring ? (cl - 1) * kSkRows * ldr * 4 : 0;
    uint64_t* full = reinterpret_cast<uint64_t*>(sComm + (MODE == kModeAG ? 2 * kPieceBytes : 0) + red_bytes);
    uint64_t* empty = full + kSkMaxStages;
    uint64_t* tfull = empty + kSkMaxStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* cbar = tempty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cbar + 2);
    int* red_slot = reinterpret_cast<int*>(tmem_slot + 2);
    uint64_t* red_bar = reinterpret_cast<uint64_t*>(red_slot + 4);  // [0] leader: segments in, [1] buffer free
    static_assert((2 * kSkMaxStages + 6) * 8 + 8 + 16 + 16 <= kSkBarBytes, "barrier region");  // red_slot[0..3], red_bar[0..1]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tmem_cols = 2u * static_cast<uint32_t>(p.sk_acc_cols);
    if (warp == 0 && lane == 0) {
        trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 0, 0);
        for (int l = 0; l < kMaxRanks; ++l) {
            if (p.c[l] == nullptr) break;
            tma_prefetch(&p.tma_a[l]);
            tma_prefetch(&p.tma_b[l]);
        }
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
            mbar_init(&cbar[a], 1);
        }
        if (cl > 1) {
            mbar_init(&red_bar[0], (cl - 1) * 128);
            mbar_init(&red_bar[1], dist ? cl - 1 : 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) tmem_alloc(tmem_slot, tmem_cols);
    tc_fence_before();
    __syncthreads();
    if (cl > 1) cluster_sync();  // every CTA's barriers initialised before remote arrivals
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const bool has_work = static_cast<int>(blockIdx.x) < p.sk_ctas;
    const long long r0 = has_work ? sk_start(p, blockIdx.x) : 0, r1 = has_work ? sk_start(p, blockIdx.x + 1) : 0;

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t ready = MODE == kModeAG && !p.ag_direct ? 0u : 0xFFFFFFFFu;  // AG: bit l = slot l's token rows landed
            int pend_stage[kSkMaxStages], pend_kb[kSkMaxStages], pend_l[kSkMaxStages];
            int np = 0;
            // AG: token loads wait for the gathered rows; weight stages stream meanwhile.
            auto flush = [&]() {
                for (int i = 0; i < np; ++i) {
                    const int l = pend_l[i];
                    if (!((ready >> l) & 1u)) {
                        if (p.sm_transfer) {
                            for (int g = 0; g * kBM < p.m; ++g)
                                wait_flag(p.ag_ctr[p.global_rank[l]] + g, p.ag_mult * ag_group_target(p, g), p, l,
                                          kErrAgFlagTimeout, static_cast<uint32_t>(g), 0xFFFD0000u);
                        } else {
                            for (int f = 0; f * p.rpct < p.m; ++f)
                                wait_flag(p.ag_flags[l] + f, p.epoch, p, l, kErrAgFlagTimeout, static_cast<uint32_t>(f),
                                          0xFFFD0000u);
                        }
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        trace_event(p, l, kEvComputeStart, p.global_rank[l], 0, 0, 0);
                        ready |= 1u << l;
                    }
                    tma_load_2d(sT + pend_stage[i] * tbytes, &p.tma_a[l], &full[pend_stage[i]], pend_kb[i] * kBK, 0);
                }
                np = 0;
            };
            SkIter it = sk_iter(p, r0, r1);
            int tt, kb0, kb1;
            while (it.next(tt, kb0, kb1)) {
                const int l = tt / p.sk_nt, j = tt % p.sk_nt;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    mbar_expect_tx(&full[stage], kSkWBytes + tbytes);
                    tma_load_2d(sW + stage * kSkWBytes, &p.tma_b[l], &full[stage], kb * kBK, j * kSkRows);
                    if ((ready >> l) & 1u) {
                        tma_load_2d(sT + stage * tbytes, &p.tma_a[l], &full[stage], kb * kBK, 0);
                    } else {
                        pend_stage[np] = stage;
                        pend_kb[np] = kb;
                        pend_l[np] = l;
                        if (++np == ns) flush();
                    }
                    if (++stage == ns) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
            flush();
            trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 2, 0);  // producer done (launch profiling)
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            const uint32_t idesc = make_idesc(kSkRows, mp);
            int stage = 0, as = 0;
            uint32_t phase = 0, aphase = 0;
            SkIter it = sk_iter(p, r0, r1);
            int tt, kb0, kb1;
            while (it.next(tt, kb0, kb1)) {
                mbar_wait(&tempty[as], aphase ^ 1u);
                tc_fence_after();
                const uint32_t d = tmem_base + static_cast<uint32_t>(as * p.sk_acc_cols);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t adesc = smem_desc_sw128(sW + stage * kSkWBytes);
                    const uint64_t bdesc = smem_desc_sw128(sT + stage * tbytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / kUmmaK; ++kk)
                        umma_bf16(d, adesc + 2ull * kk, bdesc + 2ull * kk, idesc, (kb > kb0 || kk != 0) ? 1u : 0u);
                    umma_commit(&empty[stage]);
                    if (++stage == ns) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                umma_commit(&tfull[as]);
                if (++as == 2) {
                    as = 0;
                    aphase ^= 1u;
                }
            }
        }
    } else if (warp == 3) {
        if (MODE == kModeAG && p.nvls) ag_push_nvls(p, lane);
        else if (MODE == kModeAG && p.sm_transfer && lane == 0) ag_transfer(p, sComm, cbar);
    } else if (warp >= 4) {
        // ===== epilogue: warp q holds weight rows (output columns) 32q..32q+31 of the n-tile =====
        // Whole n-tiles are stored straight from TMEM. A tile cut between CTAs
        // (K-segments) is parked as fp32 partials; the CTA whose segment arrives
        // last (a launch-tagged arrival counter per tile) sums every segment in
        // segment (K) order and stores the tile, so no CTA waits for another and
        // the result does not depend on arrival order.
        const int q = warp - 4, et = threadIdx.x - 128;
        const int cit = q * 32 + lane;  // column within the n-tile
        const int mv = min(p.m, mp);    // valid token rows
        int as = 0;
        uint32_t aphase = 0;
        int tt, kb0, kb1;
        if (cl > 1) {
            // Cluster split-K: CTA c of the cluster holds K-segment c of the tile;
            // the non-leaders put their fp32 accumulators into the leader's shared
            // memory (st.shared::cluster), the leader adds them to its own in
            // segment order and stores the tile. No global round trip, nothing
            // waits outside the cluster.
            const uint32_t crank = cluster_ctarank();
            uint32_t fphase = 0, ephase = 0;
            SkIter cit_it = sk_iter(p, r0, r1);
            while (cit_it.next(tt, kb0, kb1)) {
                const int l = tt / p.sk_nt, j = tt % p.sk_nt;
                const int col = j * kSkRows + cit;
                mbar_wait(&tfull[as], aphase);
                tc_fence_after();
                const uint32_t tbase =
                    tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(as * p.sk_acc_cols);
                if (dist) {
                    // 1. My MMAs retired: my drained ring may take the other CTAs' slices;
                    //    wait until every other CTA's ring may take mine.
                    if (et < cl && et != static_cast<int>(crank))
                        mbar_arrive_cluster(mapa(smem_u32(&red_bar[1]), static_cast<uint32_t>(et)));
                    mbar_wait_acq_cluster(&red_bar[1], 0);
                    // 2. My segment's chunks that other CTAs own, into their slot for my segment.
                    for (int m0 = 0; m0 < mv; m0 += 16) {
                        const int d = (m0 >> 4) % cl;
                        if (d == static_cast<int>(crank)) continue;
                        const int sl = static_cast<int>(crank) < d ? static_cast<int>(crank) : static_cast<int>(crank) - 1;
                        const uint32_t dst = mapa(smem_u32(sRed + (sl * kSkRows + cit) * ldd + (m0 >> 4) / cl * 16), static_cast<uint32_t>(d));
                        uint32_t r[16];
                        tmem_ld16(tbase + m0, r);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            st_shared_cluster_v4(dst + static_cast<uint32_t>(i) * 4u, r[i], r[i + 1], r[i + 2], r[i + 3]);
                    }
                    for (int d = 0; d < cl; ++d)  // release: this thread's stores
                        if (d != static_cast<int>(crank)) mbar_arrive_cluster(mapa(smem_u32(&red_bar[0]), static_cast<uint32_t>(d)));
                    mbar_wait_acq_cluster(&red_bar[0], 0);  // every slice of my chunks has landed
                    // 3. My chunks, K-segments summed in segment order (mine from TMEM): the
                    //    same additions in the same order as the leader-only reduction.
                    for (int m0 = static_cast<int>(crank) * 16; m0 < mv; m0 += 16 * cl) {
                        uint32_t r[16];
                        tmem_ld16(tbase + m0, r);
                        tmem_ld_wait();
                        float v[16];
                        for (int s2 = 0; s2 < cl; ++s2) {
                            if (s2 == static_cast<int>(crank)) {
#pragma unroll
                                for (int i = 0; i < 16; ++i) v[i] = s2 == 0 ? __uint_as_float(r[i]) : v[i] + __uint_as_float(r[i]);
                            } else {
                                const int sl = s2 < static_cast<int>(crank) ? s2 : s2 - 1;
                                const float4* src = reinterpret_cast<const float4*>(sRed + (sl * kSkRows + cit) * ldd + (m0 >> 4) / cl * 16);
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const float4 w = src[i];
                                    if (s2 == 0) {
                                        v[4 * i] = w.x;
                                        v[4 * i + 1] = w.y;
                                        v[4 * i + 2] = w.z;
                                        v[4 * i + 3] = w.w;
                                    } else {
                                        v[4 * i] += w.x;
                                        v[4 * i + 1] += w.y;
                                        v[4 * i + 2] += w.z;
                                        v[4 * i + 3] += w.w;
                                    }
                                }
                            }
                        }
                        sk_store<MODE, PB, ACT>(p, l, col, m0, mv, v);
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[as]);
                    if (et == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 5, static_cast<uint32_t>(tt));
                } else if (crank != 0) {
                    // Buffer mode: the leader has read this slot's previous tile (the first
                    // wait passes). Ring mode: the leader's own MMAs are done, so its stage
                    // ring is free to receive.
                    mbar_wait(&red_bar[1], ring ? ephase : (ephase ^ 1u));
                    ephase ^= 1u;
                    const uint32_t dst = mapa(smem_u32(sRed + ((crank - 1) * kSkRows + cit) * ldr), 0);
                    for (int m0 = 0; m0 < mv; m0 += 16) {
                        uint32_t r[16];
                        tmem_ld16(tbase + m0, r);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            st_shared_cluster_v4(dst + static_cast<uint32_t>(m0 + i) * 4u, r[i], r[i + 1], r[i + 2], r[i + 3]);
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[as]);
                    mbar_arrive_cluster(mapa(smem_u32(&red_bar[0]), 0));  // release: this thread's stores
                } else {
                    if (ring && et >= 1 && et < cl)  // my MMAs retired: the ring may take the slots
                        mbar_arrive_cluster(mapa(smem_u32(&red_bar[1]), static_cast<uint32_t>(et)));
                    mbar_wait_acq_cluster(&red_bar[0], fphase);
                    fphase ^= 1u;
                    for (int m0 = 0; m0 < mv; m0 += 16) {
                        uint32_t r[16];
                        tmem_ld16(tbase + m0, r);
                        tmem_ld_wait();
                        float v[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
                        for (int s2 = 1; s2 < cl; ++s2) {
                            const float4* src = reinterpret_cast<const float4*>(sRed + ((s2 - 1) * kSkRows + cit) * ldr + m0);
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float4 w = src[i];
                                v[4 * i] += w.x;
                                v[4 * i + 1] += w.y;
                                v[4 * i + 2] += w.z;
                                v[4 * i + 3] += w.w;
                            }
                        }
                        sk_store<MODE, PB, ACT>(p, l, col, m0, mv, v);
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[as]);
                    named_bar_sync(1, 128);  // every leader thread has read the slots
                    if (!ring && et >= 1 && et < cl)
                        mbar_arrive_cluster(mapa(smem_u32(&red_bar[1]), static_cast<uint32_t>(et)));
                    if (et == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 5, static_cast<uint32_t>(tt));
                    if (MODE == kModeRSUnits) sk_rs_finish<PB>(p, l, j, mv, et);
                }
                if (++as == 2) {
                    as = 0;
                    aphase ^= 1u;
                }
            }
        }
        SkIter it{r0, r1, kbn};
        if (cl > 1) it.end = it.cur;  // (the cluster path above did the work)
        while (it.next(tt, kb0, kb1)) {
            const int l = tt / p.sk_nt, j = tt % p.sk_nt;
            const int col = j * kSkRows + cit;
            const long long tfirst = static_cast<long long>(tt) * kbn;
            const int c_first = sk_cta_of(p, tfirst);
            const int nseg = sk_cta_of(p, tfirst + kbn - 1) - c_first + 1;
            mbar_wait(&tfull[as], aphase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(as * p.sk_acc_cols);
            float* mine = nseg > 1 ? sk_slot(p, blockIdx.x, tt) : nullptr;
            for (int m0 = 0; m0 < mv; m0 += 16) {
                uint32_t r[16];
                tmem_ld16(tbase + m0, r);
                tmem_ld_wait();
                if (nseg == 1) {
                    float v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
                    sk_store<MODE, PB, ACT>(p, l, col, m0, mv, v);
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (m0 + i < mv) mine[(m0 + i) * kSkRows + cit] = __uint_as_float(r[i]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[as]);
            if (++as == 2) {
                as = 0;
                aphase ^= 1u;
            }
            if (et == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 3, static_cast<uint32_t>(tt));
            bool done = nseg == 1;
            if (!done) {
                // Arrival (acq_rel, after the CTA barrier: every thread's parked
                // stores are released; the last arrival acquires the others').
                named_bar_sync(1, 128);
                if (et == 0) red_slot[3] = static_cast<int>(tail_arrive(p.sk_ctr + tt, p.tail_seq));
                named_bar_sync(1, 128);
                done = red_slot[3] == nseg;
                if (done) {
                    if (et == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 4, static_cast<uint32_t>(tt));
                    const float* slot[kSkMaxSegs];
#pragma unroll
                    for (int s2 = 0; s2 < kSkMaxSegs; ++s2) slot[s2] = s2 < nseg ? sk_slot(p, c_first + s2, tt) : nullptr;
                    // float4 groups of the [mv x 128] tile, two per thread in flight
                    // with every segment's load (one L2 round trip per two groups).
                    const int E4 = mv * (kSkRows / 4);
                    for (int fb = et; fb < E4; fb += 128 * 2) {
                        float4 w[2][kSkMaxSegs];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int f = fb + u * 128;
#pragma unroll
                            for (int s2 = 0; s2 < kSkMaxSegs; ++s2)
                                if (s2 < nseg && f < E4) w[u][s2] = ld_cg_f4(slot[s2] + 4 * f);
                        }
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int f = fb + u * 128;
                            if (f >= E4) break;
                            float v[4] = {w[u][0].x, w[u][0].y, w[u][0].z, w[u][0].w};
#pragma unroll
                            for (int s2 = 1; s2 < kSkMaxSegs; ++s2)
                                if (s2 < nseg) {
                                    v[0] += w[u][s2].x;
                                    v[1] += w[u][s2].y;
                                    v[2] += w[u][s2].z;
                                    v[3] += w[u][s2].w;
                                }
                            const int m = f / (kSkRows / 4), c2 = j * kSkRows + (f % (kSkRows / 4)) * 4;
                            if (c2 >= p.n) continue;
                            if (MODE == kModeRSUnits) {
                                const int o = m / p.rpr;
                                long long pl;
                                float* const dst = rs_plane_base(p, o, p.global_rank[l], pl);
                                const long long se = static_cast<long long>(p.epoch & 1u) * p.stage_parity + pl +
                                                     static_cast<long long>(m - o * p.rpr) * p.ld_stage + c2;
                                st_part4<PB>(dst, se, make_float4(v[0], v[1], v[2], v[3]));
                            } else {
                                if (ACT) {
#pragma unroll
                                    for (int i = 0; i < 4; ++i) v[i] = act_fwd(p.act, v[i]);
                                }
                                store_row<4>(p.c[l], static_cast<long long>(m) * p.ldc_l[l] + c2, c2, p.n, p.out_f32, v);
                            }
                        }
                    }
                    if (et == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 5, static_cast<uint32_t>(tt));
                }
            }
            if (done && MODE == kModeRSUnits) sk_rs_finish<PB>(p, l, j, mv, et);
        }
        if (et == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 7, 0);  // epilogue done (profiling)
    }
    if (threadIdx.x % 32 == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 24 + warp, 0);  // warp at the exit barrier (profiling)
    __syncthreads();
    if (cl > 1) cluster_sync();  // no CTA exits while a peer may still arrive on its barriers
    if (warp == 0 && lane == 0) trace_event(p, 0, kEvLaunch, p.global_rank[0], blockIdx.x, 1, 0);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, tmem_cols);
    }
}

// Serial reduction of the rank partial planes in source order (reference
// run_nonoverlap RS branch, engine.cpp:595-602, and the WriteAlltoAll reduce
// agent, engine.cpp:335-339): C[i, j] = sum_{s=0..tp-1} P_s[owner*rpr + i, j].
__global__ void rs_reduce_kernel(RsReduceParams p) {
    const long long total = static_cast<long long>(p.rows) * p.n;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx / p.n), j = static_cast<int>(idx % p.n);
        const long long src = (static_cast<long long>(p.src_row0) + i) * p.ld_src + j;
        const long long dst = (static_cast<long long>(p.dst_row0) + i) * p.ldc + j;
        float acc = 0.0f;
        for (int s = 0; s < p.tp; ++s) acc += __ldcg(p.partials[s] + src);
        if (p.out_f32) static_cast<float*>(p.c)[dst] = acc;
        else static_cast<__nv_bfloat16*>(p.c)[dst] = __float2bfloat16_rn(acc);
    }
}

__global__ void zero_ranges_kernel(ZeroParams p) {
    char* h = p.heap[blockIdx.x];
    for (int r = 0; r < p.nranges; ++r) {
        uint32_t* w = reinterpret_cast<uint32_t*>(h + p.off[r]);
        for (uint32_t i = threadIdx.x; i < p.bytes[r] / 4; i += blockDim.x) w[i] = 0u;
    }
}

__global__ void rank_barrier_kernel(BarrierParams p) {
    if (threadIdx.x != 0) return;
    const uint32_t g = atomicAdd(p.gen, 1u) + 1u;
    for (int q = 0; q < p.tp; ++q)
        if (q != p.me) red_release_sys_add(p.peer_arr[q], 1u);
    const uint32_t target = g * static_cast<uint32_t>(p.tp - 1);
    const uint64_t t0 = globaltimer();
    uint32_t ns = 32;
    while (static_cast<int32_t>(ld_acquire_sys(p.arr) - target) < 0) {
        if (globaltimer() - t0 > p.timeout_ns) {
            if (atomicCAS(p.err, 0u, kErrBarrierTimeout) == 0u) {
                p.err[1] = g;
                p.err[2] = ld_acquire_sys(p.arr);
                p.err[3] = target;
                p.err[kCtrlErrEpoch / 4] = p.epoch;
                p.err[kCtrlErrEpoch / 4 + 1] = static_cast<uint32_t>(p.me) + 1u;
                if (p.err_host) {
                    volatile uint32_t* hh = p.err_host + 8 * p.me;
                    hh[1] = g;
                    hh[3] = target;
                    hh[5] = static_cast<uint32_t>(p.me) + 1u;
                    __threadfence_system();
                    hh[0] = kErrBarrierTimeout;
                }
            }
            return;
        }
        __nanosleep(ns);
        if (ns < 1024) ns <<= 1;
    }
}

cudaError_t launch_rank_barrier(const BarrierParams& p, cudaStream_t stream) {
    rank_barrier_kernel<<<1, 32, 0, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_zero_ranges(const ZeroParams& p, int nheaps, cudaStream_t stream) {
    zero_ranges_kernel<<<nheaps, 512, 0, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_rs_reduce(const RsReduceParams& p, int grid, cudaStream_t stream) {
    rs_reduce_kernel<<<grid, 256, 0, stream>>>(p);
    return cudaGetLastError();
}

int gemm_tile_rows(int cg) { return kBM * cg; }

// Function attributes belong to each device's context: the dynamic shared
// memory opt-in is set once per (kernel variant, device), tracked in a bitmask
// that concurrent host threads update atomically (setting it twice is harmless).
template <int MODE, int CG, int PB = 0, int EPI = 0>
static cudaError_t launch_one(const GemmParams& p, int grid, cudaStream_t stream) {
    static std::atomic<uint64_t> configured{0};
    auto fn = flux_gemm_kernel<MODE, CG, PB, EPI>;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
    if (bit == 0 || !(configured.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<CG, MODE>::kSmem);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Geo<CG, MODE>::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, p);
}

int stream_smem_bytes(int mode, int mp, int stages, int cluster) {
    return 1024 + stages * (kSkWBytes + mp * kBK * 2) + (mode == kModeAG ? 2 * kPieceBytes : 0) + kSkBarBytes +
           (cluster > 1 ? (cluster - 1) * kSkRows * (mp + 4) * 4 : 0);
}

template <int MODE, int PB = 0, int ACT = 0>
static cudaError_t stream_config(const GemmParams& p, int grid, int smem, cudaStream_t stream,
                                 cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attr) {
    static std::atomic<uint64_t> configured{0};
    auto fn = flux_stream_kernel<MODE, PB, ACT>;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
    if (bit == 0 || !(configured.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSkSmemMax);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    cfg = cudaLaunchConfig_t{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.sk_cluster > 1 ? p.sk_cluster : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaSuccess;
}

template <int MODE, int PB = 0, int ACT = 0>
static cudaError_t launch_stream_one(const GemmParams& p, int grid, int smem, cudaStream_t stream) {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[1];
    cudaError_t e = stream_config<MODE, PB, ACT>(p, grid, smem, stream, cfg, attr);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, flux_stream_kernel<MODE, PB, ACT>, p);
}

template <int MODE, int PB = 0, int ACT = 0>
static int max_clusters_one(const GemmParams& p, int smem) {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[1];
    if (stream_config<MODE, PB, ACT>(p, p.sk_cluster, smem, nullptr, cfg, attr) != cudaSuccess) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, flux_stream_kernel<MODE, PB, ACT>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Clusters of p.sk_cluster CTAs (smem bytes each) that can be resident at once.
int stream_max_clusters(int mode, const GemmParams& p, int cluster, int smem) {
    GemmParams q = p;
    q.sk_cluster = cluster;
    switch (mode) {
        case kModePlain: return p.act ? max_clusters_one<kModePlain, 0, 1>(q, smem) : max_clusters_one<kModePlain>(q, smem);
        case kModeAG: return p.act ? max_clusters_one<kModeAG, 0, 1>(q, smem) : max_clusters_one<kModeAG>(q, smem);
        case kModeRSUnits:
            return p.part_bf16 ? max_clusters_one<kModeRSUnits, 1>(q, smem) : max_clusters_one<kModeRSUnits>(q, smem);
    }
    return 0;
}

cudaError_t launch_stream(int mode, const GemmParams& p, int grid, int smem, cudaStream_t stream) {
    if (smem > kSkSmemMax || p.sk_stages < 2 || p.sk_stages > kSkMaxStages) return cudaErrorInvalidValue;
    switch (mode) {
        case kModePlain:
            return p.act ? launch_stream_one<kModePlain, 0, 1>(p, grid, smem, stream)
                         : launch_stream_one<kModePlain>(p, grid, smem, stream);
        case kModeAG:
            return p.act ? launch_stream_one<kModeAG, 0, 1>(p, grid, smem, stream)
                         : launch_stream_one<kModeAG>(p, grid, smem, stream);
        case kModeRSUnits:
            return p.part_bf16 ? launch_stream_one<kModeRSUnits, 1>(p, grid, smem, stream)
                               : launch_stream_one<kModeRSUnits>(p, grid, smem, stream);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_gemm(int mode, int cg, const GemmParams& p, int grid, cudaStream_t stream) {
    const bool epi = p.act || p.act_grad || p.aux_save;
    if (cg == 2) {
        grid &= ~1;
        if (grid < 2) grid = 2;
        switch (mode) {
            case kModePlain:
                return epi ? launch_one<kModePlain, 2, 0, 1>(p, grid, stream) : launch_one<kModePlain, 2>(p, grid, stream);
            case kModeAG:
                return epi ? launch_one<kModeAG, 2, 0, 1>(p, grid, stream) : launch_one<kModeAG, 2>(p, grid, stream);
            case kModeRS:
                return p.part_bf16 ? launch_one<kModeRS, 2, 1>(p, grid, stream) : launch_one<kModeRS, 2>(p, grid, stream);
            case kModeRSUnits:
                return p.part_bf16 ? launch_one<kModeRSUnits, 2, 1>(p, grid, stream)
                                   : launch_one<kModeRSUnits, 2>(p, grid, stream);
        }
    } else {
        switch (mode) {
            case kModePlain:
                return epi ? launch_one<kModePlain, 1, 0, 1>(p, grid, stream) : launch_one<kModePlain, 1>(p, grid, stream);
            case kModeAG:
                return epi ? launch_one<kModeAG, 1, 0, 1>(p, grid, stream) : launch_one<kModeAG, 1>(p, grid, stream);
            case kModeRS:
                return p.part_bf16 ? launch_one<kModeRS, 1, 1>(p, grid, stream) : launch_one<kModeRS, 1>(p, grid, stream);
            case kModeRSUnits:
                return p.part_bf16 ? launch_one<kModeRSUnits, 1, 1>(p, grid, stream)
                                   : launch_one<kModeRSUnits, 1>(p, grid, stream);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace fluxb200
