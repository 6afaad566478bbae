// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// extern "C" driver around the REFERENCE implementation itself, compiled from
// the unmodified sources under /root/reference/proj/core/src by oracle/Makefile
// into oracle/_ref/libref.so (git-ignored). Used (1) to pin the C restatement
// in oracle/flux_oracle.c bitwise, (2) to generate golden fixtures, and (3) as
// bench.py's CPU baseline ("reference" kind): the reference's own fused engine
// timed on the host cores.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "overlap/engine.hpp"
#include "overlap/oracle.hpp"
#include "overlap/workspace.hpp"

using namespace overlap;

namespace {

ProblemSpec spec(int pattern, int m, int n, int k, int tp) {
    return ProblemSpec{m, n, k, tp, pattern == 0 ? Pattern::AllGatherGemm : Pattern::GemmReduceScatter};
}

// make_random, optionally rounding every input to bf16 with the caller's rounder.
ShardedWorkspace workspace(const ProblemSpec& p, uint64_t seed, double (*round_fn)(double)) {
    ShardedWorkspace ws = ShardedWorkspace::make_random(p, seed);
    if (round_fn)
        for (int r = 0; r < p.tp; ++r) {
            for (double& v : ws.rank(r).a_shard.data()) v = round_fn(v);
            for (double& v : ws.rank(r).b_shard.data()) v = round_fn(v);
        }
    return ws;
}

void concat(const std::vector<Matrix>& outs, double* dst) {
    size_t off = 0;
    for (const Matrix& m : outs) {
        std::memcpy(dst + off, m.data().data(), m.data().size() * sizeof(double));
        off += m.data().size();
    }
}

}  // namespace

extern "C" {

// dense_oracle (oracle.cpp:28-62); outputs of all ranks concatenated.
int ref_dense_oracle(int pattern, int m, int n, int k, int tp, uint64_t seed, double (*round_fn)(double),
                     double* out) {
    try {
        ProblemSpec p = spec(pattern, m, n, k, tp);
        ShardedWorkspace ws = workspace(p, seed, round_fn);
        concat(dense_oracle(p, ws), out);
        return 0;
    } catch (...) {
        return 1;
    }
}

// The reference's fused engine / baselines. which: 0 fused AG, 1 fused RS,
// 2 run_nonoverlap. Returns seconds spent inside the engine call, or < 0 on
// error. Budgets are raised so long CPU GEMMs do not trip DeadlockError.
double ref_run(int which, int pattern, int m, int n, int k, int tp, uint64_t seed, double (*round_fn)(double), int tm,
               int tn, int rpct, int transfer, int write_mode, int swizzle_on, int workers, double* out) {
    try {
        ProblemSpec p = spec(pattern, m, n, k, tp);
        ShardedWorkspace ws = workspace(p, seed, round_fn);
        EngineOptions o;
        o.workers_per_rank = workers;
        o.poll_budget = std::numeric_limits<long long>::max() / 2;
        o.wall_budget_s = 1e6;
        std::vector<Matrix> outs;
        const auto t0 = std::chrono::steady_clock::now();
        if (which == 0) {
            const TransferMode tmode = transfer == 0 ? TransferMode::Pull : TransferMode::Push;
            auto comm = make_comm_specs(p, Topology{}, rpct, tmode);
            outs = run_fused_allgather_gemm(p, ws, {tm, tn}, comm, tmode, swizzle_on != 0, o).outputs;
        } else if (which == 1) {
            outs = run_fused_gemm_reducescatter(p, ws, {tm, tn},
                                                write_mode == 0 ? WriteMode::WriteAlltoAll : WriteMode::FusedReduce,
                                                swizzle_on != 0, o)
                       .outputs;
        } else {
            outs = run_nonoverlap(p, ws, {tm, tn});
        }
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (out) concat(outs, out);
        return secs;
    } catch (...) {
        return -1.0;
    }
}

// tile_order (swizzle.cpp:75-80) of SwizzlePolicy{kind, rank, tp, shift, arrival}.
int ref_tile_order(int pattern, int m, int n, int k, int tp, int tm, int tn, int kind, int rank, int shift,
                   const int* arrival, int n_arrival, int* rows, int* cols) {
    try {
        ProblemSpec p = spec(pattern, m, n, k, tp);
        GridDims g = grid_for(p, {tm, tn});
        SwizzlePolicy pol;
        pol.kind = kind == 0 ? SwizzleKind::Naive : kind == 1 ? SwizzleKind::RankShifted : SwizzleKind::ArrivalAligned;
        pol.rank = rank;
        pol.tp = tp;
        pol.shift_offset = shift;
        for (int i = 0; i < n_arrival; ++i) pol.arrival_blocks.push_back(arrival[i]);
        std::vector<TileCoord> o = tile_order(pol, g);
        for (size_t i = 0; i < o.size(); ++i) {
            rows[i] = o[i].row;
            cols[i] = o[i].col;
        }
        return static_cast<int>(o.size());
    } catch (...) {
        return -1;
    }
}

// make_comm_specs(problem, Topology{}, rpct, mode)[rank].order (engine.cpp:77-99).
int ref_comm_spec(int pattern, int m, int n, int k, int tp, int rank, int rpct, int transfer, int* peer,
                  int* row_begin, int* nrows, int max) {
    try {
        ProblemSpec p = spec(pattern, m, n, k, tp);
        auto specs = make_comm_specs(p, Topology{}, rpct, transfer == 0 ? TransferMode::Pull : TransferMode::Push);
        const auto& o = specs[rank].order;
        for (size_t i = 0; i < o.size() && static_cast<int>(i) < max; ++i) {
            peer[i] = o[i].peer;
            row_begin[i] = o[i].row_begin;
            nrows[i] = o[i].rows;
        }
        return static_cast<int>(o.size());
    } catch (...) {
        return -1;
    }
}

}  // extern "C"
