// Reference call sites (test_golden.cpp, test_engine.cpp, test_swizzle.cpp,
// acceptance.cpp) compiled unchanged against the B200 drop-in header and run
// on the GPU in tolerance mode. Prints one PASS/FAIL line per check; exit 1 on
// any failure. `--host-only` runs only the checks that need no GPU.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "flux/overlap.hpp"

using namespace overlap;

static int failures = 0;
static void check(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

// fp64 oracle on bf16-rounded inputs (what the tensor cores consume).
// Round-to-nearest-even of the double itself (exact rational comparison via
// frexp; no double rounding through float).
static double bf16(double x) {
    if (x == 0.0) return x;
    int e;
    const double mant = std::frexp(std::fabs(x), &e);  // [0.5, 1)
    const double scaled = mant * 256.0;                // 8 significant bits
    double lo = std::floor(scaled);
    const double frac = scaled - lo;
    if (frac > 0.5 || (frac == 0.5 && std::fmod(lo, 2.0) == 1.0)) lo += 1.0;
    return std::copysign(std::ldexp(lo / 256.0, e), x);
}
static std::vector<Matrix> oracle(const ProblemSpec& p, const ShardedWorkspace& ws) {
    std::vector<Matrix> out;
    const int rpr = p.rows_per_rank();
    if (p.pattern == Pattern::AllGatherGemm) {
        for (int r = 0; r < p.tp; ++r) {
            Matrix c(p.m, p.local_cols());
            for (int i = 0; i < p.m; ++i)
                for (int j = 0; j < p.local_cols(); ++j) {
                    double acc = 0;
                    for (int x = 0; x < p.k; ++x)
                        acc += bf16(ws.rank(i / rpr).a_shard(i % rpr, x)) * bf16(ws.rank(r).b_shard(x, j));
                    c(i, j) = acc;
                }
            out.push_back(c);
        }
    } else {
        for (int d = 0; d < p.tp; ++d) {
            Matrix c(rpr, p.n);
            for (int i = 0; i < rpr; ++i)
                for (int j = 0; j < p.n; ++j) {
                    double sum = 0;
                    for (int s = 0; s < p.tp; ++s) {
                        double acc = 0;
                        for (int x = 0; x < p.local_k(); ++x)
                            acc += bf16(ws.rank(s).a_shard(d * rpr + i, x)) * bf16(ws.rank(s).b_shard(x, j));
                        sum += acc;
                    }
                    c(i, j) = sum;
                }
            out.push_back(c);
        }
    }
    return out;
}
static double worst(const std::vector<Matrix>& a, const std::vector<Matrix>& b) {
    double w = 0;
    for (size_t r = 0; r < a.size(); ++r) w = std::max(w, max_rel_error(a[r], b[r]));
    return w;
}

template <class E, class F>
static bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void host_checks() {
    // test_swizzle.cpp:44-56
    ProblemSpec rs{4, 4, 4, 4, Pattern::GemmReduceScatter};
    auto o = tile_order(SwizzlePolicy{SwizzleKind::RankShifted, 1, 4, 1, {}}, grid_for(rs, {1, 4}));
    check(o[0].row == 2 && o[1].row == 3 && o[2].row == 0 && o[3].row == 1, "RankShifted tp=4 r=1 visits 2,3,0,1");
    ProblemSpec ag{8, 8, 8, 8, Pattern::AllGatherGemm};
    auto a = tile_order(SwizzlePolicy{SwizzleKind::ArrivalAligned, 5, 8, 1, {}}, grid_for(ag, {1, 1}));
    check(a[0].row == 5 && a[3].row == 0 && a[7].row == 4, "ArrivalAligned tp=8 r=5 visits 5,6,7,0..4");
    auto ring = comm_order(Topology{}, 5, 8, 4, 4);
    check(ring.size() == 7 && ring[0].peer == 6 && ring[2].peer == 0, "NVLinkRing order of rank 5 is 6,7,0..4");
    check(throws<ConfigError>([] { validate_tiling({16, 16, 16, 4, Pattern::AllGatherGemm}, {3, 2}); }),
          "non-dividing tile raises ConfigError");
    check(throws<ConfigError>([] { ProblemSpec{10, 16, 16, 4, Pattern::AllGatherGemm}.validate(); }),
          "m % tp != 0 raises ConfigError");
    auto specs = make_comm_specs(ag, Topology{}, 1, TransferMode::Push);
    check(specs.size() == 8 && specs[2].order.size() == 7, "push comm specs carry the local tile to 7 peers");
    check(throws<BoundsError>([] { map_tile({}, 99, GridDims{2, 2, 1}); }), "map_tile out of range raises BoundsError");
    // test_engine.cpp:141-156: medium-grained schedule shape
    {
        ProblemSpec p{8, 4, 4, 2, Pattern::GemmReduceScatter};
        auto steps = medium_schedule(p, 2);
        bool shape = steps.size() == 12;
        for (int r = 0; r < 2 && shape; ++r) {
            const int base = r * 6;
            shape = steps[base + 0].kind == MediumStep::Kind::ChunkGemm &&
                    steps[base + 2].kind == MediumStep::Kind::ChunkAdd &&
                    steps[base + 3].kind == MediumStep::Kind::ChunkGemm &&
                    steps[base + 5].kind == MediumStep::Kind::ChunkAdd && steps[base + 3].deps.size() == 1 &&
                    steps[base + 3].deps[0] == base + 2;
        }
        check(shape, "medium schedule tp=2 partitions=2 alternates chunk gemm and add");
        ProblemSpec q{16, 8, 8, 4, Pattern::GemmReduceScatter};
        check(throws<ConfigError>([&] { medium_schedule(q, 3); }), "invalid partition count raises ConfigError");
        ProblemSpec ag{16, 8, 8, 4, Pattern::AllGatherGemm};
        auto a = medium_schedule(ag, 4);
        int xfers = 0;
        for (const MediumStep& s : a) xfers += s.rank == 0 && s.kind == MediumStep::Kind::ChunkTransfer;
        check(a.size() == 4 * 7 && xfers == 3, "medium schedule AG: 3 remote chunk transfers + 4 chunk GEMMs per rank");
    }
}

static void device_checks() {
    // test_golden.cpp: the frozen 16x16x16 tp=4 seed-42 workspace, every strategy.
    for (Pattern pat : {Pattern::AllGatherGemm, Pattern::GemmReduceScatter}) {
        ProblemSpec p{16, 16, 16, 4, pat};
        ShardedWorkspace ws = ShardedWorkspace::make_random(p, 42);
        const auto want = oracle(p, ws);
        if (pat == Pattern::GemmReduceScatter) {
            auto res = run_fused_gemm_reducescatter(p, ws, {2, 2}, WriteMode::FusedReduce, true);
            check(worst(res.outputs, want) <= 1e-4, "fused reduce-scatter golden config within 1e-4");
        } else {
            auto comm = make_comm_specs(p, Topology{}, p.rows_per_rank(), TransferMode::Pull);
            auto res = run_fused_allgather_gemm(p, ws, {2, 2}, comm, TransferMode::Pull, true);
            check(worst(res.outputs, want) <= 1e-4, "fused all-gather golden config within 1e-4");
        }
        check(worst(run_nonoverlap(p, ws, {2, 2}), want) <= 1e-4, "nonoverlap golden config within 1e-4");
        // test_golden.cpp:70 / acceptance.cpp:102: the medium-grained baseline
        auto med = run_medium_grained(p, ws, {2, 2}, 8);
        int gemms = 0;
        for (const MediumStep& s : med.trace) gemms += s.rank == 0 && s.kind == MediumStep::Kind::ChunkGemm;
        check(gemms == 8 && worst(med.outputs, want) <= 1e-4, "medium-grained (8 chunks) golden config within 1e-4");
    }
    // test_engine.cpp:63-74 push == pull bitwise
    ProblemSpec p{64, 32, 48, 4, Pattern::AllGatherGemm};
    ShardedWorkspace ws = ShardedWorkspace::make_random(p, 42);
    auto pull = run_fused_allgather_gemm(p, ws, {4, 4}, make_comm_specs(p, Topology{}, 4, TransferMode::Pull),
                                         TransferMode::Pull, true);
    auto push = run_fused_allgather_gemm(p, ws, {4, 4}, make_comm_specs(p, Topology{}, 4, TransferMode::Push),
                                         TransferMode::Push, true);
    bool same = true;
    for (int r = 0; r < p.tp; ++r) same = same && bitwise_equal(pull.outputs[r], push.outputs[r]);
    check(same, "push and pull transfers produce identical outputs");
    // test_engine.cpp:190-213 on EngineResult::log (the device event trace): every
    // compute_start follows the signal_set of the group it consumed.
    {
        bool causal = !pull.log.empty();
        int starts = 0;
        for (const CausalityEvent& e : pull.log) {
            if (e.kind != "compute_start") continue;
            ++starts;
            bool seen = false;
            for (const CausalityEvent& f : pull.log)
                seen = seen || (f.kind == "signal_set" && f.rank == e.rank && f.target == e.target &&
                                f.logical_ts < e.logical_ts);
            causal = causal && seen;
        }
        check(causal && starts > 0, "EngineResult::log: compute_start after its group's signal_set");
    }
    check(worst(pull.outputs, oracle(p, ws)) <= 1e-4, "all-gather 64x32x48 tp=4 within 1e-4");
    // acceptance.cpp criterion 1 style: random shapes, every tp
    Rng rng(42);
    double w = 0;
    for (int i = 0; i < 24; ++i) {
        const int tps[] = {1, 2, 4, 8};
        const int tp = tps[rng.next_below(4)];
        const Pattern pat = i % 2 ? Pattern::GemmReduceScatter : Pattern::AllGatherGemm;
        ProblemSpec q{8 * tp * (1 + int(rng.next_below(3))), 0, 0, tp, pat};
        q.n = pat == Pattern::AllGatherGemm ? 8 * tp * (1 + int(rng.next_below(3))) : 8 * (1 + int(rng.next_below(5)));
        q.k = pat == Pattern::AllGatherGemm ? 8 * (1 + int(rng.next_below(4))) : 8 * tp * (1 + int(rng.next_below(3)));
        ShardedWorkspace s = ShardedWorkspace::make_random(q, 100 + i);
        std::vector<Matrix> got;
        if (pat == Pattern::AllGatherGemm)
            got = run_fused_allgather_gemm(q, s, {q.rows_per_rank(), q.local_cols()},
                                           make_comm_specs(q, Topology{}, q.rows_per_rank(), TransferMode::Pull),
                                           TransferMode::Pull, true)
                      .outputs;
        else
            got = run_fused_gemm_reducescatter(q, s, {q.rows_per_rank(), q.local_cols()}, WriteMode::WriteAlltoAll,
                                               true)
                      .outputs;
        w = std::max(w, worst(got, oracle(q, s)));
    }
    check(w <= 1e-4, "24 random cases, all tp, worst rel err " + std::to_string(w));
    // test_engine.cpp:102-115 on the device: the copy-engine transfer loop walks the
    // caller's comm order (here each rank's ring list reversed) and records, per
    // descriptor, device times with copy_done <= flag_set and copy tick < flag tick.
    {
        ProblemSpec q{64, 32, 48, 4, Pattern::AllGatherGemm};
        ShardedWorkspace s = ShardedWorkspace::make_random(q, 7);
        auto specs = make_comm_specs(q, Topology{}, 8, TransferMode::Pull);
        for (auto& sp : specs) std::reverse(sp.order.begin(), sp.order.end());
        std::vector<std::vector<TransferRecord>> traces;
        auto res = run_fused_allgather_gemm(q, s, {8, 8}, specs, TransferMode::Pull, true, EngineOptions{}, &traces);
        bool timed = traces.size() == 4, ordered = true;
        for (int r = 0; r < 4 && timed; ++r) {
            timed = timed && traces[r].size() == specs[r].order.size();
            for (size_t i = 0; i < traces[r].size() && timed; ++i) {
                const TransferRecord& t = traces[r][i];
                timed = timed && t.copy_done_ns <= t.flag_set_ns && t.copy_logical_ts < t.flag_logical_ts;
                ordered = ordered && t.desc.row_begin == specs[r].order[i].row_begin && t.desc.peer == specs[r].order[i].peer;
            }
        }
        check(timed, "TransferRecords: copy_done_ns <= flag_set_ns, copy tick before flag tick, one per descriptor");
        check(ordered, "the transfer loop walks the caller's (non-ring) comm order");
        check(worst(res.outputs, oracle(q, s)) <= 1e-4, "all-gather on a caller comm order within 1e-4");
        auto bad = make_comm_specs(q, Topology{}, 8, TransferMode::Pull);
        bad[1].order[0] = bad[1].order[1];
        check(throws<ConfigError>([&] { run_fused_allgather_gemm(q, s, {8, 8}, bad, TransferMode::Pull, true); }),
              "comm order covering a tile twice raises ConfigError");
    }
    // test_engine.cpp:182-188 DirectoryError
    ShardedWorkspace d = ShardedWorkspace::make_random(p, 1);
    d.drop_directory_entry(1, 2);
    check(throws<DirectoryError>([&] {
              run_fused_allgather_gemm(p, d, {4, 4}, make_comm_specs(p, Topology{}, 4, TransferMode::Pull),
                                       TransferMode::Pull, true);
          }),
          "dropped directory entry raises DirectoryError");
}

int main(int argc, char** argv) {
    host_checks();
    if (!(argc > 1 && std::string(argv[1]) == "--host-only")) device_checks();
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
