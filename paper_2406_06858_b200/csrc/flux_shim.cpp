// C++ drop-in for the reference operator API (include/flux/overlap.hpp), on
// top of the C ABI (include/flux_b200.h). Host-side schedule logic comes from
// the ABI (one implementation); this file adapts types and errors and moves
// the reference's fp64 host matrices into / out of the symmetric heaps.
#include "flux/overlap.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>

#include "flux_b200.h"

namespace overlap {

namespace {

[[noreturn]] void raise(int rc) {
    const std::string msg = flux_last_error();
    switch (rc) {
        case FLUX_ERR_CONFIG: throw ConfigError(msg);
        case FLUX_ERR_SHAPE: throw ShapeError(msg);
        case FLUX_ERR_DIRECTORY: throw DirectoryError(msg);
        case FLUX_ERR_DEADLOCK: throw DeadlockError(msg);
        case FLUX_ERR_BOUNDS: throw BoundsError(msg);
        case FLUX_ERR_RUNTIME: throw std::runtime_error(msg);  // e.g. "flag 3 on rank 1 set twice"
        default: throw std::runtime_error("flux: " + msg);
    }
}
void ok(int rc) {
    if (rc != FLUX_OK) raise(rc);
}

flux_problem cprob(const ProblemSpec& p) {
    return flux_problem{p.m, p.n, p.k, p.tp, p.pattern == Pattern::AllGatherGemm ? FLUX_ALLGATHER_GEMM
                                                                               : FLUX_GEMM_REDUCESCATTER};
}

std::string dims(const Matrix& m) { return "[" + std::to_string(m.rows()) + "," + std::to_string(m.cols()) + "]"; }

// double -> bf16 bits, round to nearest even on the exact double value.
uint16_t to_bf16(double x) {
    if (std::isnan(x)) return 0x7FC0;
    const float f = static_cast<float>(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t base = u & 0xFFFF0000u, low = u & 0xFFFFu;
    uint32_t out = base;
    if (low > 0x8000u) {
        out = base + 0x10000u;
    } else if (low == 0x8000u) {  // float sits on a bf16 midpoint: decide on the double
        float lo, hi;
        const uint32_t up = base + 0x10000u;
        std::memcpy(&lo, &base, 4);
        std::memcpy(&hi, &up, 4);
        const double mid = 0.5 * (static_cast<double>(lo) + static_cast<double>(hi));
        if (std::fabs(x) > std::fabs(mid) || (std::fabs(x) == std::fabs(mid) && ((base >> 16) & 1u))) out = up;
    }
    return static_cast<uint16_t>(out >> 16);
}

double from_bf16(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

std::vector<int> pick_devices(int tp) {
    std::vector<int> devs;
    if (const char* env = std::getenv("FLUX_DEVICES")) {
        std::stringstream ss(env);
        std::string item;
        while (std::getline(ss, item, ',')) devs.push_back(std::atoi(item.c_str()));
        if (static_cast<int>(devs.size()) >= tp) {
            devs.resize(tp);
            return devs;
        }
        devs.clear();
    }
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    for (int r = 0; r < tp; ++r) devs.push_back(count >= tp ? r : 0);
    return devs;
}

// One communicator per (tp, devices), grown when a larger problem arrives.
struct Session {
    flux_comm* comm = nullptr;
    int tp = 0;
    std::vector<int> devices;
    size_t heap = 0;
};
std::mutex g_mu;
Session g_session;

flux_comm* session_for(const ProblemSpec& p) {
    const flux_problem cp = cprob(p);
    const size_t need = flux_required_heap_bytes(&cp);
    const std::vector<int> devs = pick_devices(p.tp);
    if (g_session.comm && g_session.tp == p.tp && g_session.devices == devs && g_session.heap >= need)
        return g_session.comm;
    if (g_session.comm) flux_comm_destroy(g_session.comm);
    g_session = Session{};
    flux_comm_opts o{std::max<size_t>(need, size_t(16) << 20)};
    flux_comm* c = nullptr;
    ok(flux_comm_create(p.tp, devs.data(), &o, &c));
    g_session = Session{c, p.tp, devs, o.heap_bytes};
    return c;
}

// Host fp64 matrix -> bf16 device buffer. transpose: reference B [k, cols] ->
// device K-major [cols, k].
void upload(flux_comm* c, int rank, int kind, const flux_problem& cp, const Matrix& m, bool transpose) {
    const int rows = transpose ? m.cols() : m.rows(), cols = transpose ? m.rows() : m.cols();
    std::vector<uint16_t> host(static_cast<size_t>(rows) * cols);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) host[size_t(i) * cols + j] = to_bf16(transpose ? m(j, i) : m(i, j));
    ok(flux_copy_in(c, rank, kind, &cp, host.data(), cols, nullptr));
    ok(flux_sync(c));
}

Matrix download_f32(flux_comm* c, int rank, int kind, const flux_problem& cp) {
    flux_buffer_desc d;
    ok(flux_buffer(c, rank, kind, &cp, &d));
    std::vector<float> host(static_cast<size_t>(d.rows) * d.cols);
    ok(flux_copy_out(c, rank, kind, &cp, host.data(), d.cols, nullptr));
    ok(flux_sync(c));
    Matrix m(d.rows, d.cols);
    for (size_t i = 0; i < host.size(); ++i) m.data()[i] = host[i];
    return m;
}

Matrix download_bf16(flux_comm* c, int rank, int kind, const flux_problem& cp) {
    flux_buffer_desc d;
    ok(flux_buffer(c, rank, kind, &cp, &d));
    std::vector<uint16_t> host(static_cast<size_t>(d.rows) * d.cols);
    ok(flux_copy_out(c, rank, kind, &cp, host.data(), d.cols, nullptr));
    ok(flux_sync(c));
    Matrix m(d.rows, d.cols);
    for (size_t i = 0; i < host.size(); ++i) m.data()[i] = from_bf16(host[i]);
    return m;
}

flux_opts copts(const EngineOptions& o) {
    flux_opts f;
    flux_default_opts(&f);
    f.workers_per_rank = o.workers_per_rank;
    f.deterministic_reduce = o.deterministic_reduce ? 1 : 0;
    f.poll_budget = o.poll_budget;
    f.wall_budget_s = o.wall_budget_s;
    f.interleave_seed = o.interleave_seed;
    f.shift_offset = o.shift_offset;
    f.out_dtype = FLUX_F32;  // fp64 host outputs: keep the fp32 accumulator
    return f;
}

void check_directory(const ShardedWorkspace& ws) {
    if (!ws.dropped().empty()) {
        const auto& d = ws.dropped().front();
        throw DirectoryError("missing peer buffer: rank " + std::to_string(d.first) +
                             " has no directory entry for peer " + std::to_string(d.second));
    }
}

void upload_inputs(flux_comm* c, const ProblemSpec& p, const ShardedWorkspace& ws) {
    const flux_problem cp = cprob(p);
    for (int r = 0; r < p.tp; ++r) {
        upload(c, r, FLUX_BUF_A_SHARD, cp, ws.rank(r).a_shard, false);
        upload(c, r, FLUX_BUF_B_SHARD, cp, ws.rank(r).b_shard, true);
    }
}

EngineResult collect(flux_comm* c, const ProblemSpec& p, ShardedWorkspace& ws) {
    const flux_problem cp = cprob(p);
    EngineResult res;
    for (int r = 0; r < p.tp; ++r) {
        ws.rank(r).c_out = download_f32(c, r, 5 /* C as fp32 */, cp);
        if (p.pattern == Pattern::AllGatherGemm) ws.rank(r).a_agg = download_bf16(c, r, FLUX_BUF_A_AGG, cp);
        res.outputs.push_back(ws.rank(r).c_out);
    }
    return res;
}

// EngineResult::log from the device event trace (CausalityLog schema,
// engine.hpp:37-63): every rank's records ordered by %globaltimer, logical
// timestamps 1..n in that order, wall_ns relative to the first event. The
// launch-latency records (kind 6) are not part of the reference schema.
std::vector<CausalityEvent> device_log(flux_comm* c, const ProblemSpec& p) {
    static const char* kKinds[] = {"", "compute_start", "signal_set", "tile_write", "reduce", "wait"};
    const flux_problem cp = cprob(p);
    std::vector<std::pair<uint64_t, CausalityEvent>> all;
    std::vector<uint64_t> buf(2u << 18);
    for (int r = 0; r < p.tp; ++r) {
        size_t n = 0;
        ok(flux_trace_read(c, r, &cp, buf.data(), buf.size() / 2, &n));
        for (size_t i = 0; i < n; ++i) {
            const uint64_t ts = buf[2 * i], w = buf[2 * i + 1];
            const unsigned kind = static_cast<unsigned>(w >> 60);
            if (kind == 0 || kind > 5) continue;
            CausalityEvent e;
            e.kind = kKinds[kind];
            e.rank = static_cast<int>((w >> 56) & 0xF);
            e.target = static_cast<int>((w >> 32) & 0xFFFFFF);
            e.tile_row = static_cast<int>((w >> 16) & 0xFFFF);
            e.tile_col = static_cast<int>(w & 0xFFFF);
            all.emplace_back(ts, e);
        }
    }
    std::stable_sort(all.begin(), all.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    std::vector<CausalityEvent> log;
    log.reserve(all.size());
    for (size_t i = 0; i < all.size(); ++i) {
        CausalityEvent e = all[i].second;
        e.logical_ts = i + 1;
        e.wall_ns = static_cast<int64_t>(all[i].first - all.front().first);
        log.push_back(e);
    }
    return log;
}

}  // namespace

// ---- matrix helpers ----------------------------------------------------------------
double max_rel_error(const Matrix& a, const Matrix& b) {
    if (!a.same_shape(b)) throw ShapeError("max_rel_error: shape mismatch " + dims(a) + " vs " + dims(b));
    double worst = 0.0;
    for (size_t i = 0; i < a.data().size(); ++i) {
        const double x = a.data()[i], y = b.data()[i];
        worst = std::max(worst, std::fabs(x - y) / std::max({1.0, std::fabs(x), std::fabs(y)}));
    }
    return worst;
}
bool approx_equal(const Matrix& a, const Matrix& b, double rel_tol) {
    return a.same_shape(b) && max_rel_error(a, b) <= rel_tol;
}
bool bitwise_equal(const Matrix& a, const Matrix& b) {
    return a.same_shape(b) && std::memcmp(a.data().data(), b.data().data(), a.data().size() * sizeof(double)) == 0;
}
uint64_t Rng::next_u64() {
    uint64_t z = (s_ += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
double Rng::next_uniform() { return static_cast<double>(next_u64() >> 11) * (2.0 / 9007199254740992.0) - 1.0; }
void fill_uniform(Matrix& m, Rng& rng) {
    for (double& v : m.data()) v = rng.next_uniform();
}

// ---- problem / tiling -----------------------------------------------------------------
std::string to_string(Pattern p) { return p == Pattern::AllGatherGemm ? "AllGatherGemm" : "GemmReduceScatter"; }
Pattern pattern_from_string(const std::string& s) {
    if (s == "AllGatherGemm") return Pattern::AllGatherGemm;
    if (s == "GemmReduceScatter") return Pattern::GemmReduceScatter;
    throw ConfigError("unknown pattern: '" + s + "' (expected AllGatherGemm or GemmReduceScatter)");
}
void ProblemSpec::validate() const {
    const flux_problem cp = cprob(*this);
    ok(flux_problem_validate(&cp, nullptr));
}
void validate_tiling(const ProblemSpec& p, const TileShape& t) {
    const flux_problem cp = cprob(p);
    const flux_tile ct{t.tm, t.tn};
    ok(flux_problem_validate(&cp, &ct));
}
GridDims grid_for(const ProblemSpec& p, const TileShape& t) {
    const flux_problem cp = cprob(p);
    const flux_tile ct{t.tm, t.tn};
    GridDims g;
    ok(flux_grid_for(&cp, &ct, &g.tile_rows, &g.tile_cols, &g.row_blocks));
    return g;
}
std::vector<TileCoord> tile_grid(const ProblemSpec& p, const TileShape& t) {
    const GridDims g = grid_for(p, t);
    std::vector<TileCoord> out;
    for (int r = 0; r < g.tile_rows; ++r)
        for (int c = 0; c < g.tile_cols; ++c) out.push_back({r, c});
    return out;
}

// ---- comm order / swizzle -----------------------------------------------------------------
std::vector<TransferDesc> comm_order(const Topology&, int rank, int tp, int rpr, int rpct, bool) {
    std::vector<int> peer(tp * std::max(1, rpr / std::max(1, rpct))), begin(peer.size()), rows(peer.size());
    int n = 0;
    ok(flux_comm_order(rank, tp, rpr, rpct, peer.data(), begin.data(), rows.data(), static_cast<int>(peer.size()), &n));
    std::vector<TransferDesc> out;
    for (int i = 0; i < n; ++i) out.push_back({peer[i], begin[i], rows[i], LinkClass::IntraNuma, -1, -1});
    return out;
}
std::vector<int> peer_order(const std::vector<TransferDesc>& order, int rank, int rpr) {
    std::vector<int> seq;
    for (const TransferDesc& d : order) {
        const int b = d.row_begin / rpr;
        if (b != rank && std::find(seq.begin(), seq.end(), b) == seq.end()) seq.push_back(b);
    }
    return seq;
}
SwizzlePolicy arrival_aligned_policy(int rank, int tp, const std::vector<TransferDesc>& order, int rpr) {
    SwizzlePolicy p{SwizzleKind::ArrivalAligned, rank, tp, 1, {rank}};
    for (int b : peer_order(order, rank, rpr)) p.arrival_blocks.push_back(b);
    return p;
}
TileCoord map_tile(const SwizzlePolicy& policy, int i, const GridDims& g) {
    static const int kKind[] = {FLUX_SWIZZLE_NAIVE, FLUX_SWIZZLE_RANK_SHIFTED, FLUX_SWIZZLE_ARRIVAL_ALIGNED};
    TileCoord t;
    ok(flux_map_tile(kKind[static_cast<int>(policy.kind)], policy.rank, policy.tp, policy.shift_offset,
                     policy.arrival_blocks.data(), static_cast<int>(policy.arrival_blocks.size()), g.tile_rows,
                     g.tile_cols, g.row_blocks, i, &t.row, &t.col));
    return t;
}
std::vector<TileCoord> tile_order(const SwizzlePolicy& policy, const GridDims& g) {
    std::vector<TileCoord> out;
    for (int i = 0; i < g.tiles(); ++i) out.push_back(map_tile(policy, i, g));
    return out;
}

// ---- workspace ------------------------------------------------------------------------------
ShardedWorkspace ShardedWorkspace::make_random(const ProblemSpec& p, uint64_t seed) {
    p.validate();
    ShardedWorkspace ws;
    ws.ranks_.resize(p.tp);
    for (int r = 0; r < p.tp; ++r) {
        RankBuffers& b = ws.ranks_[r];
        Rng rng(seed * 0x100000001b3ull + static_cast<uint64_t>(r) + 1);
        if (p.pattern == Pattern::AllGatherGemm) {
            b.a_shard = Matrix(p.rows_per_rank(), p.k);
            b.b_shard = Matrix(p.k, p.local_cols());
            b.a_agg = Matrix(p.m, p.k);
            b.c_out = Matrix(p.m, p.local_cols());
        } else {
            b.a_shard = Matrix(p.m, p.local_k());
            b.b_shard = Matrix(p.local_k(), p.n);
            b.c_out = Matrix(p.rows_per_rank(), p.n);
        }
        fill_uniform(b.a_shard, rng);
        fill_uniform(b.b_shard, rng);
    }
    return ws;
}
void ShardedWorkspace::validate(const ProblemSpec& p) const {
    p.validate();
    if (num_ranks() != p.tp)
        throw ShapeError("workspace has " + std::to_string(num_ranks()) + " ranks, problem tp=" + std::to_string(p.tp));
    auto want = [](const Matrix& m, int rows, int cols, const std::string& what) {
        if (m.rows() != rows || m.cols() != cols)
            throw ShapeError(what + " shape " + dims(m) + " expected [" + std::to_string(rows) + "," +
                             std::to_string(cols) + "]");
    };
    for (int r = 0; r < num_ranks(); ++r) {
        const std::string tag = "rank " + std::to_string(r) + " ";
        if (p.pattern == Pattern::AllGatherGemm) {
            want(ranks_[r].a_shard, p.rows_per_rank(), p.k, tag + "a_shard");
            want(ranks_[r].b_shard, p.k, p.local_cols(), tag + "b_shard");
            want(ranks_[r].a_agg, p.m, p.k, tag + "a_agg");
        } else {
            want(ranks_[r].a_shard, p.m, p.local_k(), tag + "a_shard");
            want(ranks_[r].b_shard, p.local_k(), p.n, tag + "b_shard");
        }
    }
}
RankBuffers& ShardedWorkspace::peer(int from, int to) {
    if (from < 0 || from >= num_ranks() || to < 0 || to >= num_ranks())
        throw DirectoryError("directory lookup out of range: rank " + std::to_string(from) + " -> peer " +
                             std::to_string(to));
    for (const auto& d : dropped_)
        if (d.first == from && d.second == to)
            throw DirectoryError("missing peer buffer: rank " + std::to_string(from) +
                                 " has no directory entry for peer " + std::to_string(to));
    return ranks_[to];
}
void ShardedWorkspace::drop_directory_entry(int from, int to) { dropped_.emplace_back(from, to); }
void ShardedWorkspace::clear_outputs() {
    for (RankBuffers& b : ranks_) {
        b.c_out.fill(0.0);
        if (!b.a_agg.empty()) b.a_agg.fill(0.0);
        b.staging.clear();
    }
}

// ---- engine ----------------------------------------------------------------------------------
std::string to_string(TransferMode m) { return m == TransferMode::Pull ? "Pull" : "Push"; }
TransferMode transfer_mode_from_string(const std::string& s) {
    if (s == "Pull") return TransferMode::Pull;
    if (s == "Push") return TransferMode::Push;
    throw ConfigError("unknown transfer mode: '" + s + "'");
}
std::string to_string(WriteMode m) { return m == WriteMode::WriteAlltoAll ? "WriteAlltoAll" : "FusedReduce"; }
WriteMode write_mode_from_string(const std::string& s) {
    if (s == "WriteAlltoAll") return WriteMode::WriteAlltoAll;
    if (s == "FusedReduce") return WriteMode::FusedReduce;
    throw ConfigError("unknown write mode: '" + s + "'");
}

void CommTileSpec::validate(const ProblemSpec& p, int rank, TransferMode mode) const {
    const flux_problem cp = cprob(p);
    std::vector<int> peer, begin, rows;
    for (const TransferDesc& d : order) {
        peer.push_back(d.peer);
        begin.push_back(d.row_begin);
        rows.push_back(d.rows);
    }
    ok(flux_validate_comm_spec(&cp, rank, rows_per_comm_tile, mode == TransferMode::Pull ? FLUX_PULL : FLUX_PUSH,
                               peer.data(), begin.data(), rows.data(), static_cast<int>(order.size())));
}

std::vector<CommTileSpec> make_comm_specs(const ProblemSpec& p, const Topology&, int rpct, TransferMode mode) {
    const flux_problem cp = cprob(p);
    std::vector<CommTileSpec> specs(p.tp);
    std::vector<int> peer(std::max(1, p.m)), begin(peer.size()), rows(peer.size());
    for (int r = 0; r < p.tp; ++r) {
        int n = 0;
        ok(flux_make_comm_spec(&cp, r, rpct, mode == TransferMode::Pull ? FLUX_PULL : FLUX_PUSH, peer.data(),
                               begin.data(), rows.data(), static_cast<int>(peer.size()), &n));
        specs[r].rows_per_comm_tile = rpct;
        for (int i = 0; i < n; ++i) specs[r].order.push_back({peer[i], begin[i], rows[i], LinkClass::IntraNuma, -1, -1});
    }
    return specs;
}

EngineResult run_fused_gemm_reducescatter(const ProblemSpec& p, ShardedWorkspace& ws, const TileShape& tile,
                                          WriteMode write_mode, bool swizzle_on, const EngineOptions& opts) {
    if (p.pattern != Pattern::GemmReduceScatter)
        throw ConfigError("run_fused_gemm_reducescatter requires GemmReduceScatter pattern");
    grid_for(p, tile);
    ws.validate(p);
    check_directory(ws);
    ws.clear_outputs();
    std::lock_guard<std::mutex> g(g_mu);
    flux_comm* c = session_for(p);
    upload_inputs(c, p, ws);
    const flux_problem cp = cprob(p);
    const flux_tile ct{tile.tm, tile.tn};
    flux_opts o = copts(opts);
    o.trace = 1;  // EngineResult::log
    ok(flux_gemm_rs(c, &cp, &ct, write_mode == WriteMode::WriteAlltoAll ? FLUX_WRITE_ALLTOALL : FLUX_FUSED_REDUCE,
                    swizzle_on ? 1 : 0, &o, nullptr));
    ok(flux_sync(c));
    EngineResult res = collect(c, p, ws);
    res.log = device_log(c, p);
    return res;
}

EngineResult run_fused_allgather_gemm(const ProblemSpec& p, ShardedWorkspace& ws, const TileShape& tile,
                                      const std::vector<CommTileSpec>& comm, TransferMode transfer, bool swizzle_on,
                                      const EngineOptions& opts, std::vector<std::vector<TransferRecord>>* traces) {
    if (p.pattern != Pattern::AllGatherGemm)
        throw ConfigError("run_fused_allgather_gemm requires AllGatherGemm pattern");
    grid_for(p, tile);
    ws.validate(p);
    if (static_cast<int>(comm.size()) != p.tp) throw ConfigError("need one CommTileSpec per rank");
    for (int r = 0; r < p.tp; ++r) comm[r].validate(p, r, transfer);
    const int rpct = comm[0].rows_per_comm_tile;
    for (const CommTileSpec& s : comm)
        if (s.rows_per_comm_tile != rpct) throw ConfigError("all ranks must share one communication tile size");
    check_directory(ws);
    ws.clear_outputs();
    std::lock_guard<std::mutex> g(g_mu);
    flux_comm* c = session_for(p);
    upload_inputs(c, p, ws);
    const flux_problem cp = cprob(p);
    const flux_tile ct{tile.tm, tile.tn};
    flux_opts o = copts(opts);
    o.trace = 1;  // EngineResult::log (and the TransferRecords)
    // TransferRecords come from the copy-engine transfer loop, which walks the
    // caller's comm orders descriptor by descriptor (engine.cpp:367-423); without
    // them the library's automatic engine runs (the tiles follow the arrival
    // order the comm orders imply either way).
    if (traces) o.ag_engine = 1;
    const size_t count = comm[0].order.size();
    std::vector<int> peer, begin, rows;
    for (int r = 0; r < p.tp; ++r) {
        if (comm[r].order.size() != count) throw ConfigError("all ranks' comm orders must have the same length");
        for (const TransferDesc& d : comm[r].order) {
            peer.push_back(d.peer);
            begin.push_back(d.row_begin);
            rows.push_back(d.rows);
        }
    }
    ok(flux_ag_gemm_ordered(c, &cp, &ct, rpct, transfer == TransferMode::Pull ? FLUX_PULL : FLUX_PUSH,
                            swizzle_on ? 1 : 0, &o, nullptr, nullptr, peer.data(), begin.data(), rows.data(),
                            static_cast<int>(count)));
    ok(flux_sync(c));
    if (traces) {
        // Device times of every descriptor's copy completion and flag write
        // (CUDA events on the copy stream); logical timestamps order all of
        // them, copies before flags on equal times (the reference's run clock).
        traces->assign(p.tp, {});
        struct Tick {
            int64_t ns;
            int phase, rank;
            size_t idx;
        };
        std::vector<Tick> ticks;
        for (int r = 0; r < p.tp; ++r) {
            std::vector<flux_transfer_record> recs(count);
            int n = 0;
            ok(flux_transfer_log(c, r, recs.data(), static_cast<int>(count), &n));
            for (int i = 0; i < n && i < static_cast<int>(count); ++i) {
                TransferRecord tr;
                tr.desc = TransferDesc{recs[i].peer, recs[i].row_begin, recs[i].rows, LinkClass::IntraNuma, -1, -1};
                for (const TransferDesc& d : comm[r].order)
                    if (d.row_begin == recs[i].row_begin && d.peer == recs[i].peer) tr.desc = d;
                tr.copy_done_ns = recs[i].copy_done_ns;
                tr.flag_set_ns = recs[i].flag_set_ns;
                (*traces)[r].push_back(tr);
                ticks.push_back({tr.copy_done_ns, 0, r, (*traces)[r].size() - 1});
                ticks.push_back({tr.flag_set_ns, 1, r, (*traces)[r].size() - 1});
            }
        }
        std::stable_sort(ticks.begin(), ticks.end(), [](const Tick& a, const Tick& b) {
            return a.ns != b.ns ? a.ns < b.ns : a.phase < b.phase;
        });
        for (size_t i = 0; i < ticks.size(); ++i) {
            TransferRecord& tr = (*traces)[ticks[i].rank][ticks[i].idx];
            (ticks[i].phase == 0 ? tr.copy_logical_ts : tr.flag_logical_ts) = i + 1;
        }
    }
    EngineResult res = collect(c, p, ws);
    res.log = device_log(c, p);
    return res;
}

std::vector<Matrix> run_nonoverlap(const ProblemSpec& p, ShardedWorkspace& ws, const TileShape& tile) {
    validate_tiling(p, tile);
    ws.validate(p);
    check_directory(ws);
    ws.clear_outputs();
    std::lock_guard<std::mutex> g(g_mu);
    flux_comm* c = session_for(p);
    upload_inputs(c, p, ws);
    const flux_problem cp = cprob(p);
    flux_opts o;
    flux_default_opts(&o);
    o.out_dtype = FLUX_F32;
    ok(flux_nonoverlap(c, &cp, &o, nullptr));
    ok(flux_sync(c));
    return collect(c, p, ws).outputs;
}

// Reference medium_schedule (engine.cpp:607-651): a partition count of tp or
// 2*tp (or 1 at tp=1) dividing m. RS, per rank and chunk: the chunk GEMM and the
// chunk transfer both follow the previous chunk's add, and the add joins them.
// AG, per rank: the transfers of the chunks owned by other ranks first, then
// one GEMM per chunk gated on its own chunk's transfer.
std::vector<MediumStep> medium_schedule(const ProblemSpec& p, int partitions) {
    p.validate();
    const bool valid = partitions == p.tp || partitions == 2 * p.tp || (p.tp == 1 && partitions == 1);
    if (!valid)
        throw ConfigError("partitions=" + std::to_string(partitions) + " must be tp or 2*tp (tp=" +
                          std::to_string(p.tp) + ")");
    if (p.m % partitions != 0) throw ConfigError("m must be divisible by the partition count");
    const int rows = p.m / partitions;
    std::vector<MediumStep> steps;
    auto step = [&](int r, MediumStep::Kind kind, int chunk, std::vector<int> deps) {
        MediumStep s;
        s.rank = r;
        s.kind = kind;
        s.chunk = chunk;
        s.deps = std::move(deps);
        steps.push_back(std::move(s));
        return static_cast<int>(steps.size()) - 1;
    };
    for (int r = 0; r < p.tp; ++r) {
        if (p.pattern == Pattern::GemmReduceScatter) {
            std::vector<int> after_add;
            for (int chunk = 0; chunk < partitions; ++chunk) {
                const int g = step(r, MediumStep::Kind::ChunkGemm, chunk, after_add);
                const int x = step(r, MediumStep::Kind::ChunkTransfer, chunk, after_add);
                after_add = {step(r, MediumStep::Kind::ChunkAdd, chunk, {g, x})};
            }
        } else {
            std::vector<std::vector<int>> gate(partitions);
            for (int chunk = 0; chunk < partitions; ++chunk)
                if (p.owner_of_row(chunk * rows) != r) gate[chunk] = {step(r, MediumStep::Kind::ChunkTransfer, chunk, {})};
            for (int chunk = 0; chunk < partitions; ++chunk) step(r, MediumStep::Kind::ChunkGemm, chunk, gate[chunk]);
        }
    }
    return steps;
}

MediumResult run_medium_grained(const ProblemSpec& p, ShardedWorkspace& ws, const TileShape& tile, int partitions) {
    validate_tiling(p, tile);
    MediumResult res;
    res.trace = medium_schedule(p, partitions);
    ws.validate(p);
    check_directory(ws);
    ws.clear_outputs();
    std::lock_guard<std::mutex> g(g_mu);
    flux_comm* c = session_for(p);
    upload_inputs(c, p, ws);
    const flux_problem cp = cprob(p);
    const flux_tile ct{tile.tm, tile.tn};
    flux_opts o;
    flux_default_opts(&o);
    o.out_dtype = FLUX_F32;
    ok(flux_medium_grained(c, &cp, &ct, partitions, &o, nullptr));
    ok(flux_sync(c));
    res.outputs = collect(c, p, ws).outputs;
    return res;
}

}  // namespace overlap
