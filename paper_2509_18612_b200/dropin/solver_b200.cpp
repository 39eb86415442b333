// solver_b200.cpp — drop-in replacement of proj/src/solver.cpp (header solver.hpp
// unchanged).  pquco / pluco / pdeco / solve_per_component run through lcb_solve:
// batches stay resident on the B200, the (alpha, T) schedule and seeding stay host-side
// inside libliftcut_b200.so.  Results are bit-identical to the reference in fp64 mode.
#include <string>
#include <vector>

#include "liftcut/solver.hpp"
#include "lcb_bridge.hpp"

namespace liftcut {

const char* to_string(Algorithm a) {
    switch (a) {
        case Algorithm::pQUCO: return "pquco";
        case Algorithm::pLUCO: return "pluco";
        case Algorithm::pDECO: return "pdeco";
    }
    return "pquco";
}

Algorithm algorithm_from_string(const std::string& name) {
    if (name == "pquco" || name == "pQUCO") return Algorithm::pQUCO;
    if (name == "pluco" || name == "pLUCO") return Algorithm::pLUCO;
    if (name == "pdeco" || name == "pDECO") return Algorithm::pDECO;
    throw ValidationError("unknown algorithm: " + name);
}

// solver.cpp:30-47 (same checks, same messages)
void SolverConfig::validate() const {
    if (batch_size < 1) throw ValidationError("batch_size must be >= 1");
    if (num_batches < 1) throw ValidationError("num_batches must be >= 1");
    if (lift_dim < 1) throw ValidationError("lift_dim must be >= 1");
    if (algorithm != Algorithm::pQUCO && lift_dim < 2)
        throw ValidationError("lifted algorithms need lift_dim >= 2");
    ascent.validate();
    if (lifted_ascent) lifted_ascent->validate();
    if (init.beta <= 0.0 || init.beta >= 1.0) throw ValidationError("init.beta must lie in (0, 1)");
    if (init.eta <= 0.0) throw ValidationError("init.eta must be > 0");
    if (init.init_scale < 1.0) throw ValidationError("init.init_scale must be >= 1");
    if (time_budget_s && *time_budget_s <= 0.0) throw ValidationError("time_budget_s must be > 0");
    if (search) search->validate();
    if (search_refresh < 0) throw ValidationError("search_refresh must be >= 0");
    if (deco_alternations < 1) throw ValidationError("deco_alternations must be >= 1");
}

namespace {

lcb_config to_abi(const SolverConfig& s, Algorithm algo) {
    lcb_config c{};
    c.algorithm = algo == Algorithm::pQUCO ? 0 : (algo == Algorithm::pLUCO ? 1 : 2);
    c.lift_dim = s.lift_dim;
    c.batch_size = s.batch_size;
    c.num_batches = s.num_batches;
    c.alpha = s.ascent.alpha;
    c.iterations = s.ascent.iterations;
    c.momentum = s.ascent.momentum;
    c.early_exit = s.ascent.early_exit;
    const AscentParams la = s.lifted_ascent.value_or(s.ascent);
    c.has_lifted_ascent = s.lifted_ascent.has_value();
    c.l_alpha = la.alpha;
    c.l_iterations = la.iterations;
    c.l_momentum = la.momentum;
    c.l_early_exit = la.early_exit;
    c.init_method = s.init.method == InitMethod::DUI ? 0 : 1;
    c.beta = s.init.beta;
    c.eta = s.init.eta;
    c.init_scale = s.init.init_scale;
    c.init_seed = s.init.seed;
    c.resample_idi = s.init.resample_idi;
    c.scale_noise = s.init.scale_noise;
    c.time_budget_s = s.time_budget_s.value_or(0.0);
    const SearchConfig q = s.search.value_or(SearchConfig{});
    c.has_search = s.search.has_value();
    c.population_size = q.population_size;
    c.t_lower = q.t_lower;
    c.t_upper = q.t_upper;
    c.e_lower = q.e_lower;
    c.e_upper = q.e_upper;
    c.rounds = q.rounds;
    c.search_refresh = s.search_refresh;
    c.deco_alternations = s.deco_alternations;
    c.deco_carry = s.deco_carry == DecoCarry::IncumbentColumn ? 0 : 1;
    return c;
}

void trace_trampoline(void* ctx, int64_t it, int64_t member, double obj) {
    (*static_cast<const TraceCallback*>(ctx))(it, member, obj);
}

SolveOutcome run(const Graph& g, const SolverConfig& cfg, std::uint64_t seed, Algorithm algo,
                 bool per_component, const TraceCallback& trace) {
    const b200::DeviceGraph dg = b200::upload(g);
    const lcb_config c = to_abi(cfg, algo);
    lcb_run_opts o{};
    o.precision = b200::precision();
    o.host_init = -1;
    if (trace) {
        o.trace_fn = &trace_trampoline;
        o.trace_ctx = const_cast<TraceCallback*>(&trace);
    }
    lcb_outcome r{};
    std::vector<std::uint8_t> z(g.node_count());
    constexpr int64_t cap = 1 << 16;
    std::vector<lcb_batch_trace> bt(cap);
    std::vector<lcb_phase_trace> pt(cap);
    std::vector<lcb_search_trace> st(cap);
    b200::check(lcb_solve(dg.get(), &c, seed, per_component, &o, &r, z.data(), bt.data(), cap, pt.data(), cap,
                          st.data(), cap));
    SolveOutcome out;
    out.best.assignment = std::move(z);
    out.best.cut_value = r.cut_value;
    out.best.algorithm = to_string(algo);
    out.best.seed = seed;
    out.best.batch_index = r.batch_index;
    out.best.member_index = r.member_index;
    out.best.wall_time_s = r.wall_s;
    for (int64_t i = 0; i < std::min(cap, r.n_batch_trace); ++i)
        out.batch_trace.push_back({bt[i].serial, bt[i].kind == 0 ? "main" : "search", bt[i].alpha,
                                   bt[i].iterations, bt[i].batch_best, bt[i].best_so_far});
    for (int64_t i = 0; i < std::min(cap, r.n_phase_trace); ++i)
        out.phase_trace.push_back({pt[i].phase, pt[i].kind == 0 ? "quco" : "luco", pt[i].best_after});
    for (int64_t i = 0; i < std::min(cap, r.n_search_trace); ++i)
        out.search_trace.push_back({st[i].round, st[i].exponent, st[i].iterations, st[i].fitness});
    out.stage_times = {r.init_s, r.ascent_s, r.rounding_s, r.search_s};
    out.batches_run = r.batches_run;
    return out;
}

void require_edges(const Graph& g) {
    if (g.edge_count() < 1) throw ValidationError("solver requires a graph with at least one edge");
}

}  // namespace

SolveOutcome pquco(const Graph& g, const SolverConfig& cfg, std::uint64_t seed, unsigned, const TraceCallback& trace) {
    cfg.validate();
    require_edges(g);
    return run(g, cfg, seed, Algorithm::pQUCO, false, trace);
}

SolveOutcome pluco(const Graph& g, const SolverConfig& cfg, std::uint64_t seed, unsigned, const TraceCallback& trace) {
    cfg.validate();
    require_edges(g);
    if (cfg.lift_dim < 2) throw ValidationError("pluco needs lift_dim >= 2");
    return run(g, cfg, seed, Algorithm::pLUCO, false, trace);
}

SolveOutcome pdeco(const Graph& g, const SolverConfig& cfg, std::uint64_t seed, unsigned, const TraceCallback& trace) {
    cfg.validate();
    require_edges(g);
    if (cfg.lift_dim < 2) throw ValidationError("pdeco needs lift_dim >= 2");
    return run(g, cfg, seed, Algorithm::pDECO, false, trace);
}

SolveOutcome solve_per_component(const Graph& g, const SolverConfig& cfg, std::uint64_t seed, unsigned,
                                 const TraceCallback& trace) {
    cfg.validate();
    if (g.edge_count() == 0) {  // every component trivial: zero assignment, nothing run
        SolveOutcome out;
        out.best.assignment.assign(g.node_count(), 0);
        out.best.algorithm = to_string(cfg.algorithm);
        out.best.seed = seed;
        out.best.batch_index = -1;
        out.best.member_index = -1;
        return out;
    }
    SolveOutcome out = run(g, cfg, seed, cfg.algorithm, true, trace);
    out.best.algorithm = to_string(cfg.algorithm);
    return out;
}

}  // namespace liftcut
