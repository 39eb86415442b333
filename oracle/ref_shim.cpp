// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" face over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests, the golden-vector generator and bench.py's reference arm call
// the reference's own code through ctypes.  The product never links this.
//
// Every entry point catches the reference's exceptions and maps them onto the
// status codes of include/liftcut_b200.h (errors.hpp:9-31 -> 1/2/3/5).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "liftcut/ascent.hpp"
#include "liftcut/errors.hpp"
#include "liftcut/graph.hpp"
#include "liftcut/init.hpp"
#include "liftcut/objectives.hpp"
#include "liftcut/oracle.hpp"
#include "liftcut/rng.hpp"
#include "liftcut/solver.hpp"

#include "lc_oracle.h"  // shared config / trace layouts

using namespace liftcut;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 2;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

SolverConfig to_cfg(const orc_config& c) {
    SolverConfig s;
    s.algorithm = c.algorithm == 0 ? Algorithm::pQUCO : (c.algorithm == 1 ? Algorithm::pLUCO : Algorithm::pDECO);
    s.batch_size = c.batch_size;
    s.lift_dim = c.lift_dim;
    s.num_batches = c.num_batches;
    s.ascent.alpha = c.alpha;
    s.ascent.iterations = c.iterations;
    s.ascent.momentum = c.momentum;
    s.ascent.early_exit = c.early_exit != 0;
    if (c.has_lifted_ascent) {
        AscentParams p;
        p.alpha = c.l_alpha;
        p.iterations = c.l_iterations;
        p.momentum = c.l_momentum;
        p.early_exit = c.l_early_exit != 0;
        s.lifted_ascent = p;
    }
    s.init.method = c.init_method == 0 ? InitMethod::DUI : InitMethod::IDI;
    s.init.beta = c.beta;
    s.init.eta = c.eta;
    s.init.init_scale = c.init_scale;
    s.init.seed = c.init_seed;
    s.init.resample_idi = c.resample_idi != 0;
    s.init.scale_noise = c.scale_noise != 0;
    if (c.time_budget_s > 0.0) s.time_budget_s = c.time_budget_s;
    if (c.has_search) {
        SearchConfig q;
        q.t_lower = c.t_lower;
        q.t_upper = c.t_upper;
        q.e_lower = c.e_lower;
        q.e_upper = c.e_upper;
        q.population_size = c.population_size;
        q.rounds = c.rounds;
        s.search = q;
    }
    s.search_refresh = c.search_refresh;
    s.deco_alternations = c.deco_alternations;
    s.deco_carry = c.deco_carry == 0 ? DecoCarry::IncumbentColumn : DecoCarry::Fresh;
    return s;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Graph handle: built by the reference constructor from an edge list.
int ref_graph_new(uint32_t n, const uint32_t* eu, const uint32_t* ev, int64_t ne, void** out) {
    return guarded([&] {
        std::vector<std::pair<NodeId, NodeId>> edges(static_cast<std::size_t>(ne));
        for (int64_t i = 0; i < ne; ++i) edges[static_cast<std::size_t>(i)] = {eu[i], ev[i]};
        *out = new Graph(n, std::move(edges));
    });
}

int ref_graph_load(const char* path, void** out) {
    return guarded([&] { *out = new Graph(load_graph_file(path)); });
}

// parse_edge_list(text) (graph.cpp:136-172, 174-177)
int ref_graph_parse(const char* text, int64_t len, void** out) {
    return guarded([&] { *out = new Graph(parse_edge_list(std::string(text, static_cast<std::size_t>(len)))); });
}

int ref_graph_er(uint32_t n, double p, uint64_t seed, void** out) {
    return guarded([&] { *out = new Graph(generate_er(n, p, seed)); });
}

void ref_graph_free(void* h) { delete static_cast<Graph*>(h); }

void ref_graph_shape(void* h, uint32_t* n, int64_t* m, int64_t* maxdeg) {
    const Graph& g = *static_cast<Graph*>(h);
    *n = g.node_count();
    *m = g.edge_count();
    *maxdeg = g.max_degree();
}

void ref_graph_csr(void* h, int64_t* off, uint32_t* adj) {
    const Graph& g = *static_cast<Graph*>(h);
    int64_t pos = 0;
    for (NodeId v = 0; v < g.node_count(); ++v) {
        off[v] = pos;
        for (NodeId u : g.neighbors(v)) adj[pos++] = u;
    }
    off[g.node_count()] = pos;
}

int ref_laplacian(void* h, const double* x, double* y) {
    const Graph& g = *static_cast<Graph*>(h);
    return guarded([&] {
        g.laplacian_apply({x, g.node_count()}, {y, g.node_count()});
    });
}

void ref_degree_stats(void* h, double* mean, double* var, double* sd) {
    const DegreeStats s = static_cast<Graph*>(h)->degree_stats();
    *mean = s.mean;
    *var = s.variance;
    *sd = s.std_dev;
}

// ascend on a [B][l][n] buffer, in place.  trace: optional [T][B] objectives.
int ref_ascend(void* h, double* values, int64_t n, int l, int64_t B, double alpha, int64_t T,
               double mu, int early_exit, unsigned workers, double* trace) {
    const Graph& g = *static_cast<Graph*>(h);
    return guarded([&] {
        DenseState s;
        s.nodes = n;
        s.lift_dim = l;
        s.batch = B;
        s.values.assign(values, values + n * l * B);
        AscentParams p;
        p.alpha = alpha;
        p.iterations = T;
        p.momentum = mu;
        p.early_exit = early_exit != 0;
        TraceCallback cb = nullptr;
        if (trace)
            cb = [&](std::int64_t it, std::int64_t j, double obj) { trace[it * B + j] = obj; };
        try {
            ascend(g, s, p, workers, cb);
        } catch (...) {
            std::copy(s.values.begin(), s.values.end(), values);
            throw;
        }
        std::copy(s.values.begin(), s.values.end(), values);
    });
}

int64_t ref_cut_value(void* h, const uint8_t* z) {
    const Graph& g = *static_cast<Graph*>(h);
    int64_t out = -1;
    int st = guarded([&] { out = cut_value(g, {z, g.node_count()}); });
    return st == 0 ? out : -1;
}

void ref_round_unlifted(const double* x, int64_t n, uint8_t* z) {
    const auto r = round_unlifted({x, static_cast<std::size_t>(n)});
    std::memcpy(z, r.data(), r.size());
}

void ref_round_lifted(const double* values, int64_t n, int l, int64_t B, int64_t member,
                      uint8_t* z) {
    DenseState s;
    s.nodes = n;
    s.lift_dim = l;
    s.batch = B;
    s.values.assign(values, values + n * l * B);
    const auto r = round_lifted(s, member);
    std::memcpy(z, r.data(), r.size());
}

int ref_dui_init(void* h, uint64_t key, double* x) {
    const Graph& g = *static_cast<Graph*>(h);
    return guarded([&] {
        const auto v = dui_init(g, RngStream(key));
        std::copy(v.begin(), v.end(), x);
    });
}

void ref_idi_init(void* h, double beta, uint64_t key, double* x) {
    const Graph& g = *static_cast<Graph*>(h);
    const auto v = idi_init(g, beta, RngStream(key));
    std::copy(v.begin(), v.end(), x);
}

int ref_gaussian_batch(const double* mean, int64_t n, int l, double eta, int64_t B,
                       uint64_t key, unsigned workers, double* out) {
    return guarded([&] {
        const DenseState s = gaussian_batch({mean, static_cast<std::size_t>(n * l)}, n, l, eta,
                                            B, RngStream(key), workers);
        std::copy(s.values.begin(), s.values.end(), out);
    });
}

void ref_lifted_init_mean(void* h, int method, double beta, int l, uint64_t key, double* mean) {
    const Graph& g = *static_cast<Graph*>(h);
    InitConfig c;
    c.method = method == 0 ? InitMethod::DUI : InitMethod::IDI;
    c.beta = beta;
    const auto v = lifted_init_mean(g, c, l, RngStream(key));
    std::copy(v.begin(), v.end(), mean);
}

uint64_t ref_split(uint64_t key, const uint64_t* path, int len) {
    uint64_t k = key;
    for (int i = 0; i < len; ++i) k = RngStream(k).split({path[i]}).key();
    return k;
}

double ref_normal(uint64_t key, uint64_t k) {
    RngStream s(key);
    double v = 0.0;
    for (uint64_t i = 0; i <= k; ++i) v = s.next_normal();
    return v;
}

int ref_solve(void* h, const orc_config* cfg, uint64_t seed, int per_component, unsigned workers,
              orc_outcome* out, uint8_t* assignment, orc_batch_trace* bt, int64_t bt_cap,
              orc_phase_trace* pt, int64_t pt_cap, orc_search_trace* st, int64_t st_cap) {
    const Graph& g = *static_cast<Graph*>(h);
    return guarded([&] {
        const SolverConfig c = to_cfg(*cfg);
        SolveOutcome o;
        if (per_component) {
            o = solve_per_component(g, c, seed, workers);
        } else if (c.algorithm == Algorithm::pQUCO) {
            o = pquco(g, c, seed, workers);
        } else if (c.algorithm == Algorithm::pLUCO) {
            o = pluco(g, c, seed, workers);
        } else {
            o = pdeco(g, c, seed, workers);
        }
        std::memset(out, 0, sizeof(*out));
        out->cut_value = o.best.cut_value;
        out->batch_index = o.best.batch_index;
        out->member_index = o.best.member_index;
        out->batches_run = o.batches_run;
        out->n_batch_trace = static_cast<int64_t>(o.batch_trace.size());
        out->n_phase_trace = static_cast<int64_t>(o.phase_trace.size());
        out->n_search_trace = static_cast<int64_t>(o.search_trace.size());
        out->init_s = o.stage_times.init_s;
        out->ascent_s = o.stage_times.ascent_s;
        out->rounding_s = o.stage_times.rounding_s;
        out->search_s = o.stage_times.search_s;
        out->wall_s = o.best.wall_time_s;
        std::memcpy(assignment, o.best.assignment.data(), o.best.assignment.size());
        for (int64_t i = 0; i < std::min<int64_t>(bt_cap, out->n_batch_trace); ++i) {
            const auto& e = o.batch_trace[static_cast<std::size_t>(i)];
            bt[i] = {e.serial, e.kind == "main" ? 0 : 1, 0, e.alpha, e.iterations, e.batch_best,
                     e.best_so_far};
        }
        for (int64_t i = 0; i < std::min<int64_t>(pt_cap, out->n_phase_trace); ++i) {
            const auto& e = o.phase_trace[static_cast<std::size_t>(i)];
            pt[i] = {e.phase, e.kind == "quco" ? 0 : 1, e.best_after};
        }
        for (int64_t i = 0; i < std::min<int64_t>(st_cap, out->n_search_trace); ++i) {
            const auto& e = o.search_trace[static_cast<std::size_t>(i)];
            st[i] = {e.round, 0, e.exponent, e.iterations, e.fitness};
        }
    });
}

int64_t ref_brute_force(void* h, uint8_t* witness, int64_t* count) {
    const Graph& g = *static_cast<Graph*>(h);
    int64_t best = -1;
    guarded([&] {
        const OracleResult r = brute_force_maxcut(g, 1);
        best = r.optimum;
        *count = r.count_optimal;
        std::memcpy(witness, r.witness.data(), r.witness.size());
    });
    return best;
}

}  // extern "C"
