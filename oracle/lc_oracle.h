/*
 * lc_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (arXiv 2509.18612 "liftcut",
 * /root/reference/proj) used as the CPU checker for the B200 build.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product library (libliftcut_b200.so) never
 * links or calls anything in this directory.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the compiled reference (oracle/_ref, recipe in
 * oracle/Makefile, generator tests/golden/make_golden.py) and against the
 * reference's own known-answer tests (proj/tests/test_*.cpp).
 *
 * All arithmetic is IEEE binary64 with contraction disabled (-ffp-contract=off)
 * so that it reproduces the reference's scalar SSE2 code bit for bit.
 */
#ifndef LC_ORACLE_H
#define LC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes, same values as include/liftcut_b200.h. */
enum { ORC_OK = 0, ORC_VALIDATION = 1, ORC_SHAPE = 2, ORC_NUMERIC = 3, ORC_ERROR = 5 };

/* ---- counter RNG (rng.hpp:14-79) --------------------------------------- */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_combine(uint64_t key, uint64_t word);
uint64_t orc_split(uint64_t key, const uint64_t* path, int len);
uint64_t orc_at(uint64_t key, uint64_t counter);
double orc_unit(uint64_t bits);
/* Box-Muller normal built from counters (2k, 2k+1): the k-th next_normal(). */
double orc_normal_at(uint64_t key, uint64_t k);

/* ---- graph (graph.cpp) ---------------------------------------------------- */
/* CSR from an edge list: normalise u<v, sort, dedupe, symmetrise, per-row
 * sorted adjacency.  off has n+1 slots, adj has 2*ne slots.  Returns the
 * deduplicated edge count m (>= 0) or -1 on a self-loop / out-of-range id. */
int64_t orc_csr_build(uint32_t n, const uint32_t* eu, const uint32_t* ev, int64_t ne,
                      int64_t* off, uint32_t* adj);
void orc_laplacian(uint32_t n, const int64_t* off, const uint32_t* adj, const double* x,
                   double* y);
void orc_degree_stats(uint32_t n, const int64_t* off, double* mean, double* var, double* sd);
/* ER generator of graph.cpp:200-213 (pair order u<v row-major). Returns m or -1
 * if cap is too small.  Writes the pairs into eu/ev. */
int64_t orc_generate_er(uint32_t n, double p, uint64_t seed, uint32_t* eu, uint32_t* ev,
                        int64_t cap);

/* ---- ascent (ascent.cpp:43-96) ------------------------------------------- */
/* values: [B][l][n] member-major (dense_state.hpp:50-54), updated in place.
 * trace (optional, [T][B]): objective after each step; disables early exit.
 * On a non-finite value returns ORC_NUMERIC with err_iter / err_member set to
 * the first failure in member order (what workers=1 reports). */
int orc_ascend(uint32_t n, const int64_t* off, const uint32_t* adj, double* values, int l,
               int64_t B, double alpha, int64_t T, double mu, int early_exit, double* trace,
               int64_t* err_iter, int64_t* err_member);

/* ---- objectives (objectives.cpp) ----------------------------------------- */
int64_t orc_cut_value(uint32_t n, const int64_t* off, const uint32_t* adj, const uint8_t* z);
void orc_round_unlifted(int64_t n, const double* x, uint8_t* z);
void orc_round_lifted(int64_t n, int l, const double* member_values, uint8_t* z);
void orc_project_box(double* v, int64_t count);

/* ---- init (init.cpp) -------------------------------------------------------- */
int orc_dui_init(uint32_t n, const int64_t* off, uint64_t key, double* x);
void orc_idi_init(uint32_t n, const int64_t* off, const uint32_t* adj, double beta,
                  uint64_t key, double* x);
void orc_gaussian_batch(const double* mean, int64_t n, int l, double eta, int64_t B,
                        uint64_t key, double* out);
/* Members [first, first+count) of the batch above (sharding: member j's stream
 * depends only on (key, j), init.cpp:80). */
void orc_gaussian_members(const double* mean, int64_t n, int l, double eta, int64_t first,
                          int64_t count, uint64_t key, double* out);
void orc_lifted_init_mean(uint32_t n, const int64_t* off, const uint32_t* adj, int method,
                          double beta, int l, uint64_t key, double* mean);

/* ---- solver (solver.cpp, evo_search.cpp) --------------------------------- */
/* Layout shared with include/liftcut_b200.h (lcb_config). */
typedef struct orc_config {
    int32_t algorithm;        /* 0 pQUCO, 1 pLUCO, 2 pDECO */
    int32_t lift_dim;
    int64_t batch_size;
    int64_t num_batches;
    double alpha;
    int64_t iterations;
    double momentum;
    int32_t early_exit;
    int32_t has_lifted_ascent;
    double l_alpha;
    int64_t l_iterations;
    double l_momentum;
    int32_t l_early_exit;
    int32_t init_method;      /* 0 DUI, 1 IDI */
    double beta;
    double eta;
    double init_scale;
    uint64_t init_seed;
    int32_t resample_idi;
    int32_t scale_noise;
    double time_budget_s;     /* <= 0: no budget */
    int32_t has_search;
    int32_t population_size;
    int64_t t_lower;
    int64_t t_upper;
    double e_lower;
    double e_upper;
    int32_t rounds;
    int32_t search_refresh;
    int32_t deco_alternations;
    int32_t deco_carry;       /* 0 IncumbentColumn, 1 Fresh */
} orc_config;

typedef struct orc_batch_trace {
    int64_t serial;
    int32_t kind;             /* 0 main, 1 search */
    int32_t pad_;
    double alpha;
    int64_t iterations;
    int64_t batch_best;
    int64_t best_so_far;
} orc_batch_trace;

typedef struct orc_phase_trace {
    int32_t phase;
    int32_t kind;             /* 0 quco, 1 luco */
    int64_t best_after;
} orc_phase_trace;

typedef struct orc_search_trace {
    int32_t round;
    int32_t pad_;
    double exponent;
    int64_t iterations;
    double fitness;
} orc_search_trace;

typedef struct orc_outcome {
    int64_t cut_value;
    int64_t batch_index;
    int64_t member_index;
    int64_t batches_run;
    int64_t n_batch_trace;
    int64_t n_phase_trace;
    int64_t n_search_trace;
    double init_s, ascent_s, rounding_s, search_s, wall_s;
} orc_outcome;

/* Runs cfg.algorithm on g (solve_per_component when per_component != 0).
 * assignment has n slots; trace arrays hold up to *_cap rows (counts in out
 * report the full number).  Returns a status; ORC_VALIDATION mirrors the
 * reference's ValidationError cases. */
int orc_solve(uint32_t n, const int64_t* off, const uint32_t* adj, const orc_config* cfg,
              uint64_t seed, int per_component, orc_outcome* out, uint8_t* assignment,
              orc_batch_trace* bt, int64_t bt_cap, orc_phase_trace* pt, int64_t pt_cap,
              orc_search_trace* st, int64_t st_cap);

/* evo_search.cpp helpers, exposed for the evolve unit tests. */
void orc_sample_population(int64_t t_lower, int64_t t_upper, double e_lower, double e_upper,
                           int pop, uint64_t key, uint64_t* counter, double* exps,
                           int64_t* iters);
double orc_perturb_exponent(double e, uint64_t key, uint64_t* counter);
int64_t orc_perturb_iterations(int64_t t0, uint64_t key, uint64_t* counter);

/* Brute-force MaxCut (oracle.cpp:50-99) for n <= 26: optimum and lexicographic witness. */
int64_t orc_brute_force_maxcut(uint32_t n, const int64_t* off, const uint32_t* adj,
                               uint8_t* witness, int64_t* count_optimal);

#ifdef __cplusplus
}
#endif
#endif
