/*
 * liftcut_b200.h — C ABI of the B200-native liftcut hot path (libliftcut_b200.so).
 *
 * Drop-in boundary for the reference solver API in /root/reference/proj/include/liftcut.
 * Every entry point names the reference interface it replaces (file:line).  Plain
 * pointers and sizes only; host buffers in, host buffers out, device residency inside
 * the handles.  All functions are re-entrant: state lives in handles, the last error
 * message is thread-local.
 *
 * Status codes map one-to-one onto the reference exception types (errors.hpp:9-31):
 *   LCB_VALIDATION -> ValidationError, LCB_SHAPE -> ShapeError,
 *   LCB_NUMERIC -> NumericError ("... iteration <i>, member <j>", ascent.cpp:70-72),
 *   LCB_CUDA / LCB_ERROR -> Error.
 */
#ifndef LIFTCUT_B200_H
#define LIFTCUT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LCB_ABI_VERSION 3

enum lcb_status {
    LCB_OK = 0,
    LCB_VALIDATION = 1,
    LCB_SHAPE = 2,
    LCB_NUMERIC = 3,
    LCB_CUDA = 4,
    LCB_ERROR = 5,
    LCB_PARSE = 6 /* ParseError (graph.cpp:145-165) */
};

/* Arithmetic of the iterate.  FP64 reproduces the reference (fp64, no FMA,
 * sequential CSR-order sums: SPEC.md:100,364) bit for bit; FP32 is the fast path
 * (fp32 state and velocity, same algorithm, checked norm-wise). */
enum lcb_precision { LCB_FP64 = 0, LCB_FP32 = 1 };

typedef struct lcb_graph lcb_graph; /* device-resident CSR */
typedef struct lcb_comm lcb_comm;   /* NCCL communicator over the ranks of one box */

const char* lcb_last_error(void);
int lcb_abi_version(void);
int lcb_device_count(int* count);

/* Kernel-selection knobs (no reference counterpart; B200 tuning and tests).  Names:
 * "resident" (K2: -1 auto, 0 never, 1 whenever it fits), "stream" (K1s streaming step:
 * -1 auto, 1 on, 0 off), "signrec" (K1 saturation codes: -1 auto, 0, 1), "chunk" (K1n panels:
 * 0 off, 1 on, -1 auto), "res_split" (K2 wave-tail split), "bank_order" / "bank_refine"
 * (K2 fp32 neighbour order, read at graph creation), "dense" (K3 adjacency at graph
 * creation: -1 auto, 0, 1), "slab_outer" (K1s order: -1 auto, 0 all slabs per launch, 1 one
 * slab at a time for all iterations), "xcode" (K1s saturated slabs kept as sign codes: 1, 0),
 * "dense_cut" (K3 graphs: unlifted cut counts on the tensor cores: 1, 0 bit-sliced).  Defaults come from the LCB_<NAME> environment variables.
 * Changing a knob while a solve runs in another thread is not supported. */
int lcb_set_option(const char* name, int64_t value);
int lcb_get_option(const char* name, int64_t* value);

/* ---- graph: replaces the CSR of liftcut::Graph (graph.hpp:21-58) ------------
 * offsets int64[n+1] / adjacency uint32[offsets[n]] exactly as Graph stores them
 * (sorted, deduplicated, symmetric — graph.cpp:15-50).  The handle keeps a device
 * copy (int32 row pointers / columns, degree vector, degree-descending row order)
 * (the adjacency is copied back to the host only for a per-component solve). */
int lcb_graph_create(uint32_t n, const int64_t* offsets, const uint32_t* adjacency, int device,
                     lcb_graph** out);
/* Graph(n, edges) (graph.hpp:24, graph.cpp:15-50) built on the device: validation with the
 * reference's messages, normalise u<v, radix sort, unique, symmetrise, CSR (rows ascending).
 * eu / ev: m endpoints (duplicates and either orientation allowed). */
int lcb_graph_from_edges(uint32_t n, const uint32_t* eu, const uint32_t* ev, int64_t m, int device,
                         lcb_graph** out);
/* parse_edge_list(text) (graph.hpp:63-64, graph.cpp:136-172) on the device: the Gset /
 * edge-list text ("n m" header, then "u v [w]" lines with 1-based ids; '%' / '#' comments
 * and blank lines skipped) parsed line-parallel, then Graph(n, edges) built as in
 * lcb_graph_from_edges.  LCB_PARSE with the reference's message ("line <k>: expected
 * header \"n m\"", "... expected edge \"u v [w]\"", "... node id out of range [1, n]",
 * "empty input: ..."), LCB_VALIDATION for a self-loop ("line <k>: self-loop at node <u>").
 * saw_weights (optional) = 1 when an edge line carried a weight (the reference warns that
 * weights are ignored). */
int lcb_graph_parse(const char* text, int64_t len, int device, lcb_graph** out, int* saw_weights);
/* The CSR of a graph handle (Graph::offsets / adjacency, graph.hpp:52-57):
 * offsets [n+1], adjacency [2m] (either may be null). */
int lcb_graph_csr(const lcb_graph* g, int64_t* offsets, uint32_t* adjacency);
void lcb_graph_destroy(lcb_graph* g);
int lcb_graph_info(const lcb_graph* g, uint32_t* n, int64_t* m, int64_t* max_degree);

/* Graph::laplacian_apply (graph.hpp:50, graph.cpp:112-122) for `count` vectors
 * stored back to back ([count][n]). */
int lcb_laplacian_apply(const lcb_graph* g, const double* x, double* y, int64_t count,
                        int32_t precision);

/* ---- ascent: liftcut::ascend (ascent.hpp:33-34, ascent.cpp:43-96) -----------
 * values: DenseState::values, [B][l][n] (dense_state.hpp:50-54), updated in place.
 * trace: optional [iterations][B] objective per step (TraceCallback, ascent.hpp:21-23);
 * when given, early exit is disabled as in the reference (ascent.cpp:91).
 * On LCB_NUMERIC err_iter / err_member name the first failure in member order. */
int lcb_ascend(const lcb_graph* g, double* values, int64_t n, int32_t l, int64_t B, double alpha,
               int64_t iterations, double momentum, int32_t early_exit, int32_t precision,
               double* trace, int64_t* err_iter, int64_t* err_member);

/* ---- objectives (objectives.hpp:25,47,50; solver.cpp:125-138) --------------- */
/* Row-sharded ascend (north star 5; SURVEY 8e "row-sharding of A" for graphs beyond one
 * HBM): the same result as lcb_ascend on the whole graph, with rank q holding only the CSR
 * rows [row_begin, row_end) -- offsets [rows+1] starting at 0, adjacency with GLOBAL ids --
 * and its slice values [B][l][rows] of the DenseState (in/out).  The ranks' ranges must
 * partition [0, n) in rank order.  Every rank keeps the whole iterate; per iteration the
 * new rows are all-gathered (NCCL grouped broadcasts, or the loopback) and, with early
 * exit, the members' exit bits are OR-reduced, so the exit test sees the whole member
 * (ascent.cpp:74-75, 91-93).  comm = NULL: one rank owning [0, n).  fp64 is bit-exact with
 * the reference's ascend on the whole graph. */
int lcb_ascend_rows(lcb_comm* comm, uint32_t n, int64_t row_begin, int64_t row_end, const int64_t* offsets,
                    const uint32_t* adjacency, double* values, int32_t l, int64_t B, double alpha, int64_t iterations,
                    double momentum, int32_t early_exit, int32_t precision, int device, int64_t* err_iter,
                    int64_t* err_member);

/* cut_value for `count` assignments z[count][n]; LCB_VALIDATION if an entry > 1. */
int lcb_cut_values(const lcb_graph* g, const uint8_t* z, int64_t count, int64_t* cuts);
/* Round every member of a [B][l][n] batch (round_unlifted when lifted == 0,
 * round_lifted otherwise), evaluate its cut, pick the first maximum.  cuts [B]
 * and best_z [n] are optional. */
int lcb_round_cut_batch(const lcb_graph* g, const double* values, int32_t l, int64_t B,
                        int32_t lifted, int64_t* cuts, int64_t* best_member, int64_t* best_cut,
                        uint8_t* best_z);

/* round_unlifted (lifted == 0: z = 1{x > 0}, strict) / round_lifted (z = 1{sum_c X[v,c] >= 0}
 * in c order, inclusive) for every member of a [B][l][n] batch (objectives.cpp:81-96);
 * z [B][n]. */
int lcb_round(int device, const double* values, int64_t n, int32_t l, int64_t B, int32_t lifted, uint8_t* z);

/* Exhaustive MaxCut (brute_force_maxcut, oracle.hpp:18-22 / oracle.cpp:50-99) on the
 * device: Gray-code scan of the 2^(n-1) assignments with node 0 fixed.
 * - count_optimal counts z and its complement separately.
 * - witness [n] is the optimal assignment with the smallest integer encoding of
 *   min(z, ~z).
 * - max_nodes = 0 keeps the reference guard (n <= 26, LCB_VALIDATION above it).
 * - Larger values, up to 40, lift the guard.
 * - count_optimal and witness are optional. */
int lcb_brute_force_maxcut(const lcb_graph* g, int32_t max_nodes, int64_t* optimum, int64_t* count_optimal,
                           uint8_t* witness);

/* ---- init (init.hpp:37-52, init.cpp:20-101) ---------------------------------
 * Stream keys are RngStream::key() values (rng.hpp:27-79).  DUI / IDI / the lifted
 * mean are integer-exact; gaussian_batch draws its normals on the device (CUDA
 * double log / cos, within a few ulp of glibc's). */
int lcb_dui_init(const lcb_graph* g, uint64_t key, double* x);
int lcb_idi_init(const lcb_graph* g, double beta, uint64_t key, double* x);
int lcb_lifted_init_mean(const lcb_graph* g, int32_t method, double beta, int32_t l,
                         uint64_t key, double* mean);
int lcb_gaussian_batch(int device, const double* mean, int64_t n, int32_t l, double eta,
                       int64_t B, uint64_t key, double* out);
/* gaussian_batch bit-identical to the reference (init.cpp:69-87: host libm Box-Muller on
 * the member streams, members on host threads) -- the seeding the fp64 mode uses. */
int lcb_gaussian_batch_exact(const double* mean, int64_t n, int32_t l, double eta, int64_t B,
                             uint64_t key, double* out);

/* ---- solver (solver.hpp:26-90) ---------------------------------------------- */
typedef struct lcb_config { /* SolverConfig + AscentParams + InitConfig + SearchConfig */
    int32_t algorithm;       /* 0 pQUCO, 1 pLUCO, 2 pDECO (solver.hpp:17) */
    int32_t lift_dim;
    int64_t batch_size;      /* members per rank (global batch = batch_size * nranks) */
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
    int32_t init_method;     /* 0 DUI, 1 IDI */
    double beta;
    double eta;
    double init_scale;
    uint64_t init_seed;
    int32_t resample_idi;
    int32_t scale_noise;
    double time_budget_s;    /* <= 0: none */
    int32_t has_search;
    int32_t population_size;
    int64_t t_lower;
    int64_t t_upper;
    double e_lower;
    double e_upper;
    int32_t rounds;
    int32_t search_refresh;
    int32_t deco_alternations;
    int32_t deco_carry;      /* 0 IncumbentColumn, 1 Fresh */
} lcb_config;

typedef struct lcb_batch_trace { /* BatchTraceEntry (solver.hpp:43-50) */
    int64_t serial;
    int32_t kind;            /* 0 "main", 1 "search" */
    int32_t pad_;
    double alpha;
    int64_t iterations;
    int64_t batch_best;
    int64_t best_so_far;
} lcb_batch_trace;

typedef struct lcb_phase_trace { /* PhaseTraceEntry (solver.hpp:52-56) */
    int32_t phase;
    int32_t kind;            /* 0 "quco", 1 "luco" */
    int64_t best_after;
} lcb_phase_trace;

typedef struct lcb_search_trace { /* SearchTraceEntry (evo_search.hpp:40-45) */
    int32_t round;
    int32_t pad_;
    double exponent;
    int64_t iterations;
    double fitness;
} lcb_search_trace;

typedef struct lcb_outcome { /* SolveOutcome (solver.hpp:65-72) */
    int64_t cut_value;
    int64_t batch_index;
    int64_t member_index;    /* global member index */
    int64_t batches_run;
    int64_t n_batch_trace;
    int64_t n_phase_trace;
    int64_t n_search_trace;
    double init_s, ascent_s, rounding_s, search_s, wall_s; /* StageTimes + wall */
} lcb_outcome;

/* TraceCallback (ascent.hpp:21-23) for the main batches of a solve (solver.cpp:121):
 * called on the host after each main batch, member-major like workers=1. */
typedef void (*lcb_trace_fn)(void* ctx, int64_t iteration, int64_t member, double objective);

typedef struct lcb_run_opts { /* B200-side knobs; not part of the reference config */
    int32_t precision;       /* lcb_precision */
    int32_t host_init;       /* -1 auto (FP64: host glibc normals, FP32: device), 0 device, 1 host */
    int32_t batched_search;  /* evaluate each evolve() round as one multi-candidate launch */
    int32_t pad_;
    lcb_comm* comm;          /* NULL: single GPU */
    /* measurement out-params (may be NULL) */
    double* step_ms;         /* CUDA-event time of all PGA step launches */
    int64_t* step_launches;  /* number of PGA step launches */
    int64_t* node_updates;   /* sum over batches of n * B * l * iterations executed */
    double* step_bytes;      /* algorithmic bytes of all step launches */
    double* solve_ms;        /* CUDA-event time of the whole solve on its stream */
    double* kernel_stats;    /* [12]: K1 HBM-streaming {ms, launches, bytes}, K2 resident {ms, launches, bytes},
                                K3 dense tensor-core {ms, launches, algorithmic flops},
                                K1s warp-specialised streaming {ms, launches, bytes} */
    lcb_trace_fn trace_fn;   /* optional per-iteration objective trace (disables early exit) */
    void* trace_ctx;
} lcb_run_opts;

/* pquco / pluco / pdeco (solver.hpp:75-86) or solve_per_component (:88-90) when
 * per_component != 0.  assignment [n]; trace arrays are filled up to their caps, the
 * outcome reports the full counts. */
int lcb_solve(const lcb_graph* g, const lcb_config* cfg, uint64_t seed, int32_t per_component,
              const lcb_run_opts* opts, lcb_outcome* out, uint8_t* assignment,
              lcb_batch_trace* bt, int64_t bt_cap, lcb_phase_trace* pt, int64_t pt_cap,
              lcb_search_trace* st, int64_t st_cap);

/* Test hook: the K2 relabelled layout of a graph (graphs with n <= 14336).  len = entries
 * of the padded uint16 CSR (0 when the graph has none); col / col_fast [len] = CSR-order and
 * bank-balanced copies (col_fast all 0xffff when absent); row_words [n][2] = (first
 * 4-column word, degree) per relabelled row; perm [n] = relabelled -> original row. */
int lcb_debug_resident_layout(const lcb_graph* g, int64_t* len, uint16_t* col, uint16_t* col_fast,
                              int64_t* row_words, int32_t* perm);

/* Independent runs (run_bench's per-seed loop, bench.cpp:97-136: one solve — or
 * solve_per_component when per_component != 0 — per seed).  With a communicator, run i is
 * solved on rank i % nranks (no member sharding inside a run), then ONE exchange: the
 * per-run cuts (allreduce max) and the best run's outcome and assignment (first maximum in
 * run order) from its owner.  run_cuts [nruns] optional; best_out / assignment [n] are
 * filled on every rank; the measurement out-params of opts sum this rank's runs. */
int lcb_solve_runs(const lcb_graph* g, const lcb_config* cfg, const uint64_t* seeds, int64_t nruns,
                   int32_t per_component, const lcb_run_opts* opts, int64_t* run_cuts, int64_t* best_run,
                   lcb_outcome* best_out, uint8_t* assignment);

/* ---- multi-GPU (one process per GPU; NCCL over NVLink / NVSwitch) ------------
 * Members of every batch are sharded: rank r owns global members
 * [r*B, (r+1)*B).  Per batch one allreduce(max) of the packed (cut, ~member) key
 * and one allreduce(max) of the owner's winner bits; nothing inside the T loop. */
int lcb_comm_unique_id(uint8_t id[128]);
int lcb_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int device,
                    lcb_comm** out);
void lcb_comm_destroy(lcb_comm* c);
/* Loopback communicator: `nranks` ranks that are threads of ONE process (on one or several
 * GPUs); the same per-batch collectives run through device staging buffers and a host
 * barrier (no kernel waits on another).  For testing and emulating the sharded solve on
 * fewer GPUs than ranks.  Every rank must call the same sequence of solves. */
typedef struct lcb_loopback lcb_loopback;
int lcb_loopback_create(int32_t nranks, lcb_loopback** out);
void lcb_loopback_destroy(lcb_loopback* g);
int lcb_comm_create_loopback(lcb_loopback* group, int32_t rank, int device, lcb_comm** out);
/* Solves keep their device workspaces in a per-(device, precision) pool for reuse, and
 * graph arrays / ingest scratch come from each device's cached stream-ordered pool; this
 * frees every pooled workspace and trims those pools (e.g. before a large allocation
 * elsewhere). */
void lcb_release_workspaces(void);
/* process-wide counters: kernel launches and host<->device bytes since load */
void lcb_counters(int64_t* launches, int64_t* h2d_bytes, int64_t* d2h_bytes);
/* host helpers shared with the CPU tests of the exchange */
uint64_t lcb_pack_key(int64_t cut, int64_t global_member);
void lcb_unpack_key(uint64_t key, int64_t* cut, int64_t* global_member);

#ifdef __cplusplus
}
#endif
#endif
