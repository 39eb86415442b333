#define _POSIX_C_SOURCE 199309L
/*
 * lc_oracle.c — TEST INFRASTRUCTURE ONLY (see lc_oracle.h).
 *
 * Sequential plain-C restatement of the liftcut reference hot path.  Every
 * function names the reference lines it restates.  Nothing here is tuned: it
 * is the slow, obviously-ordered version the CUDA kernels are checked against.
 * Build with -ffp-contract=off (oracle/Makefile) so no FMA is formed.
 */
#include "lc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ======================================================================== */
/* counter RNG — rng.hpp:14-23 (mix64 / combine), :32-43 (split / at),     */
/* :60-65 (Box-Muller), :73-75 (53-bit unit)                               */
/* ======================================================================== */

#define GOLDEN 0x9e3779b97f4a7c15ULL

uint64_t orc_mix64(uint64_t z) {
    z += GOLDEN;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t orc_combine(uint64_t key, uint64_t word) {
    return orc_mix64(key ^ (word + GOLDEN + (key << 6) + (key >> 2)));
}

uint64_t orc_split(uint64_t key, const uint64_t* path, int len) {
    for (int i = 0; i < len; ++i) key = orc_combine(key, path[i]);
    return key;
}

static uint64_t split1(uint64_t key, uint64_t a) { return orc_combine(key, a); }
static uint64_t split2(uint64_t key, uint64_t a, uint64_t b) {
    return orc_combine(orc_combine(key, a), b);
}
static uint64_t split3(uint64_t key, uint64_t a, uint64_t b, uint64_t c) {
    return orc_combine(orc_combine(orc_combine(key, a), b), c);
}

uint64_t orc_at(uint64_t key, uint64_t counter) {
    return orc_mix64(key ^ (counter * 0xd6e8feb86659fd93ULL));
}

double orc_unit(uint64_t bits) { return (double)(bits >> 11) * 0x1p-53; }

static double box_muller(double u1, double u2) {
    if (u1 <= 0.0) u1 = 0x1p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

double orc_normal_at(uint64_t key, uint64_t k) {
    return box_muller(orc_unit(orc_at(key, 2 * k)), orc_unit(orc_at(key, 2 * k + 1)));
}

/* A stateful stream (key + advancing counter), as RngStream::next_*. */
typedef struct {
    uint64_t key;
    uint64_t ctr;
} stream_t;

static uint64_t s_u64(stream_t* s) { return orc_at(s->key, s->ctr++); }
static double s_unit(stream_t* s) { return orc_unit(s_u64(s)); }
static double s_uniform(stream_t* s, double lo, double hi) { return lo + (hi - lo) * s_unit(s); }
static int64_t s_int(stream_t* s, int64_t lo, int64_t hi) {
    uint64_t span = (uint64_t)(hi - lo) + 1;
    return lo + (int64_t)(s_u64(s) % span);
}
static double s_normal(stream_t* s) {
    double u1 = s_unit(s);
    double u2 = s_unit(s);
    return box_muller(u1, u2);
}

/* ======================================================================== */
/* graph — Graph::Graph graph.cpp:15-50, laplacian_apply :112-122,          */
/* degree_stats :61-73, generate_er :200-213                                */
/* ======================================================================== */

static int cmp_pair(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int64_t orc_csr_build(uint32_t n, const uint32_t* eu, const uint32_t* ev, int64_t ne,
                      int64_t* off, uint32_t* adj) {
    if (n == 0) return -1;
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(ne > 0 ? ne : 1));
    for (int64_t i = 0; i < ne; ++i) {
        uint32_t u = eu[i], v = ev[i];
        if (u >= n || v >= n || u == v) {
            free(keys);
            return -1;
        }
        if (u > v) { uint32_t t = u; u = v; v = t; }
        keys[i] = ((uint64_t)u << 32) | v;
    }
    qsort(keys, (size_t)ne, sizeof(uint64_t), cmp_pair);
    int64_t m = 0;
    for (int64_t i = 0; i < ne; ++i)
        if (i == 0 || keys[i] != keys[i - 1]) keys[m++] = keys[i];
    for (uint32_t v = 0; v <= n; ++v) off[v] = 0;
    for (int64_t i = 0; i < m; ++i) {
        ++off[(keys[i] >> 32) + 1];
        ++off[(keys[i] & 0xffffffffu) + 1];
    }
    for (uint32_t v = 1; v <= n; ++v) off[v] += off[v - 1];
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * n);
    memcpy(cur, off, sizeof(int64_t) * n);
    for (int64_t i = 0; i < m; ++i) {
        uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)(keys[i] & 0xffffffffu);
        adj[cur[u]++] = v;
        adj[cur[v]++] = u;
    }
    for (uint32_t v = 0; v < n; ++v)
        qsort(adj + off[v], (size_t)(off[v + 1] - off[v]), sizeof(uint32_t), cmp_u32);
    free(cur);
    free(keys);
    return m;
}

void orc_laplacian(uint32_t n, const int64_t* off, const uint32_t* adj, const double* x,
                   double* y) {
    for (uint32_t v = 0; v < n; ++v) {
        double acc = 0.0;
        for (int64_t k = off[v]; k < off[v + 1]; ++k) acc += x[adj[k]];
        y[v] = (double)(off[v + 1] - off[v]) * x[v] - acc;
    }
}

void orc_degree_stats(uint32_t n, const int64_t* off, double* mean, double* var, double* sd) {
    const double nn = (double)n;
    const double mu = (double)off[n] / nn; /* 2m / n */
    double acc = 0.0;
    for (uint32_t v = 0; v < n; ++v) {
        double d = (double)(off[v + 1] - off[v]) - mu;
        acc += d * d;
    }
    *mean = mu;
    *var = acc / nn;
    *sd = sqrt(*var);
}

int64_t orc_generate_er(uint32_t n, double p, uint64_t seed, uint32_t* eu, uint32_t* ev,
                        int64_t cap) {
    const uint64_t key = split1(seed, 0x4552u);
    uint64_t pair = 0;
    int64_t m = 0;
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t v = u + 1; v < n; ++v, ++pair)
            if (orc_unit(orc_at(key, pair)) < p) {
                if (m >= cap) return -1;
                eu[m] = u;
                ev[m] = v;
                ++m;
            }
    return m;
}

/* ======================================================================== */
/* objectives — cut_value objectives.cpp:26-35, project_box :75-79,         */
/* round_unlifted :81-85, round_lifted :87-96                               */
/* ======================================================================== */

int64_t orc_cut_value(uint32_t n, const int64_t* off, const uint32_t* adj, const uint8_t* z) {
    for (uint32_t v = 0; v < n; ++v)
        if (z[v] > 1) return -1;
    int64_t crossing = 0;
    for (uint32_t u = 0; u < n; ++u)
        for (int64_t k = off[u]; k < off[u + 1]; ++k)
            if (u < adj[k] && z[u] != z[adj[k]]) ++crossing;
    return crossing;
}

void orc_round_unlifted(int64_t n, const double* x, uint8_t* z) {
    for (int64_t v = 0; v < n; ++v) z[v] = x[v] > 0.0 ? 1 : 0;
}

void orc_round_lifted(int64_t n, int l, const double* mv, uint8_t* z) {
    for (int64_t v = 0; v < n; ++v) {
        double s = 0.0;
        for (int c = 0; c < l; ++c) s += mv[(int64_t)c * n + v];
        z[v] = s >= 0.0 ? 1 : 0;
    }
}

static double clamp1(double r) { return r < -1.0 ? -1.0 : (r > 1.0 ? 1.0 : r); }

void orc_project_box(double* v, int64_t count) {
    for (int64_t i = 0; i < count; ++i) v[i] = clamp1(v[i]);
}

/* ======================================================================== */
/* ascend — ascent.cpp:43-96 (heavy-ball PGA, per-member early exit)       */
/* ======================================================================== */

int orc_ascend(uint32_t n, const int64_t* off, const uint32_t* adj, double* values, int l,
               int64_t B, double alpha, int64_t T, double mu, int early_exit, double* trace,
               int64_t* err_iter, int64_t* err_member) {
    if (!(alpha > 0.0) || T < 1 || !(mu >= 0.0 && mu < 1.0)) return ORC_VALIDATION;
    const int64_t entries = (int64_t)n * l;
    double* vel = (double*)malloc(sizeof(double) * (size_t)entries);
    double* dir = (double*)malloc(sizeof(double) * (size_t)entries);
    double* lx = (double*)malloc(sizeof(double) * n);
    int status = ORC_OK;
    for (int64_t j = 0; j < B && status == ORC_OK; ++j) {
        double* x = values + j * entries;
        memset(vel, 0, sizeof(double) * (size_t)entries);
        for (int64_t it = 0; it < T; ++it) {
            for (int c = 0; c < l; ++c)
                orc_laplacian(n, off, adj, x + (int64_t)c * n, dir + (int64_t)c * n);
            double max_change = 0.0;
            int boundary = 1;
            for (int64_t k = 0; k < entries; ++k) {
                vel[k] = mu * vel[k] + dir[k];
                const double raw = x[k] + alpha * vel[k];
                if (!isfinite(raw)) {
                    *err_iter = it;
                    *err_member = j;
                    status = ORC_NUMERIC;
                    break;
                }
                const double cl = clamp1(raw);
                const double ch = fabs(cl - x[k]);
                if (ch > max_change) max_change = ch;
                if (cl != 1.0 && cl != -1.0) boundary = 0;
                x[k] = cl;
            }
            if (status != ORC_OK) break;
            if (trace) {
                double obj = 0.0;
                for (int c = 0; c < l; ++c) {
                    const double* xc = x + (int64_t)c * n;
                    orc_laplacian(n, off, adj, xc, lx);
                    for (uint32_t v = 0; v < n; ++v) obj += xc[v] * lx[v];
                }
                trace[it * B + j] = obj;
            }
            if (early_exit && !trace) {
                if (boundary ? max_change == 0.0 : max_change <= 1e-12) break;
            }
        }
    }
    free(vel);
    free(dir);
    free(lx);
    return status;
}

/* ======================================================================== */
/* init — dui_init init.cpp:20-30, idi_init :32-62, gaussian_batch :69-87,  */
/* lifted_init_mean :89-101                                                 */
/* ======================================================================== */

int orc_dui_init(uint32_t n, const int64_t* off, uint64_t key, double* x) {
    int64_t maxdeg = 0;
    for (uint32_t v = 0; v < n; ++v)
        if (off[v + 1] - off[v] > maxdeg) maxdeg = off[v + 1] - off[v];
    if (maxdeg < 1) return ORC_VALIDATION;
    const double md = (double)maxdeg;
    for (uint32_t v = 0; v < n; ++v) {
        const double bound = 1.0 - (double)(off[v + 1] - off[v]) / md;
        x[v] = (2.0 * orc_unit(orc_at(key, v)) - 1.0) * bound;
    }
    return ORC_OK;
}

void orc_idi_init(uint32_t n, const int64_t* off, const uint32_t* adj, double beta,
                  uint64_t key, double* x) {
    double mean, var, sd;
    orc_degree_stats(n, off, &mean, &var, &sd);
    const double thr = mean + beta * sd;
    signed char* sgn = (signed char*)calloc(n ? n : 1, 1);
    for (uint32_t v = 0; v < n; ++v)
        if ((double)(off[v + 1] - off[v]) > thr) sgn[v] = (orc_at(key, v) & 1u) ? 1 : -1;
    const uint64_t tie = split1(key, 0x7469u);
    for (uint32_t v = 0; v < n; ++v) {
        if (sgn[v]) {
            x[v] = (double)sgn[v];
            continue;
        }
        int64_t plus = 0, minus = 0;
        for (int64_t k = off[v]; k < off[v + 1]; ++k) {
            plus += sgn[adj[k]] > 0;
            minus += sgn[adj[k]] < 0;
        }
        if (plus == minus)
            x[v] = (orc_at(tie, v) & 1u) ? 1.0 : -1.0;
        else
            x[v] = plus < minus ? 1.0 : -1.0;
    }
    free(sgn);
}

void orc_gaussian_batch(const double* mean, int64_t n, int l, double eta, int64_t B,
                        uint64_t key, double* out) {
    const int64_t entries = n * l;
    const double ns = sqrt(eta);
    for (int64_t j = 0; j < B; ++j) {
        const uint64_t mk = split2(key, 0x6d62u, (uint64_t)j);
        double* o = out + j * entries;
        for (int64_t k = 0; k < entries; ++k) o[k] = clamp1(mean[k] + ns * orc_normal_at(mk, (uint64_t)k));
    }
}

void orc_gaussian_members(const double* mean, int64_t n, int l, double eta, int64_t first,
                          int64_t count, uint64_t key, double* out) {
    const int64_t entries = n * l;
    const double ns = sqrt(eta);
    for (int64_t j = 0; j < count; ++j) {
        const uint64_t mk = split2(key, 0x6d62u, (uint64_t)(first + j));
        double* o = out + j * entries;
        for (int64_t k = 0; k < entries; ++k) o[k] = clamp1(mean[k] + ns * orc_normal_at(mk, (uint64_t)k));
    }
}

void orc_lifted_init_mean(uint32_t n, const int64_t* off, const uint32_t* adj, int method,
                          double beta, int l, uint64_t key, double* mean) {
    for (int c = 0; c < l; ++c) {
        const uint64_t ck = split2(key, 0x636fu, (uint64_t)c);
        if (method == 0)
            orc_dui_init(n, off, ck, mean + (int64_t)c * n);
        else
            orc_idi_init(n, off, adj, beta, ck, mean + (int64_t)c * n);
    }
}

/* ======================================================================== */
/* evolutionary search — evo_search.cpp:26-90                               */
/* ======================================================================== */

void orc_sample_population(int64_t t_lower, int64_t t_upper, double e_lower, double e_upper,
                           int pop, uint64_t key, uint64_t* counter, double* exps,
                           int64_t* iters) {
    stream_t s = {key, *counter};
    for (int i = 0; i < pop; ++i) {
        iters[i] = s_int(&s, t_lower, t_upper);
        exps[i] = s_uniform(&s, e_lower, e_upper);
    }
    *counter = s.ctr;
}

static double perturb_e(double e, stream_t* s) {
    double moved = e + 0.2 * s_normal(s);
    return moved < -4.0 ? -4.0 : (moved > -1.0 ? -1.0 : moved);
}

static int64_t perturb_t(int64_t t0, stream_t* s) {
    const double eps = s_unit(s);
    int64_t scaled = (int64_t)floor((double)t0 * (1.0 + 0.2 * (2.0 * eps - 1.0)));
    return scaled < 1 ? 1 : scaled;
}

double orc_perturb_exponent(double e, uint64_t key, uint64_t* counter) {
    stream_t s = {key, *counter};
    double r = perturb_e(e, &s);
    *counter = s.ctr;
    return r;
}

int64_t orc_perturb_iterations(int64_t t0, uint64_t key, uint64_t* counter) {
    stream_t s = {key, *counter};
    int64_t r = perturb_t(t0, &s);
    *counter = s.ctr;
    return r;
}

/* ======================================================================== */
/* solver — solver.cpp:92-312 (run_batch, note_batch, run_search, run_phase, */
/* pquco/pluco/pdeco) and :314-364 (solve_per_component)                     */
/* ======================================================================== */

typedef struct {
    double exponent;
    int64_t iterations;
    int has_fit;
    double fitness;
} cand_t;

typedef struct {
    /* graph */
    uint32_t n;
    const int64_t* off;
    const uint32_t* adj;
    const orc_config* cfg;
    uint64_t base;
    struct timespec t0;
    /* global best */
    int has_best;
    int64_t best_cut, best_serial, best_member;
    uint8_t* best_z;
    int64_t serial;
    int has_tuned[2];
    cand_t tuned[2];
    int64_t main_batches[2];
    uint64_t search_runs[2];
    /* traces */
    orc_batch_trace* bt;
    int64_t bt_cap, nbt;
    orc_phase_trace* pt;
    int64_t pt_cap, npt;
    orc_search_trace* st;
    int64_t st_cap, nst;
    double init_s, ascent_s, rounding_s, search_s;
    int status;
} ctx_t;

static double now_s(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

static double elapsed(const ctx_t* c) {
    return now_s() - ((double)c->t0.tv_sec + 1e-9 * (double)c->t0.tv_nsec);
}

static int budget_gone(const ctx_t* c) {
    return c->cfg->time_budget_s > 0.0 && elapsed(c) >= c->cfg->time_budget_s;
}

/* pm1_scaled — solver.cpp:92-101 */
static void pm1_scaled(const uint8_t* z, uint32_t n, int l, double scale, double* mean) {
    for (uint32_t v = 0; v < n; ++v) mean[v] = (z[v] ? 1.0 : -1.0) / scale;
    for (int c = 1; c < l; ++c) memcpy(mean + (int64_t)c * n, mean, sizeof(double) * n);
}

typedef struct {
    int64_t cut, serial, member;
    uint8_t* z; /* n bytes, owned by caller */
} bres_t;

/* run_batch — solver.cpp:106-143 */
static int run_batch(ctx_t* c, int lifted, int l, const double* mean, double alpha, int64_t T,
                     double mu, int early_exit, int book_stages, double* trace, bres_t* out) {
    const orc_config* cfg = c->cfg;
    const uint32_t n = c->n;
    const int64_t B = cfg->batch_size;
    const int64_t serial = c->serial++;
    const uint64_t bkey = split2(c->base, 0x6261u, (uint64_t)serial);
    const double eta_eff =
        cfg->scale_noise ? cfg->eta / (cfg->init_scale * cfg->init_scale) : cfg->eta;
    double* vals = (double*)malloc(sizeof(double) * (size_t)(B * l * (int64_t)n));
    double t = now_s();
    orc_gaussian_batch(mean, n, l, eta_eff, B, bkey, vals);
    if (book_stages) c->init_s += now_s() - t;
    t = now_s();
    int64_t ei, ej;
    int st = orc_ascend(n, c->off, c->adj, vals, l, B, alpha, T, mu, early_exit, trace, &ei, &ej);
    if (book_stages) c->ascent_s += now_s() - t;
    if (st != ORC_OK) {
        free(vals);
        return st;
    }
    t = now_s();
    uint8_t* z = (uint8_t*)malloc(n);
    int64_t best_cut = -1, best_j = 0;
    for (int64_t j = 0; j < B; ++j) {
        const double* mv = vals + j * l * (int64_t)n;
        if (lifted)
            orc_round_lifted(n, l, mv, z);
        else
            orc_round_unlifted(n, mv, z);
        const int64_t cut = orc_cut_value(n, c->off, c->adj, z);
        if (j == 0 || cut > best_cut) {
            best_cut = cut;
            best_j = j;
        }
    }
    const double* bv = vals + best_j * l * (int64_t)n;
    if (lifted)
        orc_round_lifted(n, l, bv, out->z);
    else
        orc_round_unlifted(n, bv, out->z);
    out->cut = best_cut;
    out->serial = serial;
    out->member = best_j;
    if (book_stages) c->rounding_s += now_s() - t;
    free(z);
    free(vals);
    return ORC_OK;
}

/* note_batch — solver.cpp:145-150 */
static void note_batch(ctx_t* c, const bres_t* r, int kind, double alpha, int64_t T) {
    if (!c->has_best || r->cut > c->best_cut) {
        c->has_best = 1;
        c->best_cut = r->cut;
        c->best_serial = r->serial;
        c->best_member = r->member;
        memcpy(c->best_z, r->z, c->n);
    }
    if (c->nbt < c->bt_cap) {
        orc_batch_trace* e = &c->bt[c->nbt];
        e->serial = r->serial;
        e->kind = kind;
        e->pad_ = 0;
        e->alpha = alpha;
        e->iterations = T;
        e->batch_best = r->cut;
        e->best_so_far = c->best_cut;
    }
    ++c->nbt;
}

static int ranks_before(const cand_t* a, const cand_t* b) {
    const double fa = a->has_fit ? a->fitness : -INFINITY;
    const double fb = b->has_fit ? b->fitness : -INFINITY;
    if (fa != fb) return fa > fb;
    if (a->iterations != b->iterations) return a->iterations < b->iterations;
    return a->exponent < b->exponent;
}

/* stable insertion sort == std::stable_sort under ranks_before */
static void stable_rank(cand_t* p, int count) {
    for (int i = 1; i < count; ++i) {
        cand_t key = p[i];
        int j = i - 1;
        while (j >= 0 && ranks_before(&key, &p[j])) {
            p[j + 1] = p[j];
            --j;
        }
        p[j + 1] = key;
    }
}

/* run_search — solver.cpp:154-180 driving evolve — evo_search.cpp:61-90 */
static int run_search(ctx_t* c, int lifted, int l, const uint8_t* incumbent, double mu,
                      int early_exit, cand_t* winner) {
    const orc_config* cfg = c->cfg;
    const double t_start = now_s();
    const int kind = lifted ? 1 : 0;
    stream_t s = {split3(c->base, 0x6576u, (uint64_t)kind, c->search_runs[kind]++), 0};
    double* mean = (double*)malloc(sizeof(double) * (size_t)c->n * l);
    pm1_scaled(incumbent, c->n, l, cfg->init_scale, mean);
    const int pop = cfg->population_size;
    cand_t* P = (cand_t*)calloc((size_t)pop, sizeof(cand_t));
    for (int i = 0; i < pop; ++i) {
        P[i].iterations = s_int(&s, cfg->t_lower, cfg->t_upper);
        P[i].exponent = s_uniform(&s, cfg->e_lower, cfg->e_upper);
    }
    bres_t r;
    r.z = (uint8_t*)malloc(c->n);
    const int half = pop / 2;
    for (int round = 1; round <= cfg->rounds; ++round) {
        for (int i = 0; i < pop; ++i) {
            if (P[i].has_fit) continue;
            double fit;
            if (budget_gone(c)) {
                fit = -INFINITY;
            } else {
                const double a = pow(10.0, P[i].exponent);
                int st = run_batch(c, lifted, l, mean, a, P[i].iterations, mu, early_exit, 0, NULL, &r);
                if (st == ORC_OK) {
                    note_batch(c, &r, 1, a, P[i].iterations);
                    fit = (double)r.cut;
                } else {
                    fit = -INFINITY;
                }
            }
            P[i].has_fit = 1;
            P[i].fitness = fit;
            if (c->nst < c->st_cap) {
                orc_search_trace* e = &c->st[c->nst];
                e->round = round;
                e->pad_ = 0;
                e->exponent = P[i].exponent;
                e->iterations = P[i].iterations;
                e->fitness = fit;
            }
            ++c->nst;
        }
        stable_rank(P, pop);
        for (int slot = half; slot < pop; ++slot) {
            const cand_t* parent = &P[s_int(&s, 0, half - 1)];
            cand_t child = {0};
            child.exponent = perturb_e(parent->exponent, &s);
            child.iterations = perturb_t(parent->iterations, &s);
            P[slot] = child;
        }
    }
    *winner = P[0];
    free(r.z);
    free(P);
    free(mean);
    c->search_s += now_s() - t_start;
    return ORC_OK;
}

static int search_due(const ctx_t* c, int kind) {
    if (!c->cfg->has_search) return 0;
    const int64_t count = c->main_batches[kind];
    if (c->cfg->search_refresh > 0) return (count - 1) % c->cfg->search_refresh == 0;
    return !c->has_tuned[kind] && count == 1;
}

/* run_phase — solver.cpp:191-246.  carry: in/out n-byte buffer, *has_carry flag. */
static int run_phase(ctx_t* c, int lifted, int phase_idx, uint8_t* carry, int* has_carry,
                     double* trace_buf) {
    const orc_config* cfg = c->cfg;
    const uint32_t n = c->n;
    const int l = lifted ? cfg->lift_dim : 1;
    const int kind = lifted ? 1 : 0;
    double alpha = cfg->alpha, mu = cfg->momentum;
    int64_t T = cfg->iterations;
    int ee = cfg->early_exit;
    if (lifted && cfg->has_lifted_ascent) {
        alpha = cfg->l_alpha;
        T = cfg->l_iterations;
        mu = cfg->l_momentum;
        ee = cfg->l_early_exit;
    }
    if (c->has_tuned[kind]) {
        alpha = pow(10.0, c->tuned[kind].exponent);
        T = c->tuned[kind].iterations;
    }
    double* mean = (double*)malloc(sizeof(double) * (size_t)n * l);
    uint8_t* recenter = (uint8_t*)malloc(n);
    int has_recenter = *has_carry;
    if (has_recenter) memcpy(recenter, carry, n);
    int has_pbest = 0;
    int64_t pbest_cut = 0;
    uint8_t* pbest_z = (uint8_t*)malloc(n);
    bres_t r;
    r.z = (uint8_t*)malloc(n);
    int status = ORC_OK;
    for (int64_t b = 0; b < cfg->num_batches; ++b) {
        if (c->serial > 0 && budget_gone(c)) break;
        if (b == 0) {
            const double t = now_s();
            const uint64_t word = cfg->resample_idi ? (uint64_t)c->serial : 0u;
            const uint64_t ikey = split3(c->base, 0x696eu, cfg->init_seed, word);
            const int carry_col0 = has_recenter && (l == 1 || cfg->deco_carry == 0);
            orc_lifted_init_mean(n, c->off, c->adj, cfg->init_method, cfg->beta, l, ikey, mean);
            if (carry_col0)
                for (uint32_t v = 0; v < n; ++v) mean[v] = recenter[v] ? 1.0 : -1.0;
            for (int64_t k = 0; k < (int64_t)n * l; ++k) mean[k] /= cfg->init_scale;
            c->init_s += now_s() - t;
        } else {
            pm1_scaled(recenter, n, l, cfg->init_scale, mean);
        }
        status = run_batch(c, lifted, l, mean, alpha, T, mu, ee, 1, trace_buf, &r);
        if (status != ORC_OK) break;
        note_batch(c, &r, 0, alpha, T);
        if (!has_pbest || r.cut > pbest_cut) {
            has_pbest = 1;
            pbest_cut = r.cut;
            memcpy(pbest_z, r.z, n);
        }
        memcpy(recenter, r.z, n);
        has_recenter = 1;
        ++c->main_batches[kind];
        if (search_due(c, kind) && !budget_gone(c)) {
            cand_t w;
            status = run_search(c, lifted, l, recenter, mu, ee, &w);
            if (status != ORC_OK) break;
            alpha = pow(10.0, w.exponent);
            T = w.iterations;
            c->tuned[kind] = w;
            c->has_tuned[kind] = 1;
        }
    }
    if (status == ORC_OK) {
        if (!has_pbest) {
            if (has_recenter) memcpy(carry, recenter, n);
            *has_carry = has_recenter;
        } else {
            if (c->npt < c->pt_cap) {
                c->pt[c->npt].phase = phase_idx;
                c->pt[c->npt].kind = kind;
                c->pt[c->npt].best_after = pbest_cut;
            }
            ++c->npt;
            memcpy(carry, pbest_z, n);
            *has_carry = 1;
        }
    }
    free(r.z);
    free(pbest_z);
    free(recenter);
    free(mean);
    return status;
}

static int validate_cfg(const orc_config* c) {
    if (c->batch_size < 1 || c->num_batches < 1 || c->lift_dim < 1) return ORC_VALIDATION;
    if (c->algorithm != 0 && c->lift_dim < 2) return ORC_VALIDATION;
    if (!(c->alpha > 0.0) || c->iterations < 1 || !(c->momentum >= 0.0 && c->momentum < 1.0))
        return ORC_VALIDATION;
    if (c->has_lifted_ascent &&
        (!(c->l_alpha > 0.0) || c->l_iterations < 1 || !(c->l_momentum >= 0.0 && c->l_momentum < 1.0)))
        return ORC_VALIDATION;
    if (c->beta <= 0.0 || c->beta >= 1.0 || c->eta <= 0.0 || c->init_scale < 1.0) return ORC_VALIDATION;
    if (c->has_search) {
        if (c->t_lower < 1 || c->t_lower > c->t_upper || c->e_lower > c->e_upper ||
            c->population_size < 2 || c->population_size % 2 != 0 || c->rounds < 1)
            return ORC_VALIDATION;
    }
    if (c->search_refresh < 0 || c->deco_alternations < 1) return ORC_VALIDATION;
    return ORC_OK;
}

/* pquco / pluco / pdeco — solver.cpp:273-312 on one (sub)graph.  The ctx
 * arrives with its trace sinks set; everything else is reset here. */
static int solve_one(uint32_t n, const int64_t* off, const uint32_t* adj, const orc_config* cfg,
                     uint64_t seed, ctx_t* c, uint8_t* assignment) {
    orc_batch_trace* bt = c->bt;
    orc_phase_trace* pt = c->pt;
    orc_search_trace* st = c->st;
    const int64_t bc = c->bt_cap, pc = c->pt_cap, sc = c->st_cap;
    memset(c, 0, sizeof(*c));
    c->bt = bt; c->bt_cap = bc;
    c->pt = pt; c->pt_cap = pc;
    c->st = st; c->st_cap = sc;
    if (off[n] < 1) return ORC_VALIDATION; /* require_edges, solver.cpp:266-271 */
    c->n = n;
    c->off = off;
    c->adj = adj;
    c->cfg = cfg;
    c->base = seed;
    clock_gettime(CLOCK_MONOTONIC, &c->t0);
    c->best_z = assignment;
    uint8_t* carry = (uint8_t*)malloc(n);
    int has_carry = 0;
    int s = ORC_OK;
    if (cfg->algorithm == 0) {
        s = run_phase(c, 0, 0, carry, &has_carry, NULL);
    } else if (cfg->algorithm == 1) {
        s = run_phase(c, 1, 0, carry, &has_carry, NULL);
    } else {
        int phase = 0;
        for (int round = 0; s == ORC_OK; ++round) {
            if (cfg->time_budget_s > 0.0) {
                if (c->serial > 0 && budget_gone(c)) break;
            } else if (round >= cfg->deco_alternations) {
                break;
            }
            const int64_t before = c->serial;
            s = run_phase(c, 0, phase++, carry, &has_carry, NULL);
            if (s != ORC_OK) break;
            s = run_phase(c, 1, phase++, carry, &has_carry, NULL);
            if (cfg->time_budget_s > 0.0 && c->serial == before) break;
        }
    }
    free(carry);
    if (s == ORC_OK && !c->has_best) s = ORC_ERROR;
    return s;
}

/* connected components, graph.cpp:75-99 (roots ascending, members sorted) */
static int64_t components(uint32_t n, const int64_t* off, const uint32_t* adj, uint32_t* order,
                          int64_t* comp_start) {
    uint8_t* seen = (uint8_t*)calloc(n, 1);
    uint32_t* stack = (uint32_t*)malloc(sizeof(uint32_t) * n);
    int64_t nc = 0, pos = 0;
    for (uint32_t root = 0; root < n; ++root) {
        if (seen[root]) continue;
        comp_start[nc++] = pos;
        int64_t sp = 0, begin = pos;
        seen[root] = 1;
        stack[sp++] = root;
        while (sp) {
            uint32_t v = stack[--sp];
            order[pos++] = v;
            for (int64_t k = off[v]; k < off[v + 1]; ++k)
                if (!seen[adj[k]]) {
                    seen[adj[k]] = 1;
                    stack[sp++] = adj[k];
                }
        }
        qsort(order + begin, (size_t)(pos - begin), sizeof(uint32_t), cmp_u32);
    }
    comp_start[nc] = pos;
    free(stack);
    free(seen);
    return nc;
}

static void fill_outcome(const ctx_t* c, orc_outcome* out) {
    out->cut_value = c->best_cut;
    out->batch_index = c->best_serial;
    out->member_index = c->best_member;
    out->batches_run = c->serial;
    out->n_batch_trace = c->nbt;
    out->n_phase_trace = c->npt;
    out->n_search_trace = c->nst;
    out->init_s = c->init_s;
    out->ascent_s = c->ascent_s;
    out->rounding_s = c->rounding_s;
    out->search_s = c->search_s;
}

static int64_t room(int64_t cap, int64_t used) { return cap > used ? cap - used : 0; }

int orc_solve(uint32_t n, const int64_t* off, const uint32_t* adj, const orc_config* cfg,
              uint64_t seed, int per_component, orc_outcome* out, uint8_t* assignment,
              orc_batch_trace* bt, int64_t bt_cap, orc_phase_trace* pt, int64_t pt_cap,
              orc_search_trace* st, int64_t st_cap) {
    int s = validate_cfg(cfg);
    if (s != ORC_OK) return s;
    memset(out, 0, sizeof(*out));
    const double t0 = now_s();
    ctx_t c;
    memset(&c, 0, sizeof(c));
    c.bt = bt; c.bt_cap = bt_cap;
    c.pt = pt; c.pt_cap = pt_cap;
    c.st = st; c.st_cap = st_cap;

    uint32_t* order = NULL;
    int64_t* cstart = NULL;
    int64_t nc = 1;
    if (per_component) {
        order = (uint32_t*)malloc(sizeof(uint32_t) * n);
        cstart = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
        nc = components(n, off, adj, order, cstart);
    }
    if (!per_component || (nc == 1 && off[n] > 0)) {
        s = solve_one(n, off, adj, cfg, seed, &c, assignment);
        if (s == ORC_OK) fill_outcome(&c, out);
        out->wall_s = now_s() - t0;
        free(order);
        free(cstart);
        return s;
    }
    /* solve_per_component — solver.cpp:314-364 */
    memset(assignment, 0, n);
    out->batch_index = -1;
    out->member_index = -1;
    uint32_t* local = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t v = 0; v < n; ++v) local[v] = n;
    int solved = 0;
    for (int64_t ci = 0; ci < nc && s == ORC_OK; ++ci) {
        const int64_t k = cstart[ci + 1] - cstart[ci];
        const uint32_t* comp = order + cstart[ci];
        if (k < 2) continue;
        for (int64_t i = 0; i < k; ++i) local[comp[i]] = (uint32_t)i;
        int64_t ne = 0;
        for (int64_t i = 0; i < k; ++i) ne += off[comp[i] + 1] - off[comp[i]];
        uint32_t* eu = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(ne / 2 + 1));
        uint32_t* ev = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(ne / 2 + 1));
        int64_t m = 0;
        for (int64_t i = 0; i < k; ++i) {
            const uint32_t v = comp[i];
            for (int64_t q = off[v]; q < off[v + 1]; ++q)
                if (v < adj[q] && local[adj[q]] != n) {
                    eu[m] = local[v];
                    ev[m] = local[adj[q]];
                    ++m;
                }
        }
        int64_t* soff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k + 1));
        uint32_t* sadj = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(2 * m + 1));
        orc_csr_build((uint32_t)k, eu, ev, m, soff, sadj);
        for (int64_t i = 0; i < k; ++i) local[comp[i]] = n;
        if (soff[k] > 0) {
            const uint64_t sub_seed = orc_at(split2(seed, 0x6370u, (uint64_t)ci), 0);
            uint8_t* za = (uint8_t*)malloc((size_t)k);
            ctx_t sc;
            memset(&sc, 0, sizeof(sc));
            sc.bt = bt ? bt + (out->n_batch_trace < bt_cap ? out->n_batch_trace : bt_cap) : NULL;
            sc.bt_cap = room(bt_cap, out->n_batch_trace);
            sc.pt = pt ? pt + (out->n_phase_trace < pt_cap ? out->n_phase_trace : pt_cap) : NULL;
            sc.pt_cap = room(pt_cap, out->n_phase_trace);
            sc.st = st ? st + (out->n_search_trace < st_cap ? out->n_search_trace : st_cap) : NULL;
            sc.st_cap = room(st_cap, out->n_search_trace);
            s = solve_one((uint32_t)k, soff, sadj, cfg, sub_seed, &sc, za);
            if (s == ORC_OK) {
                for (int64_t i = 0; i < k; ++i) assignment[comp[i]] = za[i];
                out->cut_value += sc.best_cut;
                out->batch_index = sc.best_serial;
                out->member_index = sc.best_member;
                out->batches_run += sc.serial;
                out->init_s += sc.init_s;
                out->ascent_s += sc.ascent_s;
                out->rounding_s += sc.rounding_s;
                out->search_s += sc.search_s;
                out->n_batch_trace += sc.nbt;
                out->n_phase_trace += sc.npt;
                out->n_search_trace += sc.nst;
                ++solved;
            }
            free(za);
        }
        free(soff);
        free(sadj);
        free(eu);
        free(ev);
    }
    if (solved != 1) {
        out->batch_index = -1;
        out->member_index = -1;
    }
    out->wall_s = now_s() - t0;
    free(local);
    free(order);
    free(cstart);
    return s;
}

int64_t orc_brute_force_maxcut(uint32_t n, const int64_t* off, const uint32_t* adj,
                               uint8_t* witness, int64_t* count_optimal) {
    if (n > 26 || n == 0) return -1;
    const uint64_t full = (n >= 64) ? ~0ULL : ((1ULL << n) - 1);
    int64_t best = -1, count = 0;
    uint64_t best_enc = ~0ULL;
    for (uint64_t c = 0; c < (1ULL << (n - 1)); ++c) {
        const uint64_t enc = c << 1; /* node 0 fixed on side 0 */
        int64_t cut = 0;
        for (uint32_t u = 0; u < n; ++u)
            for (int64_t k = off[u]; k < off[u + 1]; ++k)
                if (u < adj[k] && ((enc >> u) & 1u) != ((enc >> adj[k]) & 1u)) ++cut;
        const uint64_t cand = enc < (full ^ enc) ? enc : (full ^ enc);
        if (cut > best) {
            best = cut;
            count = 2;
            best_enc = cand;
        } else if (cut == best) {
            count += 2;
            if (cand < best_enc) best_enc = cand;
        }
    }
    for (uint32_t v = 0; v < n; ++v) witness[v] = (uint8_t)((best_enc >> v) & 1u);
    *count_optimal = count;
    return best;
}
