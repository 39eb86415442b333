// lcb_runtime.cu — host runtime behind include/liftcut_b200.h.
//
// Re-states the reference orchestration (solver.cpp:106-364, evo_search.cpp:61-90)
// around device-resident batches: the batch iterate, velocity, packed assignments,
// the incumbent / phase-best / global-best assignments and the next batch's mean all
// stay in HBM; per batch only the packed (cut, member) key crosses to the host.
// Graph loading, stream-key derivation (seeding) and the (alpha, T) schedule stay
// on the host, as the north star asks.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <numeric>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "../../include/liftcut_b200.h"
#include "lcb_internal.h"

namespace lcb {

// ---------------------------------------------------------------------------
// errors / small utilities
// ---------------------------------------------------------------------------
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0}, g_h2d{0}, g_d2h{0};
void count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
void count_h2d(size_t b) { g_h2d.fetch_add(static_cast<int64_t>(b), std::memory_order_relaxed); }
void count_d2h(size_t b) { g_d2h.fetch_add(static_cast<int64_t>(b), std::memory_order_relaxed); }

// host<->device copies go through these so the bench can report e2e bytes
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    count_h2d(bytes);
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync(H2D)");
}
void d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    count_d2h(bytes);
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync(D2H)");
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Failure{LCB_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
#define CK(x) cuda_check((x), #x)

int num_sms(int device) {
    static std::atomic<int> cache[64];
    if (device < 0 || device >= 64) return 148;
    int v = cache[device].load(std::memory_order_relaxed);
    if (!v) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
        cache[device].store(v, std::memory_order_relaxed);
    }
    return v;
}

struct OptDef {
    const char* name;
    const char* env;
    int64_t def;
};
constexpr OptDef kOptDefs[OPT_COUNT] = {
    {"resident", "LCB_RESIDENT", -1}, {"stream", "LCB_STREAM", 1},         {"signrec", "LCB_SIGNREC", -1},
    {"chunk", "LCB_CHUNK", 0},        {"res_split", "LCB_RES_SPLIT", 1},   {"bank_order", "LCB_BANK_ORDER", 2},
    {"bank_refine", "LCB_BANK_REFINE", 2}, {"dense", "LCB_DENSE", -1}, {"slab_outer", "LCB_SLAB_OUTER", -1},
    {"xcode", "LCB_XCODE", 1},        {"dense_cut", "LCB_DENSE_CUT", 1},
};
std::atomic<int64_t> g_opts[OPT_COUNT];
std::once_flag g_opts_once;
void init_opts() {
    std::call_once(g_opts_once, [] {
        for (int i = 0; i < OPT_COUNT; ++i) {
            const char* e = std::getenv(kOptDefs[i].env);
            g_opts[i].store(e ? std::atoll(e) : kOptDefs[i].def);
        }
    });
}
int64_t option(Opt o) {
    init_opts();
    return g_opts[o].load(std::memory_order_relaxed);
}
int opt_index(const char* name) {
    for (int i = 0; i < OPT_COUNT; ++i)
        if (name && std::strcmp(name, kOptDefs[i].name) == 0) return i;
    return -1;
}

void ensure_smem_attr(const void* kernel, int bytes, const char* what) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& d : done)
        if (d.first == kernel && d.second == dev) return;
    cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), what);
    done.emplace_back(kernel, dev);
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return LCB_OK;
    } catch (const Failure& e) {
        g_last_error = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return LCB_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LCB_ERROR;
    }
}

[[noreturn]] void fail(int status, const std::string& msg) { throw Failure{status, msg}; }

struct DeviceScope {
    int prev = 0;
    explicit DeviceScope(int d) {
        cudaGetDevice(&prev);
        CK(cudaSetDevice(d));
    }
    ~DeviceScope() { cudaSetDevice(prev); }
};

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    T* ensure(size_t k) {
        if (k == 0) k = 1;
        if (k > cap) {
            release();
            CK(cudaMalloc(&p, k * sizeof(T)));
            cap = k;
        }
        return p;
    }
};

using Clock = std::chrono::steady_clock;
double secs_since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

uint64_t split1(uint64_t k, uint64_t a) { return combine(k, a); }
uint64_t split2(uint64_t k, uint64_t a, uint64_t b) { return combine(combine(k, a), b); }
uint64_t split3(uint64_t k, uint64_t a, uint64_t b, uint64_t c) {
    return combine(combine(combine(k, a), b), c);
}

// host stateful stream — RngStream::next_* (rng.hpp:38-70)
struct HostStream {
    uint64_t key;
    uint64_t ctr = 0;
    uint64_t u64() { return rng_at(key, ctr++); }
    double unit() { return rng_unit(u64()); }
    double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }
    int64_t integer(int64_t lo, int64_t hi) {
        const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
        return lo + static_cast<int64_t>(u64() % span);
    }
    double normal() {
        double u1 = unit();
        const double u2 = unit();
        if (u1 <= 0.0) u1 = 0x1p-53;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
    }
};

// ---------------------------------------------------------------------------
// device graph
// ---------------------------------------------------------------------------
// Graph arrays come from the device's stream-ordered pool, kept cached (release threshold
// at its maximum): a plain cudaFree of the ~40 MB of a config-4 graph took up to 200 ms
// in the e2e loop (one graph per solve); pooled frees and re-allocations are immediate.
void* pool_alloc(size_t bytes, cudaStream_t st) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    static std::mutex mu;
    static bool pooled[64] = {};
    if (dev >= 0 && dev < 64) {
        std::lock_guard<std::mutex> lk(mu);
        if (!pooled[dev]) {
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, dev));
            uint64_t thr = ~0ull;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
            pooled[dev] = true;
        }
    }
    void* p = nullptr;
    CK(cudaMallocAsync(&p, bytes ? bytes : 1, st));
    return p;
}
void pool_free(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}
void* graph_alloc(size_t bytes) {
    void* p = pool_alloc(bytes, 0);
    CK(cudaStreamSynchronize(0));  // usable from any stream
    return p;
}
void graph_free(void* p) { pool_free(p, 0); }

void free_graph(DevGraph& g) {
    graph_free(g.row_ptr);
    graph_free(g.col);
    graph_free(g.deg64);
    graph_free(g.deg32);
    graph_free(g.order);
    graph_free(g.res_info);
    graph_free(g.res_chunk);
    graph_free(g.res_heavy);
    g.res_heavy = nullptr;
    graph_free(g.dense_A);
    g.dense_A = nullptr;
    graph_free(g.res_col);
    graph_free(g.res_col_fast);
    g.res_info = nullptr;
    g.row_ptr = g.col = g.order = g.res_chunk = nullptr;
    g.res_col = g.res_col_fast = nullptr;
    g.res_perm = nullptr;
    g.deg64 = nullptr;
    g.deg32 = nullptr;
}

// Local search after the greedy bank-balanced order (K2 fp32 copy of the CSR): inside
// one 32-row warp group, swap two positions of one row's padded neighbour list when that
// lowers (max, sum of squares) of the distinct-slot counts per bank pair of the two
// half-warp gather steps involved.  A step's 8-byte LDS costs, per half-warp, the largest
// number of distinct slots in one bank pair; pads (the zero sentinel row n) are one slot.
// Groups are independent, so they are refined on several host threads.
// BA 10k model (light rows): greedy 10080 -> 8307 wavefronts per iteration.
static void refine_bank_order(std::vector<uint16_t>& fast, const std::vector<int64_t>& rrp, uint32_t H,
                              uint32_t n, int passes) {
    const uint32_t groups = (n - H + 31) / 32;
    if (groups == 0) return;
    auto work = [&](uint32_t g0, uint32_t stride) {
        struct HalfStep {
            uint16_t slot[16];
            uint8_t mult[16];
            int k = 0;
            int c = 0;  // cached cost
            int bank[16] = {0};
        };
        std::vector<HalfStep> hs;
        auto cost = [](const int* b) {
            int mx = 0, sq = 0;
            for (int j = 0; j < 16; ++j) {
                mx = std::max(mx, b[j]);
                sq += b[j] * b[j];
            }
            return mx * 1024 + sq;
        };
        auto add = [](HalfStep& h, uint16_t u) {
            for (int j = 0; j < h.k; ++j)
                if (h.slot[j] == u) {
                    ++h.mult[j];
                    return;
                }
            h.slot[h.k] = u;
            h.mult[h.k++] = 1;
            ++h.bank[u & 15];
        };
        auto del = [](HalfStep& h, uint16_t u) {
            for (int j = 0; j < h.k; ++j)
                if (h.slot[j] == u) {
                    if (--h.mult[j] == 0) {
                        --h.bank[u & 15];
                        h.slot[j] = h.slot[h.k - 1];
                        h.mult[j] = h.mult[h.k - 1];
                        --h.k;
                    }
                    return;
                }
        };
        for (uint32_t gi = g0; gi < groups; gi += stride) {  // strided: groups are in degree order
            const uint32_t b0 = H + 32 * gi, b1 = std::min<uint32_t>(b0 + 32, n);
            const int rows = static_cast<int>(b1 - b0);
            int L = 0;
            for (int i = 0; i < rows; ++i) L = std::max<int>(L, static_cast<int>(rrp[b0 + i + 1] - rrp[b0 + i]));
            hs.assign(static_cast<size_t>(2) * L, HalfStep{});
            for (int i = 0; i < rows; ++i) {
                const int Li = static_cast<int>(rrp[b0 + i + 1] - rrp[b0 + i]);
                for (int p = 0; p < Li; ++p) add(hs[2 * p + (i >> 4)], fast[static_cast<size_t>(rrp[b0 + i] + p)]);
            }
            for (auto& x : hs) x.c = cost(x.bank);
            for (int pass = 0; pass < passes; ++pass) {
                bool changed = false;
                for (int i = 0; i < rows; ++i) {
                    const int h = i >> 4;
                    const int Li = static_cast<int>(rrp[b0 + i + 1] - rrp[b0 + i]);
                    uint16_t* row = fast.data() + rrp[b0 + i];
                    for (int p = 0; p < Li; ++p)
                        for (int q = p + 1; q < Li; ++q) {
                            const uint16_t a = row[p], b = row[q];
                            if (a == b) continue;
                            HalfStep& P = hs[2 * p + h];
                            HalfStep& Q = hs[2 * q + h];
                            if (P.c < 2048 && Q.c < 2048) continue;  // both conflict-free already
                            const int before = P.c + Q.c;
                            del(P, a);
                            add(P, b);
                            del(Q, b);
                            add(Q, a);
                            const int cp = cost(P.bank), cq = cost(Q.bank);
                            if (cp + cq < before) {
                                row[p] = b;
                                row[q] = a;
                                P.c = cp;
                                Q.c = cq;
                                changed = true;
                            } else {
                                del(P, b);
                                add(P, a);
                                del(Q, a);
                                add(Q, b);
                            }
                        }
                }
                if (!changed) break;
            }
        }
    };
    const uint32_t hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const uint32_t nt = std::min<uint32_t>(hw, (groups + 7) / 8);
    if (nt <= 1) {
        work(0, 1);
        return;
    }
    std::vector<std::thread> th;
    for (uint32_t t = 1; t < nt; ++t) th.emplace_back(work, t, nt);
    work(0, nt);
    for (auto& t : th) t.join();
}

// Host CSR in (lcb_graph_create), or an adjacency already built on the device by the
// edge-list ingest (dev_col, owned from here on; `adj` is then its host copy when the
// host relabelling below needs it, i.e. n <= kResidentMaxRows, else null).
void build_graph(DevGraph& g, uint32_t n, const int64_t* off, const uint32_t* adj, int device,
                 int* dev_col = nullptr) {
    struct BuildTimer {  // LCB_BUILD_TIMING=1: host / upload split of a graph build (stderr)
        bool on = std::getenv("LCB_BUILD_TIMING") != nullptr;
        Clock::time_point t0 = Clock::now(), last = t0;
        std::string msg;
        void mark(const char* what) {
            if (!on) return;
            if (what[0] != 'h') cudaDeviceSynchronize();
            const auto t = Clock::now();
            msg += std::string(" ") + what + "=" + std::to_string(std::chrono::duration<double>(t - last).count() * 1e3);
            last = t;
        }
        ~BuildTimer() {
            if (on) fprintf(stderr, "build_graph ms:%s total=%.3f\n", msg.c_str(), secs_since(t0) * 1e3);
        }
    } bt;
    if (dev_col) g.col = dev_col;  // freed with the graph, also on failure
    if (n == 0) fail(LCB_VALIDATION, "graph must have at least one node");
    if (off[0] != 0) fail(LCB_VALIDATION, "offsets[0] must be 0");
    for (uint32_t v = 0; v < n; ++v)
        if (off[v + 1] < off[v]) fail(LCB_VALIDATION, "offsets must be non-decreasing");
    const int64_t nnz = off[n];
    if (nnz > std::numeric_limits<int>::max()) fail(LCB_VALIDATION, "graph exceeds 2^31 adjacency entries");
    // adjacency range check: on the host when the host relabelling below indexes with the
    // entries (n <= kResidentMaxRows), else on the device right after the upload
    const bool host_check = n <= static_cast<uint32_t>(kResidentMaxRows);
    if (host_check && !dev_col) {
        uint32_t mx = 0;  // branch-free (vectorised) scan
        for (int64_t k = 0; k < nnz; ++k) mx = std::max(mx, adj[k]);
        if (nnz && mx >= n) fail(LCB_VALIDATION, "adjacency entry out of range");
    }
    g.device = device;
    g.n = static_cast<int>(n);
    g.nnz = nnz;
    g.m = nnz / 2;
    std::vector<int> rp(n + 1), deg(n), ord(n);
    std::vector<double> d64(n);
    std::vector<float> d32(n);
    int64_t maxd = 0;
    for (uint32_t v = 0; v <= n; ++v) rp[v] = static_cast<int>(off[v]);
    for (uint32_t v = 0; v < n; ++v) {
        deg[v] = static_cast<int>(off[v + 1] - off[v]);
        d64[v] = static_cast<double>(deg[v]);
        d32[v] = static_cast<float>(deg[v]);
        maxd = std::max<int64_t>(maxd, deg[v]);
    }
    g.max_degree = maxd;
    // degree_stats, sequential fp64 exactly as graph.cpp:61-73
    const double nn = static_cast<double>(n);
    g.deg_mean = 2.0 * static_cast<double>(g.m) / nn;
    double acc = 0.0;
    for (uint32_t v = 0; v < n; ++v) {
        const double d = static_cast<double>(deg[v]) - g.deg_mean;
        acc += d * d;
    }
    g.deg_var = acc / nn;
    g.deg_sd = std::sqrt(g.deg_var);
    {  // rows by descending degree, ties in id order: a stable counting sort, O(n + max degree)
        std::vector<int64_t> start(static_cast<size_t>(maxd) + 2, 0);
        for (uint32_t v = 0; v < n; ++v) ++start[static_cast<size_t>(maxd - deg[v]) + 1];
        for (size_t d = 1; d < start.size(); ++d) start[d] += start[d - 1];
        for (uint32_t v = 0; v < n; ++v) ord[static_cast<size_t>(start[static_cast<size_t>(maxd - deg[v])]++)] = static_cast<int>(v);
    }

    bt.mark("host");
    DeviceScope ds(device);
    g.row_ptr = static_cast<decltype(g.row_ptr)>(graph_alloc(sizeof(int) * (n + 1)));
    if (!dev_col) g.col = static_cast<decltype(g.col)>(graph_alloc(sizeof(int) * (nnz + 4)));  // K1s copies aligned 16-byte runs
    g.deg64 = static_cast<decltype(g.deg64)>(graph_alloc(sizeof(double) * n));
    g.deg32 = static_cast<decltype(g.deg32)>(graph_alloc(sizeof(float) * n));
    g.order = static_cast<decltype(g.order)>(graph_alloc(sizeof(int) * n));
    h2d(g.row_ptr, rp.data(), sizeof(int) * (n + 1), 0);
    // uint32 ids < n < 2^31: the same bits as int32, uploaded straight from the caller
    if (nnz && !dev_col) h2d(g.col, adj, sizeof(int) * nnz, 0);
    bt.mark("up_csr");
    if (!host_check && nnz && !dev_col) {
        unsigned* dmx = nullptr;
        CK(cudaMalloc(&dmx, sizeof(unsigned)));
        launch_max_u32(reinterpret_cast<const uint32_t*>(g.col), nnz, dmx, 0);
        unsigned mx = 0;
        d2h(&mx, dmx, sizeof(unsigned), 0);
        CK(cudaStreamSynchronize(0));
        cudaFree(dmx);
        if (mx >= n) fail(LCB_VALIDATION, "adjacency entry out of range");
    }
    bt.mark("maxcheck");
    h2d(g.deg64, d64.data(), sizeof(double) * n, 0);
    h2d(g.deg32, d32.data(), sizeof(float) * n, 0);
    h2d(g.order, ord.data(), sizeof(int) * n, 0);
    bt.mark("up_deg");

    g.res_perm = g.order;
    {
        // dense tensor-core path: graphs with >= 5% density (config 3), when A fits comfortably
        const int mode = static_cast<int>(option(OPT_DENSE));
        const double density = n > 1 ? static_cast<double>(nnz) / (static_cast<double>(n) * (n - 1)) : 0.0;
        size_t freeb = 0, totalb = 0;
        cudaMemGetInfo(&freeb, &totalb);
        const bool fits = dense_adjacency_bytes(static_cast<int>(n)) < freeb / 3;
        if (mode != 0 && fits && n >= 256 && (mode == 1 || (density >= 0.05 && n >= 4096))) {
            g.dense_A = static_cast<decltype(g.dense_A)>(graph_alloc(dense_adjacency_bytes(static_cast<int>(n))));
            build_dense_adjacency(g, g.dense_A, 0);
            CK(cudaDeviceSynchronize());
        }
    }
    if (static_cast<int>(n) <= kResidentMaxRows) {
        // relabelled CSR for the member-resident kernel: new id = rank in `order`,
        // each list padded to a multiple of 4 with the zero sentinel row n; per-row
        // (offset within its 1024-row chunk, degree) packed in 32 bits
        std::vector<int> inv(n);
        for (uint32_t r = 0; r < n; ++r) inv[ord[r]] = static_cast<int>(r);
        std::vector<int64_t> rrp(n + 1, 0);
        for (uint32_t r = 0; r < n; ++r) rrp[r + 1] = rrp[r] + ((deg[ord[r]] + 3) & ~3);
        // heavy rows: degree > 32 (warp-cooperative in the fp32 kernel), at most 1024
        static const int split = [] {
            const char* e = std::getenv("LCB_HEAVY_DEG");
            return e ? std::atoi(e) : 32;  // swept 16..192 on B200: 32 best with 8-lane groups
        }();
        int H = 0;
        while (H < static_cast<int>(n) && H < 1024 && deg[ord[H]] > split) ++H;  // 8 rows per subgroup max
        const uint32_t L = n - H;
        const uint32_t chunks = (L + 1023) / 1024 + 1;
        std::vector<int> cbase(chunks, 0);
        std::vector<uint32_t> info(std::max<uint32_t>(L, 1));
        std::vector<int> hinfo(2 * std::max(H, 1));
        for (int h = 0; h < H; ++h) {
            hinfo[2 * h] = static_cast<int>(rrp[h] / 4);
            hinfo[2 * h + 1] = deg[ord[h]];
        }
        // light row i: (absolute 4-column word << 8) | degree  (degree <= 255, word < 2^24)
        bool packable = rrp[n] / 4 < (int64_t(1) << 24);
        for (uint32_t i = 0; i < L && packable; ++i) {
            const uint32_t r = H + i;
            if (i % 1024 == 0) cbase[i / 1024] = static_cast<int>(rrp[r] / 4);
            const int d = deg[ord[r]];
            if (d > 255) packable = false;
            info[i] = (static_cast<uint32_t>(rrp[r] / 4) << 8) | static_cast<uint32_t>(d);
        }
        if (packable) {
            std::vector<uint16_t> rcol(static_cast<size_t>(std::max<int64_t>(rrp[n], 4)), static_cast<uint16_t>(n));
            for (uint32_t r = 0; r < n; ++r) {
                const int v = ord[r];
                int64_t o = rrp[r];
                for (int64_t k = off[v]; k < off[v + 1]; ++k) rcol[static_cast<size_t>(o++)] = static_cast<uint16_t>(inv[adj[k]]);
            }
            // fp32 copy with a bank-balanced neighbour order: the 32 light rows of a warp
            // gather their p-th neighbours in the same LDS instruction, and an 8-byte slot s
            // sits in bank pair s mod 16, so the wavefront count of that instruction is the
            // largest number of distinct slots in one bank pair.  A greedy pass picks each
            // row's p-th neighbour from its remaining ones to keep that maximum low
            // (BA 10k: 4.10 -> 3.01 on average).  fp32 only: the fp64 path keeps CSR order
            // for bit-exact sums (graph.cpp:118).
            // LCB_BANK_ORDER: 0 CSR order, 1 balance the whole warp's 32 gathers over the 16
            // bank pairs, 2 (default) balance each half-warp (rows 0-15 / 16-31 of the group:
            // an 8-byte LDS is served per half-warp, 16 lanes x 8 B = one 128-byte wavefront).
            const int bank_order = static_cast<int>(option(OPT_BANK_ORDER));
            std::vector<uint16_t> fast;
            if (bank_order) {
                fast = rcol;
                std::vector<std::vector<uint16_t>> rem(32);
                std::vector<int> idx;
                idx.reserve(32);
                std::vector<int> stamp2(2 * (static_cast<size_t>(n) + 1), -1);  // slot already gathered in this step (per half)
                int step_id = 0;
                for (uint32_t b0 = static_cast<uint32_t>(H); b0 < n; b0 += 32) {
                    const uint32_t b1 = std::min<uint32_t>(b0 + 32, n);
                    const int rows = static_cast<int>(b1 - b0);
                    int L = 0;
                    for (int i = 0; i < rows; ++i) {
                        const uint32_t r = b0 + static_cast<uint32_t>(i);
                        const int d = deg[ord[r]];
                        rem[i].assign(rcol.begin() + rrp[r], rcol.begin() + rrp[r] + d);
                        L = std::max(L, d);
                    }
                    for (int p = 0; p < L; ++p, ++step_id) {
                        int cnt2[2][16] = {{0}};
                        idx.clear();
                        for (int i = 0; i < rows; ++i)
                            if (!rem[i].empty()) idx.push_back(i);
                        std::stable_sort(idx.begin(), idx.end(),
                                         [&](int x, int y) { return rem[x].size() < rem[y].size(); });
                        for (int i : idx) {
                            const int half = bank_order == 2 ? (i >> 4) : 0;
                            int* cnt = cnt2[half];
                            int* stamp = stamp2.data() + static_cast<size_t>(half) * (n + 1);
                            const int sid = step_id;
                            int bj = 0, bc = 1 << 30;
                            for (int j = 0; j < static_cast<int>(rem[i].size()); ++j) {
                                const uint16_t u = rem[i][j];
                                const int c = stamp[u] == sid ? -1 : cnt[u & 15];
                                if (c < bc) {
                                    bc = c;
                                    bj = j;
                                }
                            }
                            const uint16_t u = rem[i][bj];
                            rem[i].erase(rem[i].begin() + bj);
                            fast[static_cast<size_t>(rrp[b0 + i] + p)] = u;
                            if (bc >= 0) {
                                stamp[u] = sid;
                                ++cnt[u & 15];
                            }
                        }
                    }
                }
            }
            const int refine_passes = static_cast<int>(std::max<int64_t>(0, option(OPT_BANK_REFINE)));  // 0 disables
            if (!fast.empty() && refine_passes > 0 && bank_order == 2)
                refine_bank_order(fast, rrp, static_cast<uint32_t>(H), n, refine_passes);
            g.res_info = static_cast<decltype(g.res_info)>(graph_alloc(sizeof(uint32_t) * info.size()));
            g.res_chunk = static_cast<decltype(g.res_chunk)>(graph_alloc(sizeof(int) * chunks));
            g.res_heavy = static_cast<decltype(g.res_heavy)>(graph_alloc(sizeof(int) * hinfo.size()));
            g.res_col = static_cast<decltype(g.res_col)>(graph_alloc(sizeof(uint16_t) * rcol.size()));
            h2d(g.res_info, info.data(), sizeof(uint32_t) * info.size(), 0);
            h2d(g.res_chunk, cbase.data(), sizeof(int) * chunks, 0);
            h2d(g.res_heavy, hinfo.data(), sizeof(int) * hinfo.size(), 0);
            g.res_nheavy = H;
            h2d(g.res_col, rcol.data(), sizeof(uint16_t) * rcol.size(), 0);
            g.res_len = static_cast<int64_t>(rcol.size());
            if (!fast.empty()) {
                g.res_col_fast = static_cast<decltype(g.res_col_fast)>(graph_alloc(sizeof(uint16_t) * fast.size()));
                h2d(g.res_col_fast, fast.data(), sizeof(uint16_t) * fast.size(), 0);
            }
        }
    }
}

template <class T>
const T* deg_of(const DevGraph& g);
template <>
const float* deg_of<float>(const DevGraph& g) { return g.deg32; }
template <>
const double* deg_of<double>(const DevGraph& g) { return g.deg64; }

// ---------------------------------------------------------------------------
// NCCL, resolved at run time from the process's libnccl.so.2 (torch's when loaded)
// ---------------------------------------------------------------------------
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    // row-sharded ascent (all-gather of row ranges as grouped broadcasts)
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = dlerror();
            return a;
        }
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(dlsym(h, "ncclBroadcast"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.CommDestroy && a.GetErrorString;
        if (!a.ok) a.why = "libnccl.so.2 lacks required symbols";
        return a;
    }();
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(LCB_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace lcb

struct lcb_graph {
    lcb::DevGraph g;
};
namespace lcb {
// In-process exchange between ranks that are threads of one process (one GPU or several):
// the per-batch collectives of the solver (key / winner bits / error slots) go through
// device staging buffers and a host barrier; kernels never wait on one another.  The
// test / emulation backend of the multi-rank path on fewer GPUs than ranks.
struct LoopGroup {
    int nranks = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t gen = 0;
    std::vector<void*> slot;  // rank r's contribution, on rank r's device
    std::vector<size_t> cap;
    std::vector<int> dev;
    explicit LoopGroup(int n) : nranks(n), slot(static_cast<size_t>(n), nullptr), cap(static_cast<size_t>(n), 0),
                                dev(static_cast<size_t>(n), 0) {}
    ~LoopGroup() {
        for (int r = 0; r < nranks; ++r)
            if (slot[static_cast<size_t>(r)]) {
                cudaSetDevice(dev[static_cast<size_t>(r)]);
                cudaFree(slot[static_cast<size_t>(r)]);
            }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const int64_t g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
}  // namespace lcb

struct lcb_loopback {
    lcb::LoopGroup g;
    explicit lcb_loopback(int n) : g(n) {}
};

struct lcb_comm {
    ncclComm_t comm = nullptr;
    lcb::LoopGroup* loop = nullptr;
    int nranks = 1;
    int rank = 0;
    int device = 0;
    void* gather = nullptr;  // loopback: local copies of every rank's contribution
    size_t gather_cap = 0;
    ~lcb_comm() {
        if (gather) {
            cudaSetDevice(device);
            cudaFree(gather);
        }
    }
};

namespace lcb {
bool comm_active(const lcb_comm* c) { return c && (c->comm || c->loop); }

// In-place allreduce of `count` u32 / u64 words on the solver stream.
void comm_allreduce(lcb_comm* c, void* buf, size_t count, int bytes, bool is_max, cudaStream_t st, const char* what) {
    if (!comm_active(c) || count == 0) return;
    if (c->comm) {
        nccl_check(nccl().AllReduce(buf, buf, count, bytes == 8 ? ncclUint64 : ncclUint32, is_max ? ncclMax : ncclMin,
                                    c->comm, st),
                   what);
        return;
    }
    LoopGroup& g = *c->loop;
    const size_t nb = count * static_cast<size_t>(bytes);
    const size_t r = static_cast<size_t>(c->rank);
    if (g.cap[r] < nb) {  // only rank r touches its slot outside the barriers
        if (g.slot[r]) cudaFree(g.slot[r]);
        g.slot[r] = nullptr;
        g.cap[r] = 0;
        CK(cudaMalloc(&g.slot[r], nb));
        g.cap[r] = nb;
        g.dev[r] = c->device;
    }
    CK(cudaMemcpyAsync(g.slot[r], buf, nb, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    g.barrier();
    if (c->gather_cap < nb * static_cast<size_t>(g.nranks)) {
        if (c->gather) cudaFree(c->gather);
        c->gather = nullptr;
        c->gather_cap = 0;
        CK(cudaMalloc(&c->gather, nb * static_cast<size_t>(g.nranks)));
        c->gather_cap = nb * static_cast<size_t>(g.nranks);
    }
    for (int q = 0; q < g.nranks; ++q)
        CK(cudaMemcpyPeerAsync(static_cast<char*>(c->gather) + nb * static_cast<size_t>(q), c->device,
                               g.slot[static_cast<size_t>(q)], g.dev[static_cast<size_t>(q)], nb, st));
    launch_reduce_rows(c->gather, g.nranks, count, bytes, is_max, buf, st);
    CK(cudaStreamSynchronize(st));
    g.barrier();  // every rank has read every slot before any slot is rewritten
}

// All-gather of row ranges of a node-major buffer: rank q owns rows [range[2q], range[2q+1])
// of `base` (row_bytes each) and every rank ends with every range.  NCCL: one broadcast per
// root inside a group; loopback: device staging + host barriers.
void comm_allgather_rows(lcb_comm* c, void* base, size_t row_bytes, const std::vector<int64_t>& range,
                         cudaStream_t st) {
    if (!comm_active(c)) return;
    char* b = static_cast<char*>(base);
    if (c->comm) {
        if (!nccl().Broadcast || !nccl().GroupStart || !nccl().GroupEnd)
            fail(LCB_CUDA, "libnccl.so.2 lacks ncclBroadcast / ncclGroupStart / ncclGroupEnd");
        nccl_check(nccl().GroupStart(), "ncclGroupStart");
        for (int q = 0; q < c->nranks; ++q) {
            const int64_t r0 = range[static_cast<size_t>(2 * q)], r1 = range[static_cast<size_t>(2 * q + 1)];
            if (r1 > r0) {
                char* p = b + static_cast<size_t>(r0) * row_bytes;
                nccl_check(nccl().Broadcast(p, p, static_cast<size_t>(r1 - r0) * row_bytes, ncclUint8, q, c->comm, st),
                           "ncclBroadcast(rows)");
            }
        }
        nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
        return;
    }
    LoopGroup& g = *c->loop;
    const size_t r = static_cast<size_t>(c->rank);
    const int64_t r0 = range[2 * r], r1 = range[2 * r + 1];
    const size_t nb = static_cast<size_t>(r1 - r0) * row_bytes;
    if (g.cap[r] < nb) {
        if (g.slot[r]) cudaFree(g.slot[r]);
        g.slot[r] = nullptr;
        g.cap[r] = 0;
        CK(cudaMalloc(&g.slot[r], nb));
        g.cap[r] = nb;
        g.dev[r] = c->device;
    }
    if (nb) CK(cudaMemcpyAsync(g.slot[r], b + static_cast<size_t>(r0) * row_bytes, nb, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    g.barrier();
    for (int q = 0; q < g.nranks; ++q) {
        if (q == c->rank) continue;
        const int64_t q0 = range[static_cast<size_t>(2 * q)], q1 = range[static_cast<size_t>(2 * q + 1)];
        if (q1 > q0)
            CK(cudaMemcpyPeerAsync(b + static_cast<size_t>(q0) * row_bytes, c->device, g.slot[static_cast<size_t>(q)],
                                   g.dev[static_cast<size_t>(q)], static_cast<size_t>(q1 - q0) * row_bytes, st));
    }
    CK(cudaStreamSynchronize(st));
    g.barrier();
}
}  // namespace lcb

namespace lcb {

// ---------------------------------------------------------------------------
// per-solve device workspace
// ---------------------------------------------------------------------------
template <class T>
struct Work {
    int device = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int64_t ld = 0;
    DBuf<T> X[2], V, Y;
    DBuf<T> alpha;
    DBuf<int> tlim;
    DBuf<uint32_t> flags;
    DBuf<unsigned long long> err, cuts, keys;
    DBuf<unsigned long long> dcut;               // dense path: per-member sum_v s_v (A s)_v (cut pass)
    unsigned long long* dense_cut_req = nullptr;  // set by run_batch: fill it if K3 runs (l = 1)
    bool dense_cut_done = false;
    DBuf<uint32_t> Z;
    DBuf<uint64_t> mkeys, colkeys;
    DBuf<double> mean, dtrace, hostbatch;
    DBuf<int8_t> sign;
    DBuf<uint8_t> sgn;           // K1 saturation codes, one set per X buffer
    DBuf<unsigned> tile_ctr;     // K1s dynamic tile counters [2]
    int64_t stream_seq = 0;      // K1s launches on this workspace (counter parity)
    DBuf<float> dXm, dVm;        // dense path: member-major iterate / velocity of one column chunk
    DBuf<uint16_t> dplanes;      // dense path: 2 x 3 bf16 planes + K-step flags
    DBuf<float> dpartial;        // dense path: split-K partial sums of the tail tiles
    DBuf<uint32_t> win, recenter, pbest, gbest, carry, scratch_bits;
    DBuf<uint32_t> orbits;       // row-sharded ascent: early-exit bits, one array per bit
    DBuf<int> rs_row_ptr, rs_col, rs_order;  // row-sharded ascent: this rank's rows, global ids
    DBuf<T> rs_deg;
    DBuf<uint64_t> bf;           // exhaustive scan: masks, upper masks, degrees, block records
    unsigned long long* h_keys = nullptr;  // pinned
    uint32_t* h_flags = nullptr;
    size_t h_flags_cap = 0;
    // measurement
    double step_ms = 0.0;
    int64_t step_launches = 0;
    double step_bytes = 0.0;
    int64_t node_updates = 0;
    int64_t resident_iters = 0;  // iterations executed by the member-resident kernel
    double kstats[12] = {0};  // K1 / K2 {ms, launches, bytes}, K3 {ms, launches, flops}, K1s {ms, launches, bytes}

    explicit Work(int dev) : device(dev) {
        CK(cudaSetDevice(dev));
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        CK(cudaEventCreate(&ev0));
        CK(cudaEventCreate(&ev1));
        CK(cudaMallocHost(&h_keys, sizeof(unsigned long long) * 1024));
    }
    ~Work() {
        if (st) cudaStreamSynchronize(st);
        if (h_keys) cudaFreeHost(h_keys);
        if (h_flags) cudaFreeHost(h_flags);
        if (h_stage) cudaFreeHost(h_stage);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (st) cudaStreamDestroy(st);
    }
    void shape(int n, int W) {
        // rows padded to the K1 warp span and to the 1 KB K1s slab
        const int span = std::max(step_span<T>(W), stream_slab_cols(static_cast<int>(sizeof(T))));
        ld = ((static_cast<int64_t>(W) + span - 1) / span) * span;
        const size_t cells = static_cast<size_t>(n) * static_cast<size_t>(ld);
        X[0].ensure(cells);
        X[1].ensure(cells);
        V.ensure(cells);
    }
    double* h_stage = nullptr;  // pinned host staging of host-generated batches
    size_t h_stage_cap = 0;
    double* host_stage(size_t k) {
        if (k > h_stage_cap) {
            if (h_stage) cudaFreeHost(h_stage);
            h_stage = nullptr;
            h_stage_cap = 0;
            CK(cudaMallocHost(&h_stage, sizeof(double) * k));
            h_stage_cap = k;
        }
        return h_stage;
    }
    uint32_t* host_flags(size_t k) {
        if (k > h_flags_cap) {
            if (h_flags) cudaFreeHost(h_flags);
            CK(cudaMallocHost(&h_flags, sizeof(uint32_t) * k));
            h_flags_cap = k;
        }
        return h_flags;
    }
};

// Workspaces are pooled per (device, precision): a solve takes one, returns it on exit,
// so repeated solves (bench steps, per-component solves, service use) reuse the
// stream, events, pinned staging and device buffers instead of re-allocating them.
template <class T>
struct WorkPool {
    std::mutex mu;
    std::vector<std::unique_ptr<Work<T>>> free_list;
    static WorkPool& get() {
        static WorkPool p;
        return p;
    }
};

template <class T>
struct PooledWork {
    std::unique_ptr<Work<T>> w;
    explicit PooledWork(int device) {
        auto& p = WorkPool<T>::get();
        {
            std::lock_guard<std::mutex> lk(p.mu);
            for (size_t i = 0; i < p.free_list.size(); ++i)
                if (p.free_list[i]->device == device) {
                    w = std::move(p.free_list[i]);
                    p.free_list.erase(p.free_list.begin() + static_cast<std::ptrdiff_t>(i));
                    break;
                }
        }
        if (!w) w = std::make_unique<Work<T>>(device);
        w->step_ms = 0.0;
        w->step_launches = 0;
        w->step_bytes = 0.0;
        w->node_updates = 0;
        w->resident_iters = 0;
        for (double& k : w->kstats) k = 0.0;
    }
    ~PooledWork() {
        if (!w) return;
        cudaStreamSynchronize(w->st);
        auto& p = WorkPool<T>::get();
        std::lock_guard<std::mutex> lk(p.mu);
        p.free_list.push_back(std::move(w));
    }
    Work<T>& operator*() { return *w; }
};

// Kernel choice measured on B200 (profiles/round1_kernel_ab.md): the member-resident
// kernel wins when the on-chip slab covers the graph and the batch is wide enough to
// fill several waves (W >= 1024 columns at K=2, any W for fp64 / small graphs).
// fp32 takes K2 whenever the slab fits, at any batch width: K2 sums each row in its own
// (bank-balanced) neighbour order, so choosing the kernel by W would make a member's fp32
// trajectory depend on the batch width and the rank count (test_ascent.cpp:110-136).
// fp64 has no such constraint (every kernel is bit-exact): K2 holds one fp64 column per CTA
// and stays near 7e10 node-updates/s at any width, while K1s grows with the batch, so fp64
// streams once n * W >= 2e6 (measured on BA n = 2k / 5k / 10k, W = 256 .. 2048: config 2 at
// W = 1024 137 -> 64 us per iteration; profiles/round2_k1s.md).
bool resident_preferred(const DevGraph& g, int W, size_t elem) {
    const int64_t mode = option(OPT_RESIDENT);  // -1 auto, 0 never, 1 always (when it fits)
    if (mode == 1) return true;
    if (mode == 0) return false;
    if (elem == 8 && static_cast<int64_t>(g.n) * W >= 2000000) return false;
    return true;
}

struct IterResult {
    unsigned long long err = ~0ull;             // slot 0 (whole batch unless segmented)
    std::vector<unsigned long long> errs;        // one per error slot
    int final_buf = 0;
    int64_t iters = 0;
};

// The T-loop of ascend (ascent.cpp:58-94) over a device-resident [n][ld] batch
// whose iterate is in X[0] and velocity in V (already initialised).
template <class T>
IterResult run_iterations(const DevGraph& g, Work<T>& w, int W, int members, int l, int64_t iters,
                          T alpha_u, const T* alpha_arr, const int* tlim_arr, T mu, bool ee,
                          double* trace_host /* [iters][members] or null */, int err_seg = 0,
                          const std::vector<int64_t>* seg_iters = nullptr /* per err segment, descending */) {
    const int err_slots = err_seg > 0 ? (members + err_seg - 1) / err_seg : 1;
    StepArgs<T> a{};
    a.row_ptr = g.row_ptr;
    a.col = g.col;
    a.deg = deg_of<T>(g);
    a.order = g.order;
    a.vel = w.V.p;
    a.ld = w.ld;
    a.n = g.n;
    a.W = W;
    a.l = l;
    a.alpha = alpha_arr;
    a.tlim = tlim_arr;
    a.members = members;
    a.mu = mu;
    a.alpha_uniform = alpha_u;
    a.err = w.err.ensure(static_cast<size_t>(err_slots));
    a.err_seg = err_seg;
    CK(cudaMemsetAsync(a.err, 0xff, sizeof(unsigned long long) * err_slots, w.st));
    if (static_cast<size_t>(err_slots) > 1024) fail(LCB_VALIDATION, "too many error slots");
    uint32_t* F = nullptr;
    if (ee) {
        F = w.flags.ensure(static_cast<size_t>(3) * members);
        CK(cudaMemsetAsync(F, 0, sizeof(uint32_t) * 3 * members, w.st));
    }
    if (trace_host) w.Y.ensure(static_cast<size_t>(g.n) * w.ld);
    double* dtr = trace_host ? w.dtrace.ensure(members) : nullptr;

    IterResult r;
    int K = 0;
    const bool resident_enabled = true;
    if constexpr (std::is_same_v<T, float>) {
        if (g.dense_A && !trace_host && !ee && iters > 0 && iters <= 0x7fffffff) {
            // K3: dense adjacency on the tensor cores, column chunks of <= 256
            CK(cudaEventRecord(w.ev0, w.st));
            const int ldp = dense_ldp(g.n);
            for (int c0 = 0; c0 < W; c0 += 256) {
                const int Wc = std::min(256, W - c0);
                float* Xm = w.dXm.ensure(static_cast<size_t>(Wc) * ldp);
                float* Vm = w.dVm.ensure(static_cast<size_t>(Wc) * ldp);
                void* P = w.dplanes.ensure((dense_planes_bytes(g.n, Wc) + 1) / 2);
                // tlim/alpha are per member; chunk boundaries are member-aligned when 256 % l == 0
                int64_t chunk_iters = iters;
                if (seg_iters && err_seg > 0) {  // segments in descending T: the chunk's first one is the longest
                    const size_t seg = static_cast<size_t>(c0 / (err_seg * l));
                    if (seg < seg_iters->size()) chunk_iters = (*seg_iters)[seg];
                }
                float* part = w.dpartial.ensure(dense_partial_floats());
                unsigned long long* cs = w.dense_cut_req && l == 1 ? w.dense_cut_req + c0 : nullptr;
                run_dense_iterations(g, g.dense_A, w.X[0].p + c0, w.X[1].p + c0, w.ld, Wc, l, chunk_iters, alpha_u,
                                     alpha_arr, tlim_arr, mu, a.err, err_seg, Xm, Vm, P, w.st, c0, part, cs);
                w.dense_cut_done = cs != nullptr;
            }
            CK(cudaEventRecord(w.ev1, w.st));
            CK(cudaGetLastError());
            d2h(w.h_keys, a.err, sizeof(unsigned long long) * err_slots, w.st);
            CK(cudaStreamSynchronize(w.st));
            r.err = w.h_keys[0];
            r.errs.assign(w.h_keys, w.h_keys + err_slots);
            r.iters = iters;
            r.final_buf = 1;
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
            w.step_ms += ms;
            w.step_launches += iters * ((W + 255) / 256);
            const double bytes = static_cast<double>(iters) * (16.0 * g.n * W + 4.0 * g.nnz + 4.0 * (g.n + 1));
            w.step_bytes += bytes;
            w.kstats[6] += ms;
            w.kstats[7] += static_cast<double>(iters * ((W + 255) / 256));
            w.kstats[8] += 2.0 * static_cast<double>(g.n) * g.n * W * iters;  // algorithmic GEMM flops
            w.node_updates += iters * static_cast<int64_t>(g.n) * W;
            return r;
        }
    }
    if (resident_enabled && !trace_host && g.res_info && iters > 0 && resident_preferred(g, W, sizeof(T)) && iters <= 0x7fffffff &&
        resident_fits(g.n, W, l, ee, static_cast<int>(sizeof(T)), K)) {
        // K2: all iterations in one launch, state resident in SMEM
        ResidentArgs ra{};
        ra.rowinfo = g.res_info;
        ra.chunk_base = g.res_chunk;
        ra.heavy_info = g.res_heavy;
        ra.heavy = g.res_nheavy;
        ra.col = (sizeof(T) == 4 && g.res_col_fast) ? g.res_col_fast : g.res_col;
        ra.perm = g.res_perm;
        ra.X = w.X[0].p;
        ra.ld = w.ld;
        ra.n = g.n;
        ra.W = W;
        ra.l = l;
        ra.T = static_cast<int>(iters);
        ra.alpha_uniform = static_cast<float>(alpha_u);
        ra.mu = static_cast<float>(mu);
        ra.alpha_uniform64 = static_cast<double>(alpha_u);
        ra.mu64 = static_cast<double>(mu);
        ra.alpha = alpha_arr;
        ra.tlim = tlim_arr;
        ra.err = a.err;
        ra.err_seg = err_seg;
        CK(cudaEventRecord(w.ev0, w.st));
        const int res_launches = launch_resident(ra, K, ee, static_cast<int>(sizeof(T)), w.st);
        CK(cudaEventRecord(w.ev1, w.st));
        CK(cudaGetLastError());
        d2h(w.h_keys, a.err, sizeof(unsigned long long) * err_slots, w.st);
        CK(cudaStreamSynchronize(w.st));
        r.err = w.h_keys[0];
        r.errs.assign(w.h_keys, w.h_keys + err_slots);
        r.iters = iters;
        r.final_buf = 0;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
        w.step_ms += ms;
        w.step_launches += res_launches;
        const double bytes = static_cast<double>(iters) *
                             (4.0 * sizeof(T) * static_cast<double>(g.n) * W + 4.0 * g.nnz + 4.0 * (g.n + 1));
        w.step_bytes += bytes;
        w.kstats[3] += ms;
        w.kstats[4] += res_launches;
        w.kstats[5] += bytes;
        w.node_updates += iters * static_cast<int64_t>(g.n) * W;
        w.resident_iters += iters;
        return r;
    }
    // K1n, L2-panel member chunking (SURVEY 7 "throughput kernels"): when the iterate is
    // far larger than L2, run all T iterations on one narrow column panel at a time,
    // copied into a contiguous [n][P] buffer so the panel that the gathers read deg
    // times per iteration stays L2-resident (lcb_narrow.cu).  Velocity starts at zero
    // (ascent.cpp:57) and is not needed afterwards.
    {
        static const int64_t l2 = [] {
            int v = 0;
            cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, 0);
            return static_cast<int64_t>(v > 0 ? v : (126 << 20));
        }();
        // 0 never (default), 1 always, -1 auto (iterate > 2 x L2 and the panel pair fits).
        // Off by default: on config 4 (ER 1M, W=512) the panel kernel is latency-bound at
        // 5.5 ms/iteration vs 4.46 ms for K1 (profiles/round1_narrow.md).
        const int64_t chunk_mode = option(OPT_CHUNK);
        const int P = narrow_panel_cols(static_cast<int>(sizeof(T)));
        const int64_t panel = static_cast<int64_t>(g.n) * W * static_cast<int64_t>(sizeof(T));
        const int64_t narrow = static_cast<int64_t>(g.n) * P * static_cast<int64_t>(sizeof(T));
        const bool want = chunk_mode == 1 || (chunk_mode != 0 && panel > 2 * l2 && narrow * 3 <= l2);
        if (want && !ee && !trace_host && iters > 0 && iters <= 0x7fffffff) {
            const size_t cells = static_cast<size_t>(g.n) * P;
            T* P0 = w.Y.ensure(3 * cells);
            CK(cudaEventRecord(w.ev0, w.st));
            int64_t launches = 0;
            double updates = 0.0;
            // degree order only pays for skewed graphs (warps then hold rows of equal
            // degree); otherwise it is one more dependent load per row
            StepArgs<T> na = a;
            if (static_cast<double>(g.max_degree) <= 4.0 * g.deg_mean + 16.0) na.order = nullptr;
            for (int c0 = 0; c0 < W; c0 += P) {
                const int wc = std::min(P, W - c0);
                int64_t pit = iters;
                if (seg_iters && err_seg > 0) {  // descending T: the panel's first segment is its longest
                    const size_t seg = static_cast<size_t>(c0 / (err_seg * l));
                    if (seg < seg_iters->size()) pit = (*seg_iters)[seg];
                }
                run_narrow_panel<T>(na, w.X[0].p, w.X[1].p, w.ld, c0, wc, pit, P0, P0 + cells, P0 + 2 * cells,
                                    w.st);
                launches += pit + 2;
                updates += static_cast<double>(pit) * g.n * wc;
            }
            CK(cudaEventRecord(w.ev1, w.st));
            CK(cudaGetLastError());
            d2h(w.h_keys, a.err, sizeof(unsigned long long) * err_slots, w.st);
            CK(cudaStreamSynchronize(w.st));
            r.err = w.h_keys[0];
            r.errs.assign(w.h_keys, w.h_keys + err_slots);
            r.iters = iters;
            r.final_buf = 1;
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
            const double panels = static_cast<double>((W + P - 1) / P);
            w.step_ms += ms;
            w.step_launches += launches;
            const double bytes = static_cast<double>(iters) *
                                 (4.0 * sizeof(T) * static_cast<double>(g.n) * W + panels * (4.0 * g.nnz + 4.0 * (g.n + 1)));
            w.step_bytes += bytes;
            w.kstats[0] += ms;
            w.kstats[1] += static_cast<double>(launches);
            w.kstats[2] += bytes;
            w.node_updates += static_cast<int64_t>(updates);
            return r;
        }
    }
    // K1 saturation codes (StepArgs::sgn_*): written every iteration, read from the second
    // on; one warp span (S = 1) per slab.  They pay only when the gathers miss L2: config 4
    // (2 GB iterate) 4.44 -> 3.71 ms/iteration; with an L2-resident iterate the extra
    // dependent code load makes K1 slower (config 5: 169.6 -> 172.8 us, config 2 W=1024:
    // 51.2 -> 62.0 us; profiles/round1_kernel_ab.md).  LCB_SIGNREC=0 never, 1 always,
    // default: iterate buffer larger than L2.
    const int64_t signrec = option(OPT_SIGNREC);
    // K1s (lcb_stream.cu), the warp-specialised streaming step: LCB_STREAM=0 keeps K1
    const int64_t stream_mode = option(OPT_STREAM);
    const int sspan = stream_slab_cols(static_cast<int>(sizeof(T)));  // one 1 KB slab
    const int nslabs = (W + sspan - 1) / sspan;
    // slab-outer order (all iterations of one slab before the next: members are independent,
    // ascent.cpp:52, so the slab's codes stay L2-resident across iterations) unless early exit
    // needs every column of a member in the same launch
    // ... and only when the codes of all slabs would not stay in L2 anyway (config 4: 4 x 32 MB;
    // config 5: 2 x 3.2 MB -> one launch per iteration over both slabs, twice the tiles per launch)
    static const int64_t l2b = [] {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, 0);
        return static_cast<int64_t>(v > 0 ? v : (126 << 20));
    }();
    const int64_t so = option(OPT_SLAB_OUTER);
    // (a trace needs every column after every iteration: iteration-major then)
    const bool slab_outer = (!ee || sspan % l == 0) && nslabs > 1 && !trace_host &&
                            (so == 1 || (so < 0 && static_cast<int64_t>(g.n) * 32 * nslabs * 2 > l2b / 2));
    // default 1: K1s for every streaming step (config 4: 1.83 vs 3.6 ms/iteration, config 5:
    // 148 vs 166 us); -1: K1s only where the slab-major order is needed
    const bool use_stream = (stream_mode == 1 || (stream_mode < 0 && slab_outer)) &&
                            w.ld % sspan == 0 &&
                            static_cast<int64_t>(g.n) * 36 * (slab_outer ? 1 : nslabs) < (int64_t(1) << 32);
    static const int64_t l2_bytes = [] {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, 0);
        return static_cast<int64_t>(v > 0 ? v : (126 << 20));
    }();
    uint8_t* codes[2] = {nullptr, nullptr};
    const int span = step_span<T>(W);
    const bool codes_on = use_stream || signrec == 1 ||
                          (signrec != 0 && static_cast<int64_t>(g.n) * w.ld * static_cast<int64_t>(sizeof(T)) > l2_bytes);
    if (use_stream || (codes_on && span == 32 * static_cast<int>(16 / sizeof(T)) && w.ld % span == 0)) {
        // K1: [n][sgn_ld] interleaved; K1s: [slabs][n][32] sign bytes + [slabs][n] u32 flags
        // (one slab when slab-outer)
        a.sgn_ld = (w.ld / span) * 32;
        // second buffer 256-byte aligned (K1s copies 16-byte code lines with cp.async)
        const size_t bytes = ((use_stream ? static_cast<size_t>(g.n) * 36 * (slab_outer ? 1 : nslabs)
                                          : static_cast<size_t>(g.n) * static_cast<size_t>(a.sgn_ld)) + 255) & ~size_t(255);
        a.flag_off = static_cast<int64_t>(g.n) * 32 * (slab_outer ? 1 : nslabs);
        codes[0] = w.sgn.ensure(2 * bytes);
        codes[1] = codes[0] + bytes;
    }
    if (use_stream) {
        if (!w.tile_ctr.p) {
            w.tile_ctr.ensure(2);
            CK(cudaMemsetAsync(w.tile_ctr.p, 0, 2 * sizeof(unsigned), w.st));
            w.stream_seq = 0;
        }
        a.tile_ctr = w.tile_ctr.p;
        // x-code mode (OPT_XCODE): row slabs on the box corners are stored as their sign codes
        // only, X is completed by launch_xcode_fill after a slab's (or the run's) last
        // iteration.  Not with per-segment stop iterations: a stopped segment's X must stay
        // complete while later iterations overwrite the codes.
        a.xskip = (option(OPT_XCODE) != 0 && !seg_iters && !trace_host) ? 1 : 0;  // a trace reads X
    }
    if (use_stream && slab_outer) {
        // ---- K1s, slab-outer: for each 512-byte column slab, all its iterations
        CK(cudaEventRecord(w.ev0, w.st));
        std::vector<int64_t> slab_it(static_cast<size_t>(nslabs), 0);
        double updates = 0.0;
        int64_t launches = 0, it_max = 0;
        for (int sl = 0; sl < nslabs; ++sl) {
            const int c_lo = sl * sspan, c_hi = std::min(W, c_lo + sspan);
            int64_t ts = iters;
            if (seg_iters && err_seg > 0) {  // longest candidate among the slab's segments
                ts = 0;
                for (int c = c_lo; c < c_hi; c += err_seg * l)
                    ts = std::max(ts, (*seg_iters)[static_cast<size_t>(c / (err_seg * l))]);
                ts = std::max(ts, (*seg_iters)[static_cast<size_t>((c_hi - 1) / (err_seg * l))]);
            }
            const int m_lo = c_lo / l, m_hi = (c_hi - 1) / l + 1;  // members touching the slab
            if (ee) CK(cudaMemsetAsync(F, 0, sizeof(uint32_t) * 3 * members, w.st));
            int64_t t = 0;
            for (; t < ts; ++t) {
                a.x_in = w.X[t & 1].p;
                a.x_out = w.X[(t + 1) & 1].p;
                a.it = static_cast<int>(t);
                a.sgn_in = t > 0 ? codes[t & 1] : nullptr;
                a.sgn_out = codes[(t + 1) & 1];
                if (ee) {
                    a.flags_prev = F + ((t + 2) % 3) * members;
                    a.flags_cur = F + (t % 3) * members;
                    a.flags_zero = F + ((t + 1) % 3) * members;
                }
                a.launch_seq = w.stream_seq++;
                launch_stream<T>(a, sl, 1, ee, w.st);
                ++launches;
                if (ee && ((t + 1) % 32 == 0) && t + 1 < ts) {  // stop once the slab's members left
                    uint32_t* hf = w.host_flags(members);
                    d2h(hf, a.flags_cur, sizeof(uint32_t) * members, w.st);
                    CK(cudaStreamSynchronize(w.st));
                    bool any = false;
                    for (int m = m_lo; m < m_hi && !any; ++m) any = ex_continue(hf[m]);
                    if (!any && !tlim_arr) {
                        ++t;
                        break;
                    }
                }
            }
            if (a.xskip && t > 0) {
                launch_xcode_fill<T>(w.X[t & 1].p, w.ld, g.n, codes[t & 1], a.flag_off, sl, 1, w.st);
                ++w.step_launches;
            }
            slab_it[static_cast<size_t>(sl)] = t;
            it_max = std::max(it_max, t);
            updates += static_cast<double>(t) * g.n * (c_hi - c_lo);
        }
        // every slab's result into X[it_max & 1]
        for (int sl = 0; sl < nslabs; ++sl) {
            const int64_t t = slab_it[static_cast<size_t>(sl)];
            if ((t ^ it_max) & 1) {
                const size_t pitch = sizeof(T) * static_cast<size_t>(w.ld);
                CK(cudaMemcpy2DAsync(w.X[it_max & 1].p + static_cast<size_t>(sl) * sspan, pitch,
                                     w.X[t & 1].p + static_cast<size_t>(sl) * sspan, pitch, sizeof(T) * sspan,
                                     static_cast<size_t>(g.n), cudaMemcpyDeviceToDevice, w.st));
            }
        }
        CK(cudaEventRecord(w.ev1, w.st));
        CK(cudaGetLastError());
        d2h(w.h_keys, a.err, sizeof(unsigned long long) * err_slots, w.st);
        CK(cudaStreamSynchronize(w.st));
        r.err = w.h_keys[0];
        r.errs.assign(w.h_keys, w.h_keys + err_slots);
        r.iters = it_max;
        r.final_buf = static_cast<int>(it_max & 1);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
        w.step_ms += ms;
        w.step_launches += launches;
        const double bytes = 4.0 * sizeof(T) * updates +
                             static_cast<double>(launches) / std::max(1, nslabs) * (4.0 * g.nnz + 4.0 * (g.n + 1));
        w.step_bytes += bytes;
        w.kstats[9] += ms;
        w.kstats[10] += static_cast<double>(launches);
        w.kstats[11] += bytes;
        w.node_updates += static_cast<int64_t>(updates);
        return r;
    }
    CK(cudaEventRecord(w.ev0, w.st));
    int64_t it = 0;
    const int seg_cols = err_seg * l;
    size_t live_segs = seg_iters ? seg_iters->size() : 0;
    for (; it < iters; ++it) {
        a.x_in = w.X[it & 1].p;
        a.x_out = w.X[(it + 1) & 1].p;
        a.it = static_cast<int>(it);
        a.sgn_in = it > 0 ? codes[it & 1] : nullptr;
        a.sgn_out = codes[(it + 1) & 1];
        if (seg_iters) {  // candidates laid out by descending T: launch only the live prefix
            while (live_segs > 0 && (*seg_iters)[live_segs - 1] <= it) --live_segs;
            a.W = std::min(W, static_cast<int>(live_segs) * seg_cols);
        }
        if (ee) {
            a.flags_prev = F + ((it + 2) % 3) * members;
            a.flags_cur = F + (it % 3) * members;
            a.flags_zero = F + ((it + 1) % 3) * members;
        }
        if (use_stream)
        {
            a.launch_seq = w.stream_seq++;
            launch_stream<T>(a, 0, (a.W + sspan - 1) / sspan, ee, w.st);
        }
        else
            launch_step<T>(a, ee, MODE_STEP, w.st);
        if (trace_host) {
            // objective after the step: x'Lx per member (ascent.cpp:78-88)
            StepArgs<T> b = a;
            b.x_in = a.x_out;
            b.x_out = w.Y.p;
            b.sgn_in = nullptr;
            b.sgn_out = nullptr;
            launch_step<T>(b, false, MODE_LAPLACE, w.st);
            CK(cudaMemsetAsync(dtr, 0, sizeof(double) * members, w.st));
            launch_member_dot<T>(a.x_out, w.Y.p, g.n, W, l, w.ld, dtr, w.st);
            CK(cudaMemcpyAsync(trace_host + it * members, dtr, sizeof(double) * members,
                               cudaMemcpyDeviceToHost, w.st));
        }
        // Stop launching once every member has left (all later steps are copies).
        if (ee && ((it + 1) % 32 == 0) && it + 1 < iters) {
            uint32_t* hf = w.host_flags(members);
            d2h(hf, a.flags_cur, sizeof(uint32_t) * members, w.st);
            CK(cudaStreamSynchronize(w.st));
            bool any = false;
            for (int m = 0; m < members && !any; ++m) any = ex_continue(hf[m]);
            if (!any && !tlim_arr) {
                ++it;
                break;
            }
        }
    }
    if (use_stream && a.xskip && it > 0) {
        launch_xcode_fill<T>(w.X[it & 1].p, w.ld, g.n, codes[it & 1], a.flag_off, 0, nslabs, w.st);
        ++w.step_launches;
    }
    if (seg_iters) {
        // a segment that stopped at T_s left its final iterate in X[T_s & 1]
        for (size_t sgi = 0; sgi < seg_iters->size(); ++sgi) {
            const int64_t ts = (*seg_iters)[sgi];
            if (ts < it && ((ts ^ it) & 1)) {
                const size_t pitch = sizeof(T) * static_cast<size_t>(w.ld);
                CK(cudaMemcpy2DAsync(w.X[it & 1].p + sgi * seg_cols, pitch, w.X[ts & 1].p + sgi * seg_cols, pitch,
                                     sizeof(T) * static_cast<size_t>(seg_cols), static_cast<size_t>(g.n),
                                     cudaMemcpyDeviceToDevice, w.st));
            }
        }
    }
    CK(cudaEventRecord(w.ev1, w.st));
    CK(cudaGetLastError());
    d2h(w.h_keys, a.err, sizeof(unsigned long long) * err_slots, w.st);
    CK(cudaStreamSynchronize(w.st));
    r.err = w.h_keys[0];
    r.errs.assign(w.h_keys, w.h_keys + err_slots);
    r.iters = it;
    r.final_buf = static_cast<int>(it & 1);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
    w.step_ms += ms;
    w.step_launches += it;
    const double bytes = static_cast<double>(it) *
                         (4.0 * sizeof(T) * static_cast<double>(g.n) * W + 4.0 * g.nnz + 4.0 * (g.n + 1));
    w.step_bytes += bytes;
    const int ks = use_stream ? 9 : 0;
    w.kstats[ks] += ms;
    w.kstats[ks + 1] += static_cast<double>(it);
    w.kstats[ks + 2] += bytes;
    w.node_updates += it * static_cast<int64_t>(g.n) * W;
    return r;
}

std::string numeric_msg(int64_t it, int64_t member) {
    return "ascend: non-finite value at iteration " + std::to_string(it) + ", member " +
           std::to_string(member);
}

// ---------------------------------------------------------------------------
// solver (solver.cpp re-stated over device-resident batches)
// ---------------------------------------------------------------------------
struct Cand {
    double exponent = 0.0;
    int64_t iterations = 1;
    bool has_fit = false;
    double fitness = 0.0;
    double alpha() const { return std::pow(10.0, exponent); }
};

struct TraceSinks {
    lcb_batch_trace* bt;
    int64_t bt_cap;
    lcb_phase_trace* pt;
    int64_t pt_cap;
    lcb_search_trace* st;
    int64_t st_cap;
    int64_t nbt = 0, npt = 0, nst = 0;
};

template <class T>
struct Solver {
    const DevGraph& g;
    const lcb_config& cfg;
    Work<T>& w;
    TraceSinks& sinks;
    lcb_comm* comm;
    bool host_init;
    uint64_t base;
    lcb_trace_fn trace_fn = nullptr;
    void* trace_ctx = nullptr;
    bool batched_search = false;
    Clock::time_point t0 = Clock::now();
    int words_n;
    int64_t B;            // local members
    int64_t member_base;  // first global member of this rank

    bool has_best = false;
    int64_t best_cut = 0, best_serial = 0, best_member = 0;
    int64_t serial = 0;
    bool has_tuned[2] = {false, false};
    Cand tuned[2];
    int64_t main_batches[2] = {0, 0};
    uint64_t search_runs[2] = {0, 0};
    double init_s = 0, ascent_s = 0, rounding_s = 0, search_s = 0;

    Solver(const DevGraph& graph, const lcb_config& c, Work<T>& work, TraceSinks& s, lcb_comm* cm,
           bool hinit, uint64_t seed)
        : g(graph), cfg(c), w(work), sinks(s), comm(cm), host_init(hinit), base(seed) {
        words_n = (g.n + 31) / 32;
        B = cfg.batch_size;
        member_base = comm ? static_cast<int64_t>(comm->rank) * B : 0;
        for (auto* b : {&w.win, &w.recenter, &w.pbest, &w.gbest, &w.carry, &w.scratch_bits})
            b->ensure(words_n);
    }

    bool budget_gone() const {
        return cfg.time_budget_s > 0.0 && secs_since(t0) >= cfg.time_budget_s;
    }

    void copy_bits(uint32_t* dst, const uint32_t* src) {
        CK(cudaMemcpyAsync(dst, src, sizeof(uint32_t) * words_n, cudaMemcpyDeviceToDevice, w.st));
    }

    // With several ranks a non-finite value on one rank must stop every rank the same
    // way (the collectives that follow must match): min-reduce the error slots.
    void sync_errors(IterResult& ir) {
        if (!comm_active(comm)) return;
        const size_t slots = ir.errs.size();
        comm_allreduce(comm, w.err.p, slots, 8, false, w.st, "allreduce(err)");
        d2h(w.h_keys, w.err.p, sizeof(unsigned long long) * slots, w.st);
        CK(cudaStreamSynchronize(w.st));
        ir.errs.assign(w.h_keys, w.h_keys + slots);
        ir.err = ir.errs[0];
    }

    // member stream keys of batch serial `s` for the local members (init.cpp:80)
    void member_keys(int64_t s, std::vector<uint64_t>& out) const {
        const uint64_t bkey = split2(base, 0x6261u, static_cast<uint64_t>(s));
        for (int64_t j = 0; j < B; ++j) out.push_back(split2(bkey, 0x6d62u, static_cast<uint64_t>(member_base + j)));
    }

    // Host-side batch generation with glibc normals: gaussian_batch (init.cpp:69-87)
    // for the given member streams, identical bits to the reference.
    void host_batch(const std::vector<double>& mean, int l, const std::vector<uint64_t>& mkeys, double noise) {
        const int n = g.n;
        const size_t entries = static_cast<size_t>(n) * l;
        const size_t total = entries * mkeys.size();
        // members on host threads, as the reference's parallel_for over members (init.cpp:78-86);
        // each member's stream is independent, so the bits do not depend on the split
        double* vals = w.host_stage(total);
        auto gen = [&](size_t j0, size_t j1) {
            for (size_t j = j0; j < j1; ++j) {
                HostStream ms{mkeys[j]};
                double* o = vals + j * entries;
                for (size_t k = 0; k < entries; ++k) {
                    const double x = mean[k] + noise * ms.normal();
                    o[k] = x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x);
                }
            }
        };
        const size_t B = mkeys.size();
        const size_t nt = std::min<size_t>(B, std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
        if (nt <= 1 || total < (1u << 16)) {
            gen(0, B);
        } else {
            std::vector<std::thread> th;
            for (size_t t = 1; t < nt; ++t) th.emplace_back(gen, B * t / nt, B * (t + 1) / nt);
            gen(0, B / nt);
            for (auto& t : th) t.join();
        }
        double* d = w.hostbatch.ensure(total);
        h2d(d, vals, sizeof(double) * total, w.st);
        launch_transpose_in<T>(d, w.X[0].p, n, static_cast<int>(mkeys.size() * l), w.ld, w.st);
        CK(cudaMemsetAsync(w.V.p, 0, sizeof(T) * static_cast<size_t>(n) * w.ld, w.st));
        CK(cudaStreamSynchronize(w.st));  // the pinned stage is reused by the next batch
    }

    // batch init around a device mean or pm1(bits): glibc normals on the host or the
    // device Box-Muller kernel
    void init_batch(int l, const double* dmean, const uint32_t* bits, const std::vector<uint64_t>& mk,
                    double noise) {
        if (host_init) {
            host_batch(host_mean_from(dmean, bits, l), l, mk, noise);
        } else {
            uint64_t* dk = w.mkeys.ensure(mk.size());
            h2d(dk, mk.data(), sizeof(uint64_t) * mk.size(), w.st);
            launch_gaussian<T>(w.X[0].p, w.V.p, w.ld, g.n, static_cast<int>(mk.size()), l, dk, dmean, bits,
                               cfg.init_scale, noise, w.st);
            CK(cudaStreamSynchronize(w.st));  // mk is pageable
        }
    }

    std::vector<double> host_mean_from(const double* dmean, const uint32_t* bits, int l) {
        const int n = g.n;
        std::vector<double> mean(static_cast<size_t>(n) * l);
        if (dmean) {
            d2h(mean.data(), dmean, sizeof(double) * mean.size(), w.st);
            CK(cudaStreamSynchronize(w.st));
        } else {
            std::vector<uint32_t> hb(words_n);
            d2h(hb.data(), bits, sizeof(uint32_t) * words_n, w.st);
            CK(cudaStreamSynchronize(w.st));
            for (int v = 0; v < n; ++v)
                mean[v] = (((hb[v >> 5] >> (v & 31)) & 1u) ? 1.0 : -1.0) / cfg.init_scale;
            for (int c = 1; c < l; ++c) std::copy(mean.begin(), mean.begin() + n, mean.begin() + static_cast<size_t>(c) * n);
        }
        return mean;
    }

    struct BatchRes {
        int64_t cut, serial, member;
    };

    // run_batch — solver.cpp:106-143.  Mean: device [l][n] array (dmean) or
    // pm1_scaled(bits).  Winner assignment left in w.win.
    BatchRes run_batch(bool lifted, int l, const double* dmean, const uint32_t* bits, double alpha,
                       int64_t iters, double mu, bool ee, bool book) {
        const int n = g.n;
        const int64_t s = serial++;
        const double eta_eff = cfg.scale_noise ? cfg.eta / (cfg.init_scale * cfg.init_scale) : cfg.eta;
        const double noise = std::sqrt(eta_eff);
        const int W = static_cast<int>(B * l);
        w.shape(n, W);

        auto mark = Clock::now();
        std::vector<uint64_t> mk;
        member_keys(s, mk);
        init_batch(l, dmean, bits, mk, noise);
        if (book) init_s += secs_since(mark);

        mark = Clock::now();
        std::vector<double> tr;
        const bool tracing = book && trace_fn != nullptr;
        if (tracing) tr.assign(static_cast<size_t>(iters) * static_cast<size_t>(B), 0.0);
        // dense graphs, unlifted: K3 computes the cut counts with one more tensor-core pass
        w.dense_cut_done = false;
        w.dense_cut_req = g.dense_A && !lifted && l == 1 && option(OPT_DENSE_CUT) != 0 ? w.dcut.ensure(B) : nullptr;
        IterResult ir = run_iterations<T>(g, w, W, static_cast<int>(B), l, iters, static_cast<T>(alpha),
                                          nullptr, nullptr, static_cast<T>(mu), ee && !tracing,
                                          tracing ? tr.data() : nullptr);
        w.dense_cut_req = nullptr;
        sync_errors(ir);
        if (tracing)  // member-major, as the reference with workers=1 (ascent.cpp:52,87)
            for (int64_t j = 0; j < B; ++j)
                for (int64_t it = 0; it < iters; ++it)
                    trace_fn(trace_ctx, it, member_base + j, tr[static_cast<size_t>(it * B + j)]);
        if (book) ascent_s += secs_since(mark);
        if (ir.err != ~0ull)
            fail(LCB_NUMERIC, numeric_msg(static_cast<int64_t>(ir.err & 0xffffffffull),
                                          static_cast<int64_t>(ir.err >> 32) + member_base));

        mark = Clock::now();
        const int words = static_cast<int>((B + 31) / 32);
        uint32_t* Z = w.Z.ensure(static_cast<size_t>(words) * n);
        unsigned long long* cuts = w.cuts.ensure(static_cast<size_t>(words) * 32 + 1);
        unsigned long long* key = w.keys.ensure(8);
        // K4, one kernel: round -> cut counts -> argmax -> (single rank) winner bits
        const bool multi = comm_active(comm);
        launch_epilogue<T>(g, w.X[ir.final_buf].p, w.ld, static_cast<int>(B), l, lifted ? 1 : 0, Z, cuts,
                           static_cast<int>(B), member_base, key, multi ? nullptr : w.win.p, w.st,
                           w.dense_cut_done ? w.dcut.p : nullptr);
        w.dense_cut_done = false;
        if (multi) {
            comm_allreduce(comm, key, 1, 8, true, w.st, "allreduce(key)");
            launch_extract_winner(Z, n, key, member_base, static_cast<int>(B), w.win.p, w.st);
            comm_allreduce(comm, w.win.p, static_cast<size_t>(words_n), 4, true, w.st, "allreduce(winner)");
        }
        d2h(w.h_keys, key, sizeof(unsigned long long), w.st);
        CK(cudaStreamSynchronize(w.st));
        CK(cudaGetLastError());
        const unsigned long long k = w.h_keys[0];
        BatchRes r;
        r.cut = static_cast<int64_t>(k >> 32);
        r.member = static_cast<int64_t>(0xffffffffull - (k & 0xffffffffull));
        r.serial = s;
        if (book) rounding_s += secs_since(mark);
        return r;
    }

    // Batched evolve() round: K candidates' batches in one launch
    // sequence.  Candidate k keeps serial serial0+k (its member streams are the ones
    // the sequential order would have drawn), its own (alpha, T) per member, its own
    // error slot and argmax segment; the segments' keys come back in one copy.
    struct MultiRes {
        std::vector<BatchRes> res;
        std::vector<bool> numeric;
        std::vector<int> seg_of;  // candidate -> batch segment
        unsigned long long* d_keys = nullptr;
        uint32_t* Z = nullptr;
    };
    MultiRes run_batch_multi(bool lifted, int l, const uint32_t* bits, const std::vector<Cand*>& cs, double mu,
                             bool ee) {
        const int n = g.n;
        const int K = static_cast<int>(cs.size());
        const int64_t serial0 = serial;
        serial += K;
        const double eta_eff = cfg.scale_noise ? cfg.eta / (cfg.init_scale * cfg.init_scale) : cfg.eta;
        const int members = static_cast<int>(B) * K;
        const int W = members * l;
        w.shape(n, W);
        // segment order: candidates by descending T (stable), so finished candidates are a
        // suffix of the batch and the launches shrink as they finish
        std::vector<int> order(static_cast<size_t>(K));
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(),
                         [&](int x, int y) { return cs[x]->iterations > cs[y]->iterations; });
        std::vector<uint64_t> mk;
        for (int sgi = 0; sgi < K; ++sgi) member_keys(serial0 + order[sgi], mk);
        init_batch(l, nullptr, bits, mk, std::sqrt(eta_eff));
        std::vector<T> alpha(static_cast<size_t>(members));
        std::vector<int> tlim(static_cast<size_t>(members));
        std::vector<int64_t> seg_iters(static_cast<size_t>(K));
        int64_t tmax = 0, upd = 0;
        for (int sgi = 0; sgi < K; ++sgi) {
            const Cand& c = *cs[order[sgi]];
            seg_iters[sgi] = c.iterations;
            tmax = std::max(tmax, c.iterations);
            upd += c.iterations;
            for (int64_t j = 0; j < B; ++j) {
                alpha[static_cast<size_t>(sgi * B + j)] = static_cast<T>(c.alpha());
                tlim[static_cast<size_t>(sgi * B + j)] = static_cast<int>(c.iterations);
            }
        }
        T* da = w.alpha.ensure(alpha.size());
        int* dt = w.tlim.ensure(tlim.size());
        h2d(da, alpha.data(), sizeof(T) * alpha.size(), w.st);
        h2d(dt, tlim.data(), sizeof(int) * tlim.size(), w.st);
        const int64_t before = w.node_updates;
        IterResult ir = run_iterations<T>(g, w, W, members, l, tmax, T(0), da, dt, static_cast<T>(mu), ee,
                                          nullptr, static_cast<int>(B), &seg_iters);
        sync_errors(ir);
        w.node_updates = before + upd * static_cast<int64_t>(n) * B * l;  // active updates only
        MultiRes out;
        const int words = (members + 31) / 32;
        out.Z = w.Z.ensure(static_cast<size_t>(words) * n);
        launch_round_pack<T>(w.X[ir.final_buf].p, w.ld, n, members, l, lifted ? 1 : 0, out.Z, w.st);
        unsigned long long* cuts = w.cuts.ensure(static_cast<size_t>(words) * 32 + 1);
        out.d_keys = w.keys.ensure(static_cast<size_t>(std::max(K, 8)));
        launch_cut_argmax(g, out.Z, words, cuts, members, static_cast<int>(B), member_base, out.d_keys, w.st);
        comm_allreduce(comm, out.d_keys, static_cast<size_t>(K), 8, true, w.st, "allreduce(keys)");
        d2h(w.h_keys, out.d_keys, sizeof(unsigned long long) * K, w.st);
        CK(cudaStreamSynchronize(w.st));
        CK(cudaGetLastError());
        out.seg_of.assign(static_cast<size_t>(K), 0);
        for (int sgi = 0; sgi < K; ++sgi) out.seg_of[static_cast<size_t>(order[sgi])] = sgi;
        for (int k = 0; k < K; ++k) {
            const int sgi = out.seg_of[static_cast<size_t>(k)];
            const unsigned long long key = w.h_keys[sgi];
            BatchRes r;
            r.cut = static_cast<int64_t>(key >> 32);
            r.member = static_cast<int64_t>(0xffffffffull - (key & 0xffffffffull));
            r.serial = serial0 + k;
            out.res.push_back(r);
            out.numeric.push_back(sgi < static_cast<int>(ir.errs.size()) && ir.errs[sgi] != ~0ull);
        }
        return out;
    }

    // winner bits of segment k of the last multi batch -> w.win
    void multi_winner(const MultiRes& m, int k) {
        const int sgi = m.seg_of[static_cast<size_t>(k)];
        launch_extract_winner(m.Z, g.n, m.d_keys + sgi, member_base, static_cast<int>(B) * (sgi + 1), w.win.p, w.st,
                              static_cast<int>(B) * sgi);
        comm_allreduce(comm, w.win.p, static_cast<size_t>(words_n), 4, true, w.st, "allreduce(winner)");
    }

    // note_batch — solver.cpp:145-150 (winner bits are in w.win)
    void note_batch(const BatchRes& r, int kind, double alpha, int64_t iters) {
        if (!has_best || r.cut > best_cut) {
            has_best = true;
            best_cut = r.cut;
            best_serial = r.serial;
            best_member = r.member;
            copy_bits(w.gbest.p, w.win.p);
        }
        if (sinks.nbt < sinks.bt_cap) {
            lcb_batch_trace& e = sinks.bt[sinks.nbt];
            e.serial = r.serial;
            e.kind = kind;
            e.pad_ = 0;
            e.alpha = alpha;
            e.iterations = iters;
            e.batch_best = r.cut;
            e.best_so_far = best_cut;
        }
        ++sinks.nbt;
    }

    static bool ranks_before(const Cand& a, const Cand& b) {
        const double fa = a.has_fit ? a.fitness : -std::numeric_limits<double>::infinity();
        const double fb = b.has_fit ? b.fitness : -std::numeric_limits<double>::infinity();
        if (fa != fb) return fa > fb;
        if (a.iterations != b.iterations) return a.iterations < b.iterations;
        return a.exponent < b.exponent;
    }

    // run_search — solver.cpp:154-180 + evolve — evo_search.cpp:61-90.
    // The incumbent is w.recenter (not modified while the search runs).
    Cand run_search(bool lifted, int l, double mu, bool ee) {
        const auto mark = Clock::now();
        const int kind = lifted ? 1 : 0;
        HostStream s{split3(base, 0x6576u, static_cast<uint64_t>(kind), search_runs[kind]++)};
        std::vector<Cand> pop(static_cast<size_t>(cfg.population_size));
        for (Cand& c : pop) {  // sample_population (evo_search.cpp:26-34)
            c.iterations = s.integer(cfg.t_lower, cfg.t_upper);
            c.exponent = s.uniform(cfg.e_lower, cfg.e_upper);
        }
        const size_t half = pop.size() / 2;
        auto trace_eval = [&](int round, const Cand& c) {
            if (sinks.nst < sinks.st_cap) {
                lcb_search_trace& e = sinks.st[sinks.nst];
                e.round = round;
                e.pad_ = 0;
                e.exponent = c.exponent;
                e.iterations = c.iterations;
                e.fitness = c.fitness;
            }
            ++sinks.nst;
        };
        for (int round = 1; round <= cfg.rounds; ++round) {
            std::vector<Cand*> todo;
            for (Cand& c : pop)
                if (!c.has_fit) todo.push_back(&c);
            if (batched_search && todo.size() > 1) {
                // one budget check per round (the sequential order checks per candidate)
                if (budget_gone()) {
                    for (Cand* c : todo) {
                        c->has_fit = true;
                        c->fitness = -std::numeric_limits<double>::infinity();
                        trace_eval(round, *c);
                    }
                } else {
                    const MultiRes m = run_batch_multi(lifted, l, w.recenter.p, todo, mu, ee);
                    for (size_t k = 0; k < todo.size(); ++k) {
                        Cand& c = *todo[k];
                        double fit = -std::numeric_limits<double>::infinity();
                        if (!m.numeric[k]) {
                            const BatchRes& r = m.res[k];
                            if (!has_best || r.cut > best_cut) multi_winner(m, static_cast<int>(k));
                            note_batch(r, 1, c.alpha(), c.iterations);
                            fit = static_cast<double>(r.cut);
                        }
                        c.has_fit = true;
                        c.fitness = fit;
                        trace_eval(round, c);
                    }
                }
                todo.clear();
            }
            for (Cand* cp : todo) {
                Cand& c = *cp;
                double fit;
                if (budget_gone()) {
                    fit = -std::numeric_limits<double>::infinity();  // Error -> -inf
                } else {
                    try {
                        const BatchRes r = run_batch(lifted, l, nullptr, w.recenter.p, c.alpha(), c.iterations, mu, ee, false);
                        note_batch(r, 1, c.alpha(), c.iterations);
                        fit = static_cast<double>(r.cut);
                    } catch (const Failure& f) {
                        if (f.status != LCB_NUMERIC) throw;
                        fit = -std::numeric_limits<double>::infinity();
                    }
                }
                c.has_fit = true;
                c.fitness = fit;
                trace_eval(round, c);
            }
            std::stable_sort(pop.begin(), pop.end(), ranks_before);
            for (size_t slot = half; slot < pop.size(); ++slot) {
                const Cand& parent = pop[static_cast<size_t>(s.integer(0, static_cast<int64_t>(half) - 1))];
                Cand child;
                double moved = parent.exponent + 0.2 * s.normal();  // perturb_exponent
                child.exponent = std::clamp(moved, -4.0, -1.0);
                const double eps = s.unit();                          // perturb_iterations
                const auto scaled = static_cast<int64_t>(
                    std::floor(static_cast<double>(parent.iterations) * (1.0 + 0.2 * (2.0 * eps - 1.0))));
                child.iterations = std::max<int64_t>(1, scaled);
                pop[slot] = child;
            }
        }
        search_s += secs_since(mark);
        return pop.front();
    }

    bool search_due(int kind) const {
        if (!cfg.has_search) return false;
        const int64_t count = main_batches[kind];
        if (cfg.search_refresh > 0) return (count - 1) % cfg.search_refresh == 0;
        return !has_tuned[kind] && count == 1;
    }

    // run_phase — solver.cpp:191-246.  carry lives in w.carry (valid iff has_carry).
    void run_phase(bool lifted, int phase_idx, bool& has_carry) {
        const int n = g.n;
        const int l = lifted ? cfg.lift_dim : 1;
        const int kind = lifted ? 1 : 0;
        double alpha = cfg.alpha, mu = cfg.momentum;
        int64_t iters = cfg.iterations;
        bool ee = cfg.early_exit != 0;
        if (lifted && cfg.has_lifted_ascent) {
            alpha = cfg.l_alpha;
            iters = cfg.l_iterations;
            mu = cfg.l_momentum;
            ee = cfg.l_early_exit != 0;
        }
        if (has_tuned[kind]) {
            alpha = tuned[kind].alpha();
            iters = tuned[kind].iterations;
        }
        bool has_recenter = has_carry;
        if (has_recenter) copy_bits(w.recenter.p, w.carry.p);
        bool has_pbest = false;
        int64_t pbest_cut = 0;
        for (int64_t b = 0; b < cfg.num_batches; ++b) {
            if (serial > 0 && budget_gone()) break;
            const double* dmean = nullptr;
            const uint32_t* bits = nullptr;
            if (b == 0) {
                const auto mark = Clock::now();
                const uint64_t word = cfg.resample_idi ? static_cast<uint64_t>(serial) : 0u;
                const uint64_t ikey = split3(base, 0x696eu, cfg.init_seed, word);
                const bool carry_col0 = has_recenter && (l == 1 || cfg.deco_carry == 0);
                std::vector<uint64_t> ck(static_cast<size_t>(l));
                for (int c = 0; c < l; ++c) ck[c] = split2(ikey, 0x636fu, static_cast<uint64_t>(c));
                uint64_t* dck = w.colkeys.ensure(ck.size());
                h2d(dck, ck.data(), sizeof(uint64_t) * ck.size(), w.st);
                double* mean = w.mean.ensure(static_cast<size_t>(n) * l);
                const uint32_t* cb = carry_col0 ? w.recenter.p : nullptr;
                if (cfg.init_method == 0) {
                    if (g.max_degree < 1) fail(LCB_VALIDATION, "dui_init: graph has no edges (MaxCut is trivially 0)");
                    launch_dui(g, dck, l, cfg.init_scale, cb, mean, w.st);
                } else {
                    const double thr = g.deg_mean + cfg.beta * g.deg_sd;
                    launch_idi(g, thr, dck, l, cfg.init_scale, cb, w.sign.ensure(static_cast<size_t>(n) * l), mean, w.st);
                }
                CK(cudaStreamSynchronize(w.st));
                init_s += secs_since(mark);
                dmean = mean;
            } else {
                bits = w.recenter.p;
            }
            const BatchRes r = run_batch(lifted, l, dmean, bits, alpha, iters, mu, ee, true);
            note_batch(r, 0, alpha, iters);
            if (!has_pbest || r.cut > pbest_cut) {
                has_pbest = true;
                pbest_cut = r.cut;
                copy_bits(w.pbest.p, w.win.p);
            }
            copy_bits(w.recenter.p, w.win.p);
            has_recenter = true;
            ++main_batches[kind];
            if (search_due(kind) && !budget_gone()) {
                const Cand win = run_search(lifted, l, mu, ee);
                alpha = win.alpha();
                iters = win.iterations;
                tuned[kind] = win;
                has_tuned[kind] = true;
            }
        }
        if (!has_pbest) {
            if (has_recenter) copy_bits(w.carry.p, w.recenter.p);
            has_carry = has_recenter;
            return;
        }
        if (sinks.npt < sinks.pt_cap) {
            sinks.pt[sinks.npt].phase = phase_idx;
            sinks.pt[sinks.npt].kind = kind;
            sinks.pt[sinks.npt].best_after = pbest_cut;
        }
        ++sinks.npt;
        copy_bits(w.carry.p, w.pbest.p);
        has_carry = true;
    }

    // pquco / pluco / pdeco — solver.cpp:273-312
    void solve() {
        bool has_carry = false;
        if (cfg.algorithm == 0) {
            run_phase(false, 0, has_carry);
        } else if (cfg.algorithm == 1) {
            run_phase(true, 0, has_carry);
        } else {
            int phase = 0;
            for (int round = 0;; ++round) {
                if (cfg.time_budget_s > 0.0) {
                    if (serial > 0 && budget_gone()) break;
                } else if (round >= cfg.deco_alternations) {
                    break;
                }
                const int64_t before = serial;
                run_phase(false, phase++, has_carry);
                run_phase(true, phase++, has_carry);
                if (cfg.time_budget_s > 0.0 && serial == before) break;
            }
        }
        if (!has_best) fail(LCB_ERROR, "solver produced no batch result");
    }

    void best_assignment(uint8_t* z) {
        std::vector<uint32_t> hb(words_n);
        d2h(hb.data(), w.gbest.p, sizeof(uint32_t) * words_n, w.st);
        CK(cudaStreamSynchronize(w.st));
        for (int v = 0; v < g.n; ++v) z[v] = static_cast<uint8_t>((hb[v >> 5] >> (v & 31)) & 1u);
    }
};

void validate_config(const lcb_config& c) {
    auto bad = [](const char* m) { fail(LCB_VALIDATION, m); };
    if (c.batch_size < 1) bad("batch_size must be >= 1");
    if (c.num_batches < 1) bad("num_batches must be >= 1");
    if (c.lift_dim < 1) bad("lift_dim must be >= 1");
    if (c.algorithm != 0 && c.lift_dim < 2) bad("lifted algorithms need lift_dim >= 2");
    if (!(c.alpha > 0.0)) bad("ascent: alpha must be > 0");
    if (c.iterations < 1) bad("ascent: iterations must be >= 1");
    if (!(c.momentum >= 0.0 && c.momentum < 1.0)) bad("ascent: momentum must lie in [0, 1)");
    if (c.has_lifted_ascent) {
        if (!(c.l_alpha > 0.0)) bad("ascent: alpha must be > 0");
        if (c.l_iterations < 1) bad("ascent: iterations must be >= 1");
        if (!(c.l_momentum >= 0.0 && c.l_momentum < 1.0)) bad("ascent: momentum must lie in [0, 1)");
    }
    if (c.beta <= 0.0 || c.beta >= 1.0) bad("init.beta must lie in (0, 1)");
    if (c.eta <= 0.0) bad("init.eta must be > 0");
    if (c.init_scale < 1.0) bad("init.init_scale must be >= 1");
    if (c.has_search) {
        if (c.t_lower < 1 || c.t_lower > c.t_upper) bad("search: need 1 <= t_lower <= t_upper");
        if (c.e_lower > c.e_upper) bad("search: need e_lower <= e_upper");
        if (c.population_size < 2 || c.population_size % 2 != 0)
            bad("search: population size must be even and >= 2");
        if (c.rounds < 1) bad("search: rounds must be >= 1");
    }
    if (c.search_refresh < 0) bad("search_refresh must be >= 0");
    if (c.deco_alternations < 1) bad("deco_alternations must be >= 1");
    if (c.batch_size > 0x7fffffff) bad("batch_size too large");
}

template <class T>
void solve_graph(const DevGraph& g, const lcb_config& cfg, uint64_t seed, const lcb_run_opts& o,
                 Work<T>& w, TraceSinks& sinks, uint8_t* z, lcb_outcome& out) {
    if (g.m < 1) fail(LCB_VALIDATION, "solver requires a graph with at least one edge");
    const bool hinit = o.host_init < 0 ? (o.precision == LCB_FP64) : (o.host_init != 0);
    Solver<T> s(g, cfg, w, sinks, o.comm, hinit, seed);
    s.trace_fn = o.trace_fn;
    s.trace_ctx = o.trace_ctx;
    s.batched_search = o.batched_search != 0;
    s.solve();
    s.best_assignment(z);
    out.cut_value += s.best_cut;
    out.batch_index = s.best_serial;
    out.member_index = s.best_member;
    out.batches_run += s.serial;
    out.init_s += s.init_s;
    out.ascent_s += s.ascent_s;
    out.rounding_s += s.rounding_s;
    out.search_s += s.search_s;
}

// host copy of the device CSR, fetched only for per-component solves
struct HostCSR {
    std::vector<int> off, adj;
};
HostCSR fetch_csr(const DevGraph& g) {
    HostCSR h;
    h.off.resize(static_cast<size_t>(g.n) + 1);
    h.adj.resize(static_cast<size_t>(g.nnz));
    CK(cudaMemcpy(h.off.data(), g.row_ptr, sizeof(int) * h.off.size(), cudaMemcpyDeviceToHost));
    if (g.nnz) CK(cudaMemcpy(h.adj.data(), g.col, sizeof(int) * h.adj.size(), cudaMemcpyDeviceToHost));
    count_d2h(sizeof(int) * (h.off.size() + h.adj.size()));
    return h;
}

// connected components, graph.cpp:75-99
std::vector<std::vector<uint32_t>> components(const HostCSR& h) {
    const uint32_t n = static_cast<uint32_t>(h.off.size() - 1);
    std::vector<std::vector<uint32_t>> out;
    std::vector<char> seen(n, 0);
    std::vector<uint32_t> stack;
    for (uint32_t root = 0; root < n; ++root) {
        if (seen[root]) continue;
        std::vector<uint32_t> comp;
        seen[root] = 1;
        stack.push_back(root);
        while (!stack.empty()) {
            const uint32_t v = stack.back();
            stack.pop_back();
            comp.push_back(v);
            for (int k = h.off[v]; k < h.off[v + 1]; ++k) {
                const uint32_t u = static_cast<uint32_t>(h.adj[static_cast<size_t>(k)]);
                if (!seen[u]) {
                    seen[u] = 1;
                    stack.push_back(u);
                }
            }
        }
        std::sort(comp.begin(), comp.end());
        out.push_back(std::move(comp));
    }
    return out;
}

template <class T>
void solve_top(const DevGraph& g, const lcb_config& cfg, uint64_t seed, int per_component,
               const lcb_run_opts& o, lcb_outcome& out, uint8_t* assignment, TraceSinks& sinks) {
    PooledWork<T> pw(g.device);
    Work<T>& w = *pw;
    const auto t0 = Clock::now();
    std::memset(&out, 0, sizeof(out));
    cudaEvent_t s0 = nullptr, s1 = nullptr;
    CK(cudaEventCreate(&s0));
    CK(cudaEventCreate(&s1));
    struct EvFree {
        cudaEvent_t a, b;
        ~EvFree() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } evf{s0, s1};
    CK(cudaEventRecord(s0, w.st));
    auto finish = [&] {
        CK(cudaEventRecord(s1, w.st));
        CK(cudaEventSynchronize(s1));
        float sms = 0.f;
        CK(cudaEventElapsedTime(&sms, s0, s1));
        if (o.solve_ms) *o.solve_ms = sms;
        out.n_batch_trace = sinks.nbt;
        out.n_phase_trace = sinks.npt;
        out.n_search_trace = sinks.nst;
        out.wall_s = secs_since(t0);
        if (o.step_ms) *o.step_ms = w.step_ms;
        if (o.step_launches) *o.step_launches = w.step_launches;
        if (o.node_updates) *o.node_updates = w.node_updates;
        if (o.step_bytes) *o.step_bytes = w.step_bytes;
        if (o.kernel_stats) std::memcpy(o.kernel_stats, w.kstats, sizeof(w.kstats));
    };
    if (!per_component) {
        solve_graph<T>(g, cfg, seed, o, w, sinks, assignment, out);
        finish();
        return;
    }
    // solve_per_component — solver.cpp:314-364
    const HostCSR hc = fetch_csr(g);
    const auto comps = components(hc);
    if (comps.size() == 1 && g.m > 0) {
        solve_graph<T>(g, cfg, seed, o, w, sinks, assignment, out);
        finish();
        return;
    }
    // multi-rank: every rank walks the same components in the same order (the graph is
    // replicated) and each component solve is member-sharded with its own collectives
    std::memset(assignment, 0, static_cast<size_t>(g.n));
    out.batch_index = -1;
    out.member_index = -1;
    int solved = 0;
    std::vector<uint32_t> local(static_cast<size_t>(g.n), static_cast<uint32_t>(g.n));
    for (size_t ci = 0; ci < comps.size(); ++ci) {
        const auto& comp = comps[ci];
        if (comp.size() < 2) continue;
        const uint32_t k = static_cast<uint32_t>(comp.size());
        for (uint32_t i = 0; i < k; ++i) local[comp[i]] = i;
        // induced_subgraph (graph.cpp:101-110): relabel in component order; rows stay sorted
        std::vector<int64_t> off(k + 1, 0);
        std::vector<uint32_t> adj;
        for (uint32_t i = 0; i < k; ++i) {
            const uint32_t v = comp[i];
            for (int q = hc.off[v]; q < hc.off[v + 1]; ++q) {
                const uint32_t u = static_cast<uint32_t>(hc.adj[static_cast<size_t>(q)]);
                if (local[u] != static_cast<uint32_t>(g.n)) adj.push_back(local[u]);
            }
            off[i + 1] = static_cast<int64_t>(adj.size());
            std::sort(adj.begin() + off[i], adj.end());
        }
        for (uint32_t i = 0; i < k; ++i) local[comp[i]] = static_cast<uint32_t>(g.n);
        if (off[k] == 0) continue;
        DevGraph sub;
        build_graph(sub, k, off.data(), adj.data(), g.device);
        struct Free {
            DevGraph& d;
            ~Free() { free_graph(d); }
        } fr{sub};
        const uint64_t sub_seed = rng_at(split2(seed, 0x6370u, static_cast<uint64_t>(ci)), 0);
        std::vector<uint8_t> za(k);
        lcb_outcome part{};
        TraceSinks ps{sinks.bt ? sinks.bt + std::min(sinks.nbt, sinks.bt_cap) : nullptr,
                      std::max<int64_t>(0, sinks.bt_cap - sinks.nbt),
                      sinks.pt ? sinks.pt + std::min(sinks.npt, sinks.pt_cap) : nullptr,
                      std::max<int64_t>(0, sinks.pt_cap - sinks.npt),
                      sinks.st ? sinks.st + std::min(sinks.nst, sinks.st_cap) : nullptr,
                      std::max<int64_t>(0, sinks.st_cap - sinks.nst)};
        solve_graph<T>(sub, cfg, sub_seed, o, w, ps, za.data(), part);
        for (uint32_t i = 0; i < k; ++i) assignment[comp[i]] = za[i];
        out.cut_value += part.cut_value;
        out.batch_index = part.batch_index;
        out.member_index = part.member_index;
        out.batches_run += part.batches_run;
        out.init_s += part.init_s;
        out.ascent_s += part.ascent_s;
        out.rounding_s += part.rounding_s;
        out.search_s += part.search_s;
        sinks.nbt += ps.nbt;
        sinks.npt += ps.npt;
        sinks.nst += ps.nst;
        ++solved;
    }
    if (solved != 1) {
        out.batch_index = -1;
        out.member_index = -1;
    }
    finish();
}

// ---- boundary helpers for the single-call API -----------------------------
template <class T>
void ascend_host(const DevGraph& g, double* values, int64_t n, int l, int64_t B, double alpha,
                 int64_t iters, double mu, bool ee, double* trace, int64_t* err_it, int64_t* err_m) {
    if (!(alpha > 0.0)) fail(LCB_VALIDATION, "ascent: alpha must be > 0");
    if (iters < 1) fail(LCB_VALIDATION, "ascent: iterations must be >= 1");
    if (!(mu >= 0.0 && mu < 1.0)) fail(LCB_VALIDATION, "ascent: momentum must lie in [0, 1)");
    if (n != g.n)
        fail(LCB_SHAPE, "ascend: state row dimension " + std::to_string(n) + " != node count " +
                            std::to_string(g.n));
    if (l < 1 || B < 1) fail(LCB_VALIDATION, "DenseState: n, l, B must all be >= 1");
    const int64_t W64 = B * l;
    if (W64 > (1 << 26)) fail(LCB_VALIDATION, "batch too wide");
    const int W = static_cast<int>(W64);
    DeviceScope ds(g.device);
    PooledWork<T> pw(g.device);
    Work<T>& w = *pw;
    w.shape(g.n, W);
    const size_t count = static_cast<size_t>(W) * g.n;
    double* d = w.hostbatch.ensure(count);
    h2d(d, values, sizeof(double) * count, w.st);
    launch_transpose_in<T>(d, w.X[0].p, g.n, W, w.ld, w.st);
    CK(cudaMemsetAsync(w.V.p, 0, sizeof(T) * static_cast<size_t>(g.n) * w.ld, w.st));
    const bool use_ee = ee && trace == nullptr;  // ascent.cpp:91
    const IterResult r = run_iterations<T>(g, w, W, static_cast<int>(B), l, iters, static_cast<T>(alpha),
                                           nullptr, nullptr, static_cast<T>(mu), use_ee, trace);
    launch_transpose_out<T>(w.X[r.final_buf].p, d, g.n, W, w.ld, w.st);
    d2h(values, d, sizeof(double) * count, w.st);
    CK(cudaStreamSynchronize(w.st));
    if (r.err != ~0ull) {
        const int64_t it = static_cast<int64_t>(r.err & 0xffffffffull);
        const int64_t m = static_cast<int64_t>(r.err >> 32);
        if (err_it) *err_it = it;
        if (err_m) *err_m = m;
        fail(LCB_NUMERIC, numeric_msg(it, m));
    }
}

// Row-sharded ascend (north star 5: graphs whose adjacency does not fit one
// HBM).  Rank q holds the CSR rows [r0_q, r1_q) (global column ids) and its slice
// [B][l][r1_q - r0_q] of the state; the ranges partition [0, n).  Every rank keeps the
// whole iterate X [n][ld] (double-buffered) and its own rows of V.  Per iteration: K1 over
// the local rows (the reference's CSR-order sums, graph.cpp:116-121, so fp64 stays
// bit-exact with ascend on the whole graph), the early-exit bits OR-reduced across ranks
// (a MAX over one 0/1 array per bit), then an all-gather of the new rows.
template <class T>
void ascend_rows_host(lcb_comm* comm, uint32_t n, int64_t r0, int64_t r1, const int64_t* off, const uint32_t* adj,
                      double* values, int l, int64_t B, double alpha, int64_t iters, double mu, bool ee,
                      int device, int64_t* err_it, int64_t* err_m) {
    if (!(alpha > 0.0)) fail(LCB_VALIDATION, "ascent: alpha must be > 0");
    if (iters < 1) fail(LCB_VALIDATION, "ascent: iterations must be >= 1");
    if (!(mu >= 0.0 && mu < 1.0)) fail(LCB_VALIDATION, "ascent: momentum must lie in [0, 1)");
    if (l < 1 || B < 1) fail(LCB_VALIDATION, "DenseState: n, l, B must all be >= 1");
    if (n == 0 || r0 < 0 || r1 < r0 || r1 > static_cast<int64_t>(n)) fail(LCB_VALIDATION, "row range outside [0, n)");
    const int64_t rows = r1 - r0;
    if (off[0] != 0) fail(LCB_VALIDATION, "offsets[0] must be 0");
    for (int64_t i = 0; i < rows; ++i)
        if (off[i + 1] < off[i]) fail(LCB_VALIDATION, "offsets must be non-decreasing");
    const int64_t nnz = off[rows];
    if (nnz > std::numeric_limits<int>::max()) fail(LCB_VALIDATION, "row range exceeds 2^31 adjacency entries");
    for (int64_t k = 0; k < nnz; ++k)
        if (adj[k] >= n) fail(LCB_VALIDATION, "adjacency entry out of range");
    const int64_t W64 = B * l;
    if (W64 > (1 << 26)) fail(LCB_VALIDATION, "batch too wide");
    const int W = static_cast<int>(W64);
    const int members = static_cast<int>(B);
    DeviceScope ds(device);
    PooledWork<T> pw(device);
    Work<T>& w = *pw;
    w.shape(static_cast<int>(n), W);
    // every rank's range, checked to partition [0, n)
    const int nr = comm_active(comm) ? comm->nranks : 1, me = comm_active(comm) ? comm->rank : 0;
    std::vector<int64_t> range(static_cast<size_t>(2 * nr), 0);
    range[static_cast<size_t>(2 * me)] = r0;
    range[static_cast<size_t>(2 * me + 1)] = r1;
    if (nr > 1) {
        unsigned long long* dr = w.keys.ensure(static_cast<size_t>(2 * nr));
        std::vector<unsigned long long> hr(range.begin(), range.end());
        h2d(dr, hr.data(), sizeof(unsigned long long) * hr.size(), w.st);
        comm_allreduce(comm, dr, hr.size(), 8, true, w.st, "allreduce(row ranges)");
        d2h(hr.data(), dr, sizeof(unsigned long long) * hr.size(), w.st);
        CK(cudaStreamSynchronize(w.st));
        for (size_t i = 0; i < hr.size(); ++i) range[i] = static_cast<int64_t>(hr[i]);
    }
    for (int q = 0; q < nr; ++q)
        if (range[static_cast<size_t>(2 * q)] != (q ? range[static_cast<size_t>(2 * q - 1)] : 0))
            fail(LCB_VALIDATION, "row ranges must partition [0, n) in rank order");
    if (range[static_cast<size_t>(2 * nr - 1)] != static_cast<int64_t>(n))
        fail(LCB_VALIDATION, "row ranges must partition [0, n) in rank order");
    // this rank's rows at their global indices: row_ptr / deg hold entries r0 .. r1 only
    int* rp = w.rs_row_ptr.ensure(static_cast<size_t>(n) + 1);
    T* dg = w.rs_deg.ensure(static_cast<size_t>(n));
    int* col = w.rs_col.ensure(static_cast<size_t>(nnz) + 4);
    int* ord = w.rs_order.ensure(static_cast<size_t>(std::max<int64_t>(rows, 1)));
    {
        std::vector<int> hrp(static_cast<size_t>(rows) + 1), hord(static_cast<size_t>(rows));
        std::vector<T> hdg(static_cast<size_t>(rows));
        for (int64_t i = 0; i <= rows; ++i) hrp[static_cast<size_t>(i)] = static_cast<int>(off[i]);
        for (int64_t i = 0; i < rows; ++i) {
            hord[static_cast<size_t>(i)] = static_cast<int>(r0 + i);
            hdg[static_cast<size_t>(i)] = static_cast<T>(off[i + 1] - off[i]);
        }
        h2d(rp + r0, hrp.data(), sizeof(int) * hrp.size(), w.st);
        if (rows) {
            h2d(dg + r0, hdg.data(), sizeof(T) * hdg.size(), w.st);
            h2d(ord, hord.data(), sizeof(int) * hord.size(), w.st);
        }
        if (nnz) h2d(col, adj, sizeof(int) * static_cast<size_t>(nnz), w.st);
        CK(cudaStreamSynchronize(w.st));  // the host vectors go out of scope
    }
    // the local slice in, then every rank's rows
    const size_t cells = static_cast<size_t>(W) * static_cast<size_t>(rows);
    double* d = w.hostbatch.ensure(std::max<size_t>(cells, 1));
    if (rows) {
        h2d(d, values, sizeof(double) * cells, w.st);
        launch_transpose_in<T>(d, w.X[0].p + static_cast<size_t>(r0) * w.ld, static_cast<int>(rows), W, w.ld, w.st);
    }
    CK(cudaMemsetAsync(w.V.p, 0, sizeof(T) * static_cast<size_t>(n) * w.ld, w.st));
    const size_t row_bytes = sizeof(T) * static_cast<size_t>(w.ld);
    comm_allgather_rows(comm, w.X[0].p, row_bytes, range, w.st);

    StepArgs<T> a{};
    a.row_ptr = rp;
    a.col = col;
    a.deg = dg;
    a.order = ord;
    a.vel = w.V.p;
    a.ld = w.ld;
    a.n = static_cast<int>(rows);
    a.W = W;
    a.l = l;
    a.members = members;
    a.mu = static_cast<T>(mu);
    a.alpha_uniform = static_cast<T>(alpha);
    a.err = w.err.ensure(1);
    CK(cudaMemsetAsync(a.err, 0xff, sizeof(unsigned long long), w.st));
    uint32_t* F = nullptr;
    uint32_t* bits = nullptr;
    if (ee) {
        F = w.flags.ensure(static_cast<size_t>(3) * members);
        CK(cudaMemsetAsync(F, 0, sizeof(uint32_t) * 3 * members, w.st));
        bits = w.orbits.ensure(static_cast<size_t>(3) * members);
    }
    int64_t it = 0;
    for (; it < iters; ++it) {
        a.x_in = w.X[it & 1].p;
        a.x_out = w.X[(it + 1) & 1].p;
        a.it = static_cast<int>(it);
        if (ee) {
            a.flags_prev = F + ((it + 2) % 3) * members;
            a.flags_cur = F + (it % 3) * members;
            a.flags_zero = F + ((it + 1) % 3) * members;
        }
        if (rows) launch_step<T>(a, ee, MODE_STEP, w.st);
        else if (ee) CK(cudaMemsetAsync(a.flags_zero, 0, sizeof(uint32_t) * members, w.st));
        if (ee && nr > 1) {  // the member's exit test sees every rank's rows
            launch_bits_split(a.flags_cur, members, 3, bits, w.st);
            comm_allreduce(comm, bits, static_cast<size_t>(3) * members, 4, true, w.st, "allreduce(exit bits)");
            launch_bits_merge(bits, members, 3, a.flags_cur, w.st);
        }
        comm_allgather_rows(comm, a.x_out, row_bytes, range, w.st);
        if (ee && ((it + 1) % 32 == 0) && it + 1 < iters) {  // the same decision on every rank
            uint32_t* hf = w.host_flags(members);
            d2h(hf, a.flags_cur, sizeof(uint32_t) * members, w.st);
            CK(cudaStreamSynchronize(w.st));
            bool any = false;
            for (int m = 0; m < members && !any; ++m) any = ex_continue(hf[m]);
            if (!any) {
                ++it;
                break;
            }
        }
    }
    comm_allreduce(comm, a.err, 1, 8, false, w.st, "allreduce(err)");
    if (rows) {
        launch_transpose_out<T>(w.X[it & 1].p + static_cast<size_t>(r0) * w.ld, d, static_cast<int>(rows), W, w.ld,
                                w.st);
        d2h(values, d, sizeof(double) * cells, w.st);
    }
    unsigned long long e = 0;
    d2h(&e, a.err, sizeof(e), w.st);
    CK(cudaStreamSynchronize(w.st));
    CK(cudaGetLastError());
    w.node_updates += it * static_cast<int64_t>(rows) * W;
    if (e != ~0ull) {
        const int64_t ei = static_cast<int64_t>(e & 0xffffffffull);
        const int64_t em = static_cast<int64_t>(e >> 32);
        if (err_it) *err_it = ei;
        if (err_m) *err_m = em;
        fail(LCB_NUMERIC, numeric_msg(ei, em));
    }
}

template <class T>
void laplacian_host(const DevGraph& g, const double* x, double* y, int64_t count) {
    const int W = static_cast<int>(count);
    DeviceScope ds(g.device);
    PooledWork<T> pw(g.device);
    Work<T>& w = *pw;
    w.shape(g.n, W);
    const size_t cells = static_cast<size_t>(W) * g.n;
    double* d = w.hostbatch.ensure(cells);
    h2d(d, x, sizeof(double) * cells, w.st);
    launch_transpose_in<T>(d, w.X[0].p, g.n, W, w.ld, w.st);
    StepArgs<T> a{};
    a.row_ptr = g.row_ptr;
    a.col = g.col;
    a.deg = deg_of<T>(g);
    a.order = g.order;
    a.x_in = w.X[0].p;
    a.x_out = w.X[1].p;
    a.ld = w.ld;
    a.n = g.n;
    a.W = W;
    a.l = 1;
    a.members = W;
    launch_step<T>(a, false, MODE_LAPLACE, w.st);
    launch_transpose_out<T>(w.X[1].p, d, g.n, W, w.ld, w.st);
    d2h(y, d, sizeof(double) * cells, w.st);
    CK(cudaStreamSynchronize(w.st));
    CK(cudaGetLastError());
}

}  // namespace lcb

// ===========================================================================
// C ABI
// ===========================================================================
using namespace lcb;

extern "C" {

const char* lcb_last_error(void) { return g_last_error.c_str(); }
int lcb_abi_version(void) { return LCB_ABI_VERSION; }

int lcb_set_option(const char* name, int64_t value) {
    return guard([&] {
        const int i = opt_index(name);
        if (i < 0) fail(LCB_VALIDATION, std::string("unknown option '") + (name ? name : "") + "'");
        init_opts();
        g_opts[i].store(value);
    });
}

int lcb_get_option(const char* name, int64_t* value) {
    return guard([&] {
        const int i = opt_index(name);
        if (i < 0 || !value) fail(LCB_VALIDATION, std::string("unknown option '") + (name ? name : "") + "'");
        *value = option(static_cast<Opt>(i));
    });
}

int lcb_device_count(int* count) {
    return guard([&] { CK(cudaGetDeviceCount(count)); });
}

int lcb_graph_create(uint32_t n, const int64_t* offsets, const uint32_t* adjacency, int device,
                     lcb_graph** out) {
    return guard([&] {
        auto h = std::make_unique<lcb_graph>();
        try {
            build_graph(h->g, n, offsets, adjacency, device);
        } catch (...) {
            free_graph(h->g);
            throw;
        }
        *out = h.release();
    });
}

int lcb_graph_from_edges(uint32_t n, const uint32_t* eu, const uint32_t* ev, int64_t m, int device,
                         lcb_graph** out) {
    return guard([&] {
        if (!out || (m > 0 && (!eu || !ev))) fail(LCB_VALIDATION, "null argument");
        if (m < 0) fail(LCB_VALIDATION, "negative edge count");
        DeviceScope ds(device);
        IngestResult r = ingest_edges(n, eu, ev, m, 0);
        auto h = std::make_unique<lcb_graph>();
        try {
            // the host relabelling of small graphs needs the adjacency on the host too
            std::vector<uint32_t> hadj;
            if (n <= static_cast<uint32_t>(kResidentMaxRows) && r.nnz) {
                hadj.resize(static_cast<size_t>(r.nnz));
                d2h(hadj.data(), r.col, sizeof(int) * static_cast<size_t>(r.nnz), 0);
                CK(cudaStreamSynchronize(0));
            }
            int* col = r.col;
            r.col = nullptr;
            build_graph(h->g, n, r.off.data(), hadj.empty() ? nullptr : hadj.data(), device, col);
        } catch (...) {
            if (r.col) graph_free(r.col);
            free_graph(h->g);
            throw;
        }
        *out = h.release();
    });
}

int lcb_graph_parse(const char* text, int64_t len, int device, lcb_graph** out, int* saw_weights) {
    return guard([&] {
        if (!out || (len > 0 && !text)) fail(LCB_VALIDATION, "null argument");
        DeviceScope ds(device);
        uint32_t n = 0;
        bool weights = false;
        IngestResult r = parse_edge_text(text, len, n, weights, 0);
        auto h = std::make_unique<lcb_graph>();
        try {
            std::vector<uint32_t> hadj;
            if (n <= static_cast<uint32_t>(kResidentMaxRows) && r.nnz) {
                hadj.resize(static_cast<size_t>(r.nnz));
                d2h(hadj.data(), r.col, sizeof(int) * static_cast<size_t>(r.nnz), 0);
                CK(cudaStreamSynchronize(0));
            }
            int* col = r.col;
            r.col = nullptr;
            build_graph(h->g, n, r.off.data(), hadj.empty() ? nullptr : hadj.data(), device, col);
        } catch (...) {
            if (r.col) graph_free(r.col);
            free_graph(h->g);
            throw;
        }
        if (saw_weights) *saw_weights = weights ? 1 : 0;
        *out = h.release();
    });
}

int lcb_graph_csr(const lcb_graph* g, int64_t* offsets, uint32_t* adjacency) {
    return guard([&] {
        if (!g) fail(LCB_VALIDATION, "null graph");
        const HostCSR h = fetch_csr(g->g);
        if (offsets)
            for (size_t v = 0; v < h.off.size(); ++v) offsets[v] = h.off[v];
        if (adjacency && !h.adj.empty()) std::memcpy(adjacency, h.adj.data(), sizeof(uint32_t) * h.adj.size());
    });
}

void lcb_graph_destroy(lcb_graph* g) {
    if (!g) return;
    {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(g->g.device);
        free_graph(g->g);
        cudaSetDevice(prev);
    }
    delete g;
}

int lcb_graph_info(const lcb_graph* g, uint32_t* n, int64_t* m, int64_t* max_degree) {
    return guard([&] {
        if (!g) fail(LCB_VALIDATION, "null graph");
        if (n) *n = static_cast<uint32_t>(g->g.n);
        if (m) *m = g->g.m;
        if (max_degree) *max_degree = g->g.max_degree;
    });
}

int lcb_laplacian_apply(const lcb_graph* g, const double* x, double* y, int64_t count,
                        int32_t precision) {
    return guard([&] {
        if (!g) fail(LCB_VALIDATION, "null graph");
        if (count < 1) fail(LCB_SHAPE, "laplacian_apply: expected vectors of length " + std::to_string(g->g.n));
        if (precision == LCB_FP32)
            laplacian_host<float>(g->g, x, y, count);
        else
            laplacian_host<double>(g->g, x, y, count);
    });
}

int lcb_ascend(const lcb_graph* g, double* values, int64_t n, int32_t l, int64_t B, double alpha,
               int64_t iterations, double momentum, int32_t early_exit, int32_t precision,
               double* trace, int64_t* err_iter, int64_t* err_member) {
    return guard([&] {
        if (!g) fail(LCB_VALIDATION, "null graph");
        if (precision == LCB_FP32)
            ascend_host<float>(g->g, values, n, l, B, alpha, iterations, momentum, early_exit != 0, trace,
                               err_iter, err_member);
        else
            ascend_host<double>(g->g, values, n, l, B, alpha, iterations, momentum, early_exit != 0, trace,
                                err_iter, err_member);
    });
}

int lcb_ascend_rows(lcb_comm* comm, uint32_t n, int64_t row_begin, int64_t row_end, const int64_t* offsets,
                    const uint32_t* adjacency, double* values, int32_t l, int64_t B, double alpha, int64_t iterations,
                    double momentum, int32_t early_exit, int32_t precision, int device, int64_t* err_iter,
                    int64_t* err_member) {
    return guard([&] {
        if (!offsets || (row_end > row_begin && !values)) fail(LCB_VALIDATION, "null argument");
        if (comm_active(comm)) device = comm->device;
        if (precision == LCB_FP32)
            ascend_rows_host<float>(comm, n, row_begin, row_end, offsets, adjacency, values, l, B, alpha, iterations,
                                    momentum, early_exit != 0, device, err_iter, err_member);
        else
            ascend_rows_host<double>(comm, n, row_begin, row_end, offsets, adjacency, values, l, B, alpha, iterations,
                                     momentum, early_exit != 0, device, err_iter, err_member);
    });
}

int lcb_cut_values(const lcb_graph* g, const uint8_t* z, int64_t count, int64_t* cuts) {
    return guard([&] {
        if (!g) fail(LCB_VALIDATION, "null graph");
        const DevGraph& G = g->g;
        const size_t cells = static_cast<size_t>(count) * G.n;
        for (size_t i = 0; i < cells; ++i)
            if (z[i] > 1) fail(LCB_VALIDATION, "cut_value: assignment entries must be 0 or 1");
        if (count < 1) return;
        DeviceScope ds(G.device);
        PooledWork<double> pw(G.device);
        Work<double>& w = *pw;
        uint8_t* dz = reinterpret_cast<uint8_t*>(w.hostbatch.ensure((cells + 7) / 8));
        h2d(dz, z, cells, w.st);
        const int words = static_cast<int>((count + 31) / 32);
        uint32_t* Z = w.Z.ensure(static_cast<size_t>(words) * G.n);
        launch_pack_bytes(dz, G.n, static_cast<int>(count), Z, w.st);
        unsigned long long* c = w.cuts.ensure(static_cast<size_t>(words) * 32);
        launch_cut_count(G, Z, words, c, w.st);
        std::vector<unsigned long long> h(static_cast<size_t>(words) * 32);
        d2h(h.data(), c, sizeof(unsigned long long) * h.size(), w.st);
        CK(cudaStreamSynchronize(w.st));
        CK(cudaGetLastError());
        for (int64_t i = 0; i < count; ++i) cuts[i] = static_cast<int64_t>(h[static_cast<size_t>(i)]);
    });
}

int lcb_brute_force_maxcut(const lcb_graph* g, int32_t max_nodes, int64_t* optimum, int64_t* count_optimal,
                           uint8_t* witness) {
    return guard([&] {
        if (!g || !optimum) fail(LCB_VALIDATION, "null argument");
        const DevGraph& G = g->g;
        const int guard_n = max_nodes > 0 ? max_nodes : 26;  // oracle.cpp:53-55
        if (guard_n > 40) fail(LCB_VALIDATION, "brute_force_maxcut: max_nodes above 40 is out of reach");
        if (G.n > guard_n)
            fail(LCB_VALIDATION, "brute_force_maxcut: n = " + std::to_string(G.n) +
                                     " exceeds the exhaustive-scan guard (" + std::to_string(guard_n) + ")");
        const int n = G.n;
        const HostCSR hc = fetch_csr(G);
        // neighbour masks, one layer per multiplicity level (a raw CSR may repeat entries)
        const int max_layers = brute_force_max_layers();
        std::vector<uint64_t> masks(static_cast<size_t>(max_layers) * n, 0), upper(masks.size(), 0);
        std::vector<int> deg(static_cast<size_t>(n));
        int layers = 1;
        for (int u = 0; u < n; ++u) {
            deg[static_cast<size_t>(u)] = hc.off[static_cast<size_t>(u) + 1] - hc.off[static_cast<size_t>(u)];
            for (int k = hc.off[static_cast<size_t>(u)]; k < hc.off[static_cast<size_t>(u) + 1]; ++k) {
                const int v = hc.adj[static_cast<size_t>(k)];
                int layer = 0;
                while (layer < max_layers && (masks[static_cast<size_t>(layer) * n + u] >> v & 1ull)) ++layer;
                if (layer == max_layers) fail(LCB_VALIDATION, "brute_force_maxcut: edge multiplicity above 4");
                masks[static_cast<size_t>(layer) * n + u] |= 1ull << v;
                if (v > u) upper[static_cast<size_t>(layer) * n + u] |= 1ull << v;
                layers = std::max(layers, layer + 1);
            }
        }
        DeviceScope ds(G.device);
        PooledWork<double> pw(G.device);
        Work<double>& w = *pw;
        const size_t mwords = static_cast<size_t>(layers) * n;
        const size_t dwords = (static_cast<size_t>(n) + 1) / 2;
        const size_t swords = (brute_force_scratch_bytes() + 7) / 8;
        uint64_t* d = w.bf.ensure(2 * mwords + dwords + swords + 1);
        uint64_t* dm = d;
        uint64_t* du = d + mwords;
        int* dd = reinterpret_cast<int*>(d + 2 * mwords);
        void* scratch = d + 2 * mwords + dwords + 1;
        h2d(dm, masks.data(), sizeof(uint64_t) * mwords, w.st);
        h2d(du, upper.data(), sizeof(uint64_t) * mwords, w.st);
        h2d(dd, deg.data(), sizeof(int) * static_cast<size_t>(n), w.st);
        const void* fin = launch_brute_force(dm, du, dd, n, layers, scratch, w.st);
        unsigned long long rec[3];
        d2h(rec, fin, sizeof(rec), w.st);
        CK(cudaStreamSynchronize(w.st));
        CK(cudaGetLastError());
        *optimum = static_cast<int64_t>(static_cast<long long>(rec[0]));
        if (count_optimal) *count_optimal = static_cast<int64_t>(rec[1]);
        if (witness)
            for (int v = 0; v < n; ++v) witness[v] = static_cast<uint8_t>((rec[2] >> v) & 1ull);
    });
}

int lcb_round_cut_batch(const lcb_graph* g, const double* values, int32_t l, int64_t B, int32_t lifted,
                        int64_t* cuts, int64_t* best_member, int64_t* best_cut, uint8_t* best_z) {
    return guard([&] {
        if (!g) fail(LCB_VALIDATION, "null graph");
        const DevGraph& G = g->g;
        if (l < 1 || B < 1) fail(LCB_VALIDATION, "DenseState: n, l, B must all be >= 1");
        DeviceScope ds(G.device);
        PooledWork<double> pw(G.device);
        Work<double>& w = *pw;
        const int W = static_cast<int>(B * l);
        w.shape(G.n, W);
        const size_t cells = static_cast<size_t>(W) * G.n;
        double* d = w.hostbatch.ensure(cells);
        h2d(d, values, sizeof(double) * cells, w.st);
        launch_transpose_in<double>(d, w.X[0].p, G.n, W, w.ld, w.st);
        const int words = static_cast<int>((B + 31) / 32);
        uint32_t* Z = w.Z.ensure(static_cast<size_t>(words) * G.n);
        unsigned long long* c = w.cuts.ensure(static_cast<size_t>(words) * 32 + 1);
        unsigned long long* key = w.keys.ensure(8);
        uint32_t* bits = w.win.ensure((G.n + 31) / 32);
        launch_epilogue<double>(G, w.X[0].p, w.ld, static_cast<int>(B), l, lifted ? 1 : 0, Z, c, static_cast<int>(B), 0,
                                key, bits, w.st);
        std::vector<unsigned long long> hc(static_cast<size_t>(B));
        d2h(hc.data(), c, sizeof(unsigned long long) * B, w.st);
        d2h(w.h_keys, key, sizeof(unsigned long long), w.st);
        std::vector<uint32_t> hb((G.n + 31) / 32);
        d2h(hb.data(), bits, sizeof(uint32_t) * hb.size(), w.st);
        CK(cudaStreamSynchronize(w.st));
        CK(cudaGetLastError());
        if (cuts)
            for (int64_t j = 0; j < B; ++j) cuts[j] = static_cast<int64_t>(hc[static_cast<size_t>(j)]);
        const unsigned long long k = w.h_keys[0];
        if (best_cut) *best_cut = static_cast<int64_t>(k >> 32);
        if (best_member) *best_member = static_cast<int64_t>(0xffffffffull - (k & 0xffffffffull));
        if (best_z)
            for (int v = 0; v < G.n; ++v) best_z[v] = static_cast<uint8_t>((hb[v >> 5] >> (v & 31)) & 1u);
    });
}

int lcb_round(int device, const double* values, int64_t n, int32_t l, int64_t B, int32_t lifted, uint8_t* z) {
    return guard([&] {
        if (!values || !z) fail(LCB_VALIDATION, "null argument");
        if (n < 1 || l < 1 || B < 1) fail(LCB_VALIDATION, "DenseState: n, l, B must all be >= 1");
        if (static_cast<int64_t>(l) * B > (1 << 26) || n > 0x7fffffff) fail(LCB_VALIDATION, "batch too wide");
        DeviceScope ds(device);
        PooledWork<double> pw(device);
        Work<double>& w = *pw;
        const int W = static_cast<int>(B * l), N = static_cast<int>(n);
        w.shape(N, W);
        const size_t cells = static_cast<size_t>(W) * N;
        double* d = w.hostbatch.ensure(cells);
        h2d(d, values, sizeof(double) * cells, w.st);
        launch_transpose_in<double>(d, w.X[0].p, N, W, w.ld, w.st);
        const int words = static_cast<int>((B + 31) / 32);
        uint32_t* Z = w.Z.ensure(static_cast<size_t>(words) * N);
        launch_round_pack<double>(w.X[0].p, w.ld, N, static_cast<int>(B), l, lifted ? 1 : 0, Z, w.st);
        uint8_t* dz = reinterpret_cast<uint8_t*>(w.Y.ensure((static_cast<size_t>(B) * N + 7) / 8));
        launch_unpack_members(Z, N, static_cast<int>(B), dz, w.st);
        d2h(z, dz, static_cast<size_t>(B) * N, w.st);
        CK(cudaStreamSynchronize(w.st));
        CK(cudaGetLastError());
    });
}

static void init_mean_host(const DevGraph& G, int method, double beta, int l, const uint64_t* ck,
                           double scale, double* out) {
    DeviceScope ds(G.device);
    PooledWork<double> pw(G.device);
        Work<double>& w = *pw;
    uint64_t* dck = w.colkeys.ensure(static_cast<size_t>(l));
    h2d(dck, ck, sizeof(uint64_t) * l, w.st);
    double* mean = w.mean.ensure(static_cast<size_t>(G.n) * l);
    if (method == 0) {
        if (G.max_degree < 1) fail(LCB_VALIDATION, "dui_init: graph has no edges (MaxCut is trivially 0)");
        launch_dui(G, dck, l, scale, nullptr, mean, w.st);
    } else {
        const double thr = G.deg_mean + beta * G.deg_sd;
        launch_idi(G, thr, dck, l, scale, nullptr, w.sign.ensure(static_cast<size_t>(G.n) * l), mean, w.st);
    }
    d2h(out, mean, sizeof(double) * G.n * l, w.st);
    CK(cudaStreamSynchronize(w.st));
    CK(cudaGetLastError());
}

int lcb_dui_init(const lcb_graph* g, uint64_t key, double* x) {
    return guard([&] { init_mean_host(g->g, 0, 0.2, 1, &key, 1.0, x); });
}

int lcb_idi_init(const lcb_graph* g, double beta, uint64_t key, double* x) {
    return guard([&] { init_mean_host(g->g, 1, beta, 1, &key, 1.0, x); });
}

int lcb_lifted_init_mean(const lcb_graph* g, int32_t method, double beta, int32_t l, uint64_t key,
                         double* mean) {
    return guard([&] {
        if (l < 1) fail(LCB_VALIDATION, "lift_dim must be >= 1");
        std::vector<uint64_t> ck(static_cast<size_t>(l));
        for (int c = 0; c < l; ++c) ck[c] = split2(key, 0x636fu, static_cast<uint64_t>(c));
        init_mean_host(g->g, method, beta, l, ck.data(), 1.0, mean);
    });
}

int lcb_gaussian_batch(int device, const double* mean, int64_t n, int32_t l, double eta, int64_t B,
                       uint64_t key, double* out) {
    return guard([&] {
        if (eta <= 0.0) fail(LCB_VALIDATION, "gaussian_batch: eta must be > 0");
        if (n < 1 || l < 1 || B < 1) fail(LCB_VALIDATION, "DenseState: n, l, B must all be >= 1");
        DeviceScope ds(device);
        PooledWork<double> pw(device);
        Work<double>& w = *pw;
        const int W = static_cast<int>(B * l);
        w.shape(static_cast<int>(n), W);
        double* dm = w.mean.ensure(static_cast<size_t>(n) * l);
        h2d(dm, mean, sizeof(double) * n * l, w.st);
        std::vector<uint64_t> mk(static_cast<size_t>(B));
        for (int64_t j = 0; j < B; ++j) mk[j] = split2(key, 0x6d62u, static_cast<uint64_t>(j));
        uint64_t* dk = w.mkeys.ensure(mk.size());
        h2d(dk, mk.data(), sizeof(uint64_t) * mk.size(), w.st);
        launch_gaussian<double>(w.X[0].p, w.V.p, w.ld, static_cast<int>(n), static_cast<int>(B), l, dk, dm,
                                nullptr, 1.0, std::sqrt(eta), w.st);
        double* d = w.hostbatch.ensure(static_cast<size_t>(W) * n);
        launch_transpose_out<double>(w.X[0].p, d, static_cast<int>(n), W, w.ld, w.st);
        d2h(out, d, sizeof(double) * W * n, w.st);
        CK(cudaStreamSynchronize(w.st));
        CK(cudaGetLastError());
    });
}

int lcb_gaussian_batch_exact(const double* mean, int64_t n, int32_t l, double eta, int64_t B, uint64_t key,
                             double* out) {
    return guard([&] {
        if (eta <= 0.0) fail(LCB_VALIDATION, "gaussian_batch: eta must be > 0");
        if (n < 1 || l < 1 || B < 1) fail(LCB_VALIDATION, "DenseState: n, l, B must all be >= 1");
        if (!mean || !out) fail(LCB_VALIDATION, "null argument");
        // the stream seeding of init.cpp:69-87 (member j: split(key, {0x6d62, j}), counters 2k,
        // 2k+1 Box-Muller with the host libm), members on host threads; bit-identical
        const size_t entries = static_cast<size_t>(n) * static_cast<size_t>(l);
        const double noise = std::sqrt(eta);
        auto gen = [&](int64_t j0, int64_t j1) {
            for (int64_t j = j0; j < j1; ++j) {
                HostStream ms{split2(key, 0x6d62u, static_cast<uint64_t>(j))};
                double* o = out + static_cast<size_t>(j) * entries;
                for (size_t k = 0; k < entries; ++k) {
                    const double x = mean[k] + noise * ms.normal();
                    o[k] = x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x);
                }
            }
        };
        const int64_t nt = std::min<int64_t>(B, std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
        if (nt <= 1 || entries * static_cast<size_t>(B) < (1u << 16)) {
            gen(0, B);
            return;
        }
        std::vector<std::thread> th;
        for (int64_t t = 1; t < nt; ++t) th.emplace_back(gen, B * t / nt, B * (t + 1) / nt);
        gen(0, B / nt);
        for (auto& t : th) t.join();
    });
}

int lcb_solve(const lcb_graph* g, const lcb_config* cfg, uint64_t seed, int32_t per_component,
              const lcb_run_opts* opts, lcb_outcome* out, uint8_t* assignment, lcb_batch_trace* bt,
              int64_t bt_cap, lcb_phase_trace* pt, int64_t pt_cap, lcb_search_trace* st, int64_t st_cap) {
    return guard([&] {
        if (!g || !cfg || !out || !assignment) fail(LCB_VALIDATION, "null argument");
        validate_config(*cfg);
        lcb_run_opts o{};
        o.precision = LCB_FP64;
        o.host_init = -1;
        if (opts) o = *opts;
        DeviceScope ds(g->g.device);
        TraceSinks sinks{bt, bt ? bt_cap : 0, pt, pt ? pt_cap : 0, st, st ? st_cap : 0};
        if (o.precision == LCB_FP32)
            solve_top<float>(g->g, *cfg, seed, per_component, o, *out, assignment, sinks);
        else
            solve_top<double>(g->g, *cfg, seed, per_component, o, *out, assignment, sinks);
    });
}

int lcb_debug_resident_layout(const lcb_graph* g, int64_t* len, uint16_t* col, uint16_t* col_fast,
                              int64_t* row_words, int32_t* perm) {
    return guard([&] {
        if (!g || !len) fail(LCB_VALIDATION, "null argument");
        const DevGraph& G = g->g;
        *len = G.res_info ? G.res_len : 0;
        if (!G.res_info) return;
        DeviceScope ds(G.device);
        if (col) CK(cudaMemcpy(col, G.res_col, sizeof(uint16_t) * G.res_len, cudaMemcpyDeviceToHost));
        if (col_fast) {
            if (G.res_col_fast)
                CK(cudaMemcpy(col_fast, G.res_col_fast, sizeof(uint16_t) * G.res_len, cudaMemcpyDeviceToHost));
            else
                std::memset(col_fast, 0xff, sizeof(uint16_t) * G.res_len);
        }
        if (perm) CK(cudaMemcpy(perm, G.res_perm, sizeof(int) * G.n, cudaMemcpyDeviceToHost));
        if (row_words) {  // relabelled row r: (first 4-column word, degree)
            const int H = G.res_nheavy;
            std::vector<int> hi(static_cast<size_t>(2 * std::max(H, 1)));
            std::vector<uint32_t> info(static_cast<size_t>(std::max(G.n - H, 1)));
            CK(cudaMemcpy(hi.data(), G.res_heavy, sizeof(int) * hi.size(), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(info.data(), G.res_info, sizeof(uint32_t) * info.size(), cudaMemcpyDeviceToHost));
            for (int r = 0; r < G.n; ++r) {
                if (r < H) {
                    row_words[2 * r] = hi[static_cast<size_t>(2 * r)];
                    row_words[2 * r + 1] = hi[static_cast<size_t>(2 * r + 1)];
                } else {
                    const uint32_t pk = info[static_cast<size_t>(r - H)];
                    row_words[2 * r] = pk >> 8;
                    row_words[2 * r + 1] = pk & 0xffu;
                }
            }
        }
    });
}

int lcb_solve_runs(const lcb_graph* g, const lcb_config* cfg, const uint64_t* seeds, int64_t nruns,
                   int32_t per_component, const lcb_run_opts* opts, int64_t* run_cuts, int64_t* best_run,
                   lcb_outcome* best_out, uint8_t* assignment) {
    return guard([&] {
        if (!g || !cfg || !seeds || !best_out || !assignment) fail(LCB_VALIDATION, "null argument");
        if (nruns < 1) fail(LCB_VALIDATION, "solve_runs: need at least one run");
        validate_config(*cfg);
        lcb_run_opts o{};
        o.precision = LCB_FP64;
        o.host_init = -1;
        if (opts) o = *opts;
        lcb_comm* comm = o.comm;
        o.comm = nullptr;  // runs are independent: each is solved on one rank (bench.cpp:97-136)
        const int nr = comm ? comm->nranks : 1, rk = comm ? comm->rank : 0;
        const DevGraph& G = g->g;
        DeviceScope ds(G.device);
        const int words = (G.n + 31) / 32;
        std::vector<unsigned long long> enc(static_cast<size_t>(nruns), 0ull);  // cut + 1 where owned
        std::vector<uint8_t> z(static_cast<size_t>(G.n)), zbest(static_cast<size_t>(G.n), 0);
        lcb_outcome local_best{};
        int64_t local_run = -1, local_cut = -1;
        // measurement out-params accumulate over this rank's runs
        double acc_step_ms = 0, acc_bytes = 0, acc_solve_ms = 0, acc_k[12] = {0};
        int64_t acc_launches = 0, acc_updates = 0;
        for (int64_t i = rk; i < nruns; i += nr) {
            lcb_outcome out{};
            TraceSinks sinks{nullptr, 0, nullptr, 0, nullptr, 0};
            double r_step_ms = 0, r_bytes = 0, r_solve_ms = 0, r_k[12] = {0};
            int64_t r_launches = 0, r_updates = 0;
            lcb_run_opts ro = o;
            ro.step_ms = &r_step_ms;
            ro.step_bytes = &r_bytes;
            ro.solve_ms = &r_solve_ms;
            ro.kernel_stats = r_k;
            ro.step_launches = &r_launches;
            ro.node_updates = &r_updates;
            if (o.precision == LCB_FP32)
                solve_top<float>(G, *cfg, seeds[i], per_component, ro, out, z.data(), sinks);
            else
                solve_top<double>(G, *cfg, seeds[i], per_component, ro, out, z.data(), sinks);
            acc_step_ms += r_step_ms;
            acc_bytes += r_bytes;
            acc_solve_ms += r_solve_ms;
            acc_launches += r_launches;
            acc_updates += r_updates;
            for (int k = 0; k < 12; ++k) acc_k[k] += r_k[k];
            enc[static_cast<size_t>(i)] = static_cast<unsigned long long>(out.cut_value) + 1ull;
            if (out.cut_value > local_cut) {
                local_cut = out.cut_value;
                local_run = i;
                local_best = out;
                zbest = z;
            }
        }
        // one exchange: per-run cuts, then the winner's outcome and assignment (zeros elsewhere)
        const size_t ow = (sizeof(lcb_outcome) + 7) / 8;
        const size_t total = static_cast<size_t>(nruns) + ow + 2 * static_cast<size_t>(words);
        unsigned long long* d = nullptr;
        CK(cudaMalloc(&d, sizeof(unsigned long long) * total));
        struct Free {
            void* p;
            ~Free() { cudaFree(p); }
        } fr{d};
        cudaStream_t st = nullptr;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        struct SFree {
            cudaStream_t s;
            ~SFree() { cudaStreamDestroy(s); }
        } sf{st};
        h2d(d, enc.data(), sizeof(unsigned long long) * enc.size(), st);
        comm_allreduce(comm, d, static_cast<size_t>(nruns), 8, true, st, "allreduce(run cuts)");
        d2h(enc.data(), d, sizeof(unsigned long long) * enc.size(), st);
        CK(cudaStreamSynchronize(st));
        int64_t win = 0;
        for (int64_t i = 1; i < nruns; ++i)
            if (enc[static_cast<size_t>(i)] > enc[static_cast<size_t>(win)]) win = i;  // first maximum
        std::vector<unsigned long long> pay(ow + 2 * static_cast<size_t>(words), 0ull);
        if (win % nr == rk) {
            std::memcpy(pay.data(), &local_best, sizeof(lcb_outcome));
            uint32_t* bits = reinterpret_cast<uint32_t*>(pay.data() + ow);
            for (int v = 0; v < G.n; ++v)
                if (zbest[static_cast<size_t>(v)]) bits[v >> 5] |= 1u << (v & 31);
            if (local_run != win) fail(LCB_ERROR, "solve_runs: winner bookkeeping");
        }
        h2d(d + nruns, pay.data(), sizeof(unsigned long long) * pay.size(), st);
        comm_allreduce(comm, d + nruns, pay.size(), 8, true, st, "allreduce(winner)");
        d2h(pay.data(), d + nruns, sizeof(unsigned long long) * pay.size(), st);
        CK(cudaStreamSynchronize(st));
        std::memcpy(best_out, pay.data(), sizeof(lcb_outcome));
        const uint32_t* bits = reinterpret_cast<const uint32_t*>(pay.data() + ow);
        for (int v = 0; v < G.n; ++v) assignment[v] = static_cast<uint8_t>((bits[v >> 5] >> (v & 31)) & 1u);
        if (run_cuts)
            for (int64_t i = 0; i < nruns; ++i) run_cuts[i] = static_cast<int64_t>(enc[static_cast<size_t>(i)]) - 1;
        if (best_run) *best_run = win;
        if (o.step_ms) *o.step_ms = acc_step_ms;
        if (o.step_bytes) *o.step_bytes = acc_bytes;
        if (o.solve_ms) *o.solve_ms = acc_solve_ms;
        if (o.step_launches) *o.step_launches = acc_launches;
        if (o.node_updates) *o.node_updates = acc_updates;
        if (o.kernel_stats) std::memcpy(o.kernel_stats, acc_k, sizeof(acc_k));
    });
}

int lcb_loopback_create(int32_t nranks, lcb_loopback** out) {
    return guard([&] {
        if (nranks < 1 || !out) fail(LCB_VALIDATION, "bad nranks");
        *out = new lcb_loopback(nranks);
    });
}

void lcb_loopback_destroy(lcb_loopback* g) { delete g; }

int lcb_comm_create_loopback(lcb_loopback* group, int32_t rank, int device, lcb_comm** out) {
    return guard([&] {
        if (!group || !out) fail(LCB_VALIDATION, "null argument");
        if (rank < 0 || rank >= group->g.nranks) fail(LCB_VALIDATION, "bad rank / nranks");
        auto c = std::make_unique<lcb_comm>();
        c->loop = &group->g;
        c->nranks = group->g.nranks;
        c->rank = rank;
        c->device = device;
        *out = c.release();
    });
}

int lcb_comm_unique_id(uint8_t id[128]) {
    return guard([&] {
        if (!nccl().ok) fail(LCB_CUDA, "NCCL unavailable: " + nccl().why);
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        static_assert(sizeof(u) == 128, "ncclUniqueId size");
        std::memcpy(id, &u, 128);
    });
}

int lcb_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int device, lcb_comm** out) {
    return guard([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(LCB_VALIDATION, "bad rank / nranks");
        auto c = std::make_unique<lcb_comm>();
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        const char* force = std::getenv("LCB_FORCE_NCCL");  // 1-rank communicator: exercise the NCCL path
        if (nranks > 1 || (force && force[0] == '1')) {
            if (!nccl().ok) fail(LCB_CUDA, "NCCL unavailable: " + nccl().why);
            DeviceScope ds(device);
            ncclUniqueId u;
            std::memcpy(&u, id, 128);
            nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
        }
        *out = c.release();
    });
}

void lcb_comm_destroy(lcb_comm* c) {
    if (!c) return;
    if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
    delete c;
}

void lcb_release_workspaces(void) {
    for (auto* fl : {&WorkPool<float>::get().free_list}) {
        std::lock_guard<std::mutex> lk(WorkPool<float>::get().mu);
        fl->clear();
    }
    {
        std::lock_guard<std::mutex> lk(WorkPool<double>::get().mu);
        WorkPool<double>::get().free_list.clear();
    }
    // and the cached stream-ordered pool of graph arrays / ingest scratch on every device
    int ndev = 0, cur = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cudaGetDevice(&cur) != cudaSuccess) return;
    for (int d = 0; d < ndev; ++d) {
        cudaMemPool_t pool;
        if (cudaSetDevice(d) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
            cudaDeviceSynchronize();
            cudaMemPoolTrimTo(pool, 0);
        }
    }
    cudaSetDevice(cur);
}

void lcb_counters(int64_t* launches, int64_t* h2d_bytes, int64_t* d2h_bytes) {
    if (launches) *launches = g_launches.load();
    if (h2d_bytes) *h2d_bytes = g_h2d.load();
    if (d2h_bytes) *d2h_bytes = g_d2h.load();
}

uint64_t lcb_pack_key(int64_t cut, int64_t global_member) {
    return (static_cast<uint64_t>(cut) << 32) | (0xffffffffull - static_cast<uint64_t>(global_member));
}

void lcb_unpack_key(uint64_t key, int64_t* cut, int64_t* global_member) {
    *cut = static_cast<int64_t>(key >> 32);
    *global_member = static_cast<int64_t>(0xffffffffull - (key & 0xffffffffull));
}

}  // extern "C"
