// lcb_kernels.cu — sm_100a kernels of the liftcut PGA hot path.
//
// Data layout in HBM: the batch is node-major, X[v][col] with
// col = member * l + c (the transpose of DenseState's [B][l][n], dense_state.hpp:50-54),
// rows padded to a multiple of the warp span so every gather is a 512-B (fp32) or
// 256-B... per-slab coalesced vector load.  Velocity V has the same layout; X is
// double-buffered across iterations (Jacobi update, ascent.cpp:58-77 reads the old
// iterate for all rows).
//
// fp64 kernels use explicit round-to-nearest intrinsics and sequential CSR-order
// sums per (row, column) so they reproduce the reference's scalar, FMA-free
// arithmetic bit for bit (graph.cpp:116-121, ascent.cpp:66-77).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "lcb_internal.h"

namespace lcb {

namespace {

template <typename T>
struct Vec;
template <>
struct Vec<float> {
    using type = float4;
    static constexpr int E = 4;
};
template <>
struct Vec<double> {
    using type = double2;
    static constexpr int E = 2;
};

__device__ __forceinline__ float& el(float4& v, int e) { return (&v.x)[e]; }
__device__ __forceinline__ double& el(double2& v, int e) { return (&v.x)[e]; }
__device__ __forceinline__ float el(const float4& v, int e) { return (&v.x)[e]; }
__device__ __forceinline__ double el(const double2& v, int e) { return (&v.x)[e]; }

__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }

template <typename V>
__device__ __forceinline__ V ldg_vec(const V* p) {
    return __ldg(p);
}

template <typename T>
__device__ __forceinline__ T clamp1(T r) {
    return r < T(-1) ? T(-1) : (r > T(1) ? T(1) : r);
}

constexpr int kWarps = 8;  // warps per block of the step kernel (one row each)
#ifndef LCB_UNROLL
#define LCB_UNROLL 4
#endif
#ifndef LCB_MINB
#define LCB_MINB 1
#endif
#ifndef LCB_HOIST
#define LCB_HOIST 0
#endif
#ifndef LCB_PRED
#define LCB_PRED 0
#endif

// ---------------------------------------------------------------------------
// K1: fused PGA step, HBM-streaming.  A warp owns R rows x one column slab-group
// (S 16-byte vectors per lane).  Rows are taken in degree-descending order
// (hubs first, BA degree skew) through one 16-byte slot record {row, begin, end},
// so a row's dependent chain is slot record -> column indices -> neighbour
// gathers; the R rows' gathers are interleaved to keep more bytes in flight.
//   GEN = per-member alpha / iteration limit (batched search) or early exit
//   EE  = early-exit bits (implies GEN)
// ---------------------------------------------------------------------------
template <typename T, int S, int R, bool GEN, bool EE, int MODE>
__global__ void __launch_bounds__(kWarps * 32, LCB_MINB)
    k_step(StepArgs<T> a, int groups) {
    constexpr int E = Vec<T>::E;
    using V = typename Vec<T>::type;
    constexpr int SPAN = 32 * S * E;
    __shared__ uint32_t sbits[EE ? SPAN : 1];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int group = blockIdx.x % groups;
    const int slot0 = ((blockIdx.x / groups) * kWarps + warp) * R;

    if constexpr (EE) {
        for (int i = threadIdx.x; i < SPAN; i += blockDim.x) sbits[i] = 0;
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < a.members; i += blockDim.x) a.flags_zero[i] = 0;
        __syncthreads();
    }

    const int c0 = group * SPAN + lane * E;
    int4 si[R];
    bool live[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        live[i] = slot0 + i < a.n;
        si[i] = live[i] ? __ldg(a.slots + slot0 + i) : make_int4(0, 0, 0, 0);
    }

    // self iterate and velocity do not depend on the gathers: issue them first
    V xself[R][S], vself[R][S];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int64_t rb = static_cast<int64_t>(si[i].x) * a.ld + c0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (LCB_HOIST && live[i]) {
                xself[i][s] = ldg_vec(reinterpret_cast<const V*>(a.x_in + rb + s * 32 * E));
                if constexpr (MODE == MODE_STEP) vself[i][s] = *reinterpret_cast<const V*>(a.vel + rb + s * 32 * E);
            }
        }
    }

    V acc[R][S];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int e = 0; e < E; ++e) el(acc[i][s], e) = T(0);

    const T* xin = a.x_in + c0;
    int len[R];
    int maxlen = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        len[i] = si[i].z - si[i].y;
        maxlen = max(maxlen, len[i]);
    }
    for (int base = 0; base < maxlen; base += 32) {
        int mycol[R], cnt[R];
        int cmax = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            cnt[i] = min(32, len[i] - base);
            mycol[i] = lane < cnt[i] ? __ldg(a.col + si[i].y + base + lane) : 0;
            cmax = max(cmax, cnt[i]);
        }
        if (R == 1 && !LCB_PRED) {
            int k = 0;
            for (; k + 4 <= cnt[0]; k += 4) {
                V v[4][S];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int u = __shfl_sync(0xffffffffu, mycol[0], k + q);
                    const V* p = reinterpret_cast<const V*>(xin + static_cast<int64_t>(u) * a.ld);
#pragma unroll
                    for (int s = 0; s < S; ++s) v[q][s] = ldg_vec(p + s * 32);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int s = 0; s < S; ++s)
#pragma unroll
                        for (int e = 0; e < E; ++e) el(acc[0][s], e) = radd(el(acc[0][s], e), el(v[q][s], e));
            }
            for (; k < cnt[0]; ++k) {
                const int u = __shfl_sync(0xffffffffu, mycol[0], k);
                const V* p = reinterpret_cast<const V*>(xin + static_cast<int64_t>(u) * a.ld);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const V v = ldg_vec(p + s * 32);
#pragma unroll
                    for (int e = 0; e < E; ++e) el(acc[0][s], e) = radd(el(acc[0][s], e), el(v, e));
                }
            }
            continue;
        }
        for (int k = 0; k < cmax; k += 4) {
            V v[R][4][S];
#pragma unroll
            for (int i = 0; i < R; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int u = __shfl_sync(0xffffffffu, mycol[i], (k + q) & 31);
                    if (k + q < cnt[i]) {  // warp-uniform predicate
                        const V* p = reinterpret_cast<const V*>(xin + static_cast<int64_t>(u) * a.ld);
#pragma unroll
                        for (int s = 0; s < S; ++s) v[i][q][s] = ldg_vec(p + s * 32);
                    }
                }
            // sequential CSR order per element (graph.cpp:118)
#pragma unroll
            for (int i = 0; i < R; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (k + q < cnt[i])
#pragma unroll
                        for (int s = 0; s < S; ++s)
#pragma unroll
                            for (int e = 0; e < E; ++e)
                                el(acc[i][s], e) = radd(el(acc[i][s], e), el(v[i][q][s], e));
        }
    }

#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (!live[i]) continue;
        const int row = si[i].x;
        const T dg = static_cast<T>(len[i]);
        const int64_t rb = static_cast<int64_t>(row) * a.ld + c0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int64_t off = rb + s * 32 * E;
            if (!LCB_HOIST) {
                xself[i][s] = ldg_vec(reinterpret_cast<const V*>(a.x_in + off));
                if constexpr (MODE == MODE_STEP) vself[i][s] = *reinterpret_cast<const V*>(a.vel + off);
            }
            const V xv = xself[i][s];
            if constexpr (MODE == MODE_LAPLACE) {
                V y;
#pragma unroll
                for (int e = 0; e < E; ++e) el(y, e) = rsub(rmul(dg, el(xv, e)), el(acc[i][s], e));
                *reinterpret_cast<V*>(a.x_out + off) = y;
            } else {
                V vv = vself[i][s];
                V xo;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int colx = c0 + s * 32 * E + e;
                    const T x = el(xv, e);
                    bool act = colx < a.W;
                    T alpha = a.alpha_uniform;
                    int m = 0;
                    if constexpr (GEN) {
                        if (act) {
                            m = colx / a.l;
                            if (a.tlim) act = a.it < __ldg(a.tlim + m);
                            if constexpr (EE) {
                                if (act && a.it > 0) act = ex_continue(__ldcg(a.flags_prev + m));
                            }
                            if (a.alpha) alpha = __ldg(a.alpha + m);
                        }
                    } else {
                        m = colx / a.l;
                    }
                    if (act) {
                        const T y = rsub(rmul(dg, x), el(acc[i][s], e));  // Lx  (graph.cpp:120)
                        const T v = radd(rmul(a.mu, el(vv, e)), y);        // ascent.cpp:68
                        const T raw = radd(x, rmul(alpha, v));             // ascent.cpp:69
                        if (!isfinite(raw))                                // ascent.cpp:70-72
                            atomicMin(a.err, (static_cast<unsigned long long>(m) << 32) |
                                                 static_cast<unsigned>(a.it));
                        const T cl = clamp1(raw);                          // ascent.cpp:73
                        if constexpr (EE) {
                            const T ch = fabs(rsub(cl, x));
                            uint32_t b = 0;
                            if (ch > T(1e-12)) b |= EX_BIG;
                            if (ch > T(0)) b |= EX_NZ;
                            if (cl != T(1) && cl != T(-1)) b |= EX_NOTB;
                            if (b) atomicOr(&sbits[s * 32 * E + lane * E + e], b);
                        }
                        el(xo, e) = cl;
                        el(vv, e) = v;
                    } else {
                        el(xo, e) = x;
                    }
                }
                *reinterpret_cast<V*>(a.x_out + off) = xo;
                *reinterpret_cast<V*>(a.vel + off) = vv;
            }
        }
    }

    if constexpr (EE) {
        __syncthreads();
        for (int i = threadIdx.x; i < SPAN; i += blockDim.x) {
            const uint32_t b = sbits[i];
            const int colx = group * SPAN + i;
            if (b && colx < a.W) {
                const int m = colx / a.l;
                const uint32_t f = __ldcg(a.flags_cur + m);
                if ((f & b) != b) atomicOr(a.flags_cur + m, b);
            }
        }
    }
}

template <typename T>
int pick_s(int W) {
    static int forced = [] {
        const char* e = std::getenv("LCB_STEP_S");
        return e ? std::atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    constexpr int E = Vec<T>::E;
    (void)E;
    (void)W;
    return 1;  // measured best on B200 for W in {1024, 2048} (profiles/)
}

int pick_r() {
    static int r = [] {
        const char* e = std::getenv("LCB_ROWS");
        const int v = e ? std::atoi(e) : 1;  // R=2 measured slower: the kernel is L2-bandwidth-bound
        return v == 1 ? 1 : 2;
    }();
    return r;
}

template <typename T, bool GEN, bool EE, int MODE>
void dispatch_s(const StepArgs<T>& a, int S, cudaStream_t st) {
    constexpr int E = Vec<T>::E;
    const int R = pick_r();
    auto go = [&](auto sconst, auto rconst) {
        constexpr int SS = decltype(sconst)::value;
        constexpr int RR = decltype(rconst)::value;
        constexpr int SPAN = 32 * SS * E;
        const int groups = static_cast<int>((a.ld + SPAN - 1) / SPAN);
        const int rows_blocks = (a.n + kWarps * RR - 1) / (kWarps * RR);
        const dim3 grid(static_cast<unsigned>(rows_blocks) * groups);
        count_launch();
        k_step<T, SS, RR, GEN, EE, MODE><<<grid, kWarps * 32, 0, st>>>(a, groups);
    };
    if (S == 2) {
        if (R == 1) go(std::integral_constant<int, 2>{}, std::integral_constant<int, 1>{});
        else go(std::integral_constant<int, 2>{}, std::integral_constant<int, 2>{});
    } else {
        if (R == 1) go(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
        else go(std::integral_constant<int, 1>{}, std::integral_constant<int, 2>{});
    }
}

}  // namespace

template <typename T>
int step_span(int W) {
    return 32 * pick_s<T>(W) * Vec<T>::E;
}

template <typename T>
void launch_step(const StepArgs<T>& a, bool early_exit, int mode, cudaStream_t s) {
    const int S = pick_s<T>(a.W);
    if (mode == MODE_LAPLACE)
        dispatch_s<T, false, false, MODE_LAPLACE>(a, S, s);
    else if (early_exit)
        dispatch_s<T, true, true, MODE_STEP>(a, S, s);
    else if (a.tlim != nullptr || a.alpha != nullptr)
        dispatch_s<T, true, false, MODE_STEP>(a, S, s);
    else
        dispatch_s<T, false, false, MODE_STEP>(a, S, s);
}

template int step_span<float>(int);
template int step_span<double>(int);
template void launch_step<float>(const StepArgs<float>&, bool, int, cudaStream_t);
template void launch_step<double>(const StepArgs<double>&, bool, int, cudaStream_t);

}  // namespace lcb
