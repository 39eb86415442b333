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

// ---------------------------------------------------------------------------
// K1: fused PGA step.  One warp per (row, column slab-group); rows are visited
// in degree-descending order so hub rows start first (BA degree skew).
//   GEN = per-member alpha / iteration limit (batched search) or early exit
//   EE  = early-exit bits (implies GEN)
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ bool sat_code(uint32_t c) {
    constexpr uint32_t full = (1u << Vec<T>::E) - 1u;
    return ((c | (c >> 4)) & full) == full;
}
// add the +-1 values of a saturated code to acc (sequential order is kept by the caller)
__device__ __forceinline__ void add_code(float4& acc, uint32_t c) {
    acc.x = __fadd_rn(acc.x, (c & 1u) ? 1.f : -1.f);
    acc.y = __fadd_rn(acc.y, (c & 2u) ? 1.f : -1.f);
    acc.z = __fadd_rn(acc.z, (c & 4u) ? 1.f : -1.f);
    acc.w = __fadd_rn(acc.w, (c & 8u) ? 1.f : -1.f);
}
__device__ __forceinline__ void add_code(double2& acc, uint32_t c) {
    acc.x = __dadd_rn(acc.x, (c & 1u) ? 1.0 : -1.0);
    acc.y = __dadd_rn(acc.y, (c & 2u) ? 1.0 : -1.0);
}

#ifndef LCB_CODE_GROUP
#define LCB_CODE_GROUP 8
#endif
constexpr int kCodeGroup = LCB_CODE_GROUP;  // neighbours whose codes load together (one dependent round)

template <typename T, int S, bool GEN, bool EE, int MODE, bool REC>
__global__ void __launch_bounds__(kWarps * 32)
    k_step(StepArgs<T> a, int groups) {
    static_assert(!REC || (S == 1 && MODE == MODE_STEP), "saturation codes: one slab per warp, step mode");
    constexpr int E = Vec<T>::E;
    using V = typename Vec<T>::type;
    constexpr int SPAN = 32 * S * E;
    __shared__ uint32_t sbits[EE ? SPAN : 1];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
#if LCB_GROUP_MAJOR
    // slab-major block order: all SMs work the same column slab at a time, so the slabs
    // of hub rows (gathered by many rows) stay in L1
    const int rows_blocks = (a.n + kWarps - 1) / kWarps;
    const int group = blockIdx.x / rows_blocks;
    const int slot = (blockIdx.x % rows_blocks) * kWarps + warp;
#else
    const int group = blockIdx.x % groups;
    const int slot = (blockIdx.x / groups) * kWarps + warp;
#endif

    if constexpr (EE) {
        for (int i = threadIdx.x; i < SPAN; i += blockDim.x) sbits[i] = 0;
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < a.members; i += blockDim.x) a.flags_zero[i] = 0;
        __syncthreads();
    }

    if (slot < a.n) {
        const int row = a.order ? __ldg(a.order + slot) : slot;
        const int c0 = group * SPAN + lane * E;
        const T* xin = a.x_in + c0;
        const uint8_t* sin = REC ? a.sgn_in + group * 32 + lane : nullptr;
#if LCB_REC_EARLY
        // own x / v issued before the gathers: with coded gathers the kernel is latency-bound
        V xv_early{}, vv_early{};
        if constexpr (REC) {
            const int64_t off0 = static_cast<int64_t>(row) * a.ld + c0;
            xv_early = __ldcs(reinterpret_cast<const V*>(a.x_in + off0));
            vv_early = __ldcs(reinterpret_cast<const V*>(a.vel + off0));
        }
#endif

        V acc[S];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int e = 0; e < E; ++e) el(acc[s], e) = T(0);

        const int beg = __ldg(a.row_ptr + row);
        const int end = __ldg(a.row_ptr + row + 1);
        for (int base = beg; base < end; base += 32) {
            const int cnt = min(32, end - base);
            const int mycol = lane < cnt ? __ldg(a.col + base + lane) : 0;
            int k = 0;
            if constexpr (REC) {
                if (a.sgn_in) {
                    // codes of up to 16 neighbours in one round; when every lane's elements
                    // of all of them sit on the box corners, the sums come from the codes
                    // alone (no slab gathers), else this group gathers as usual
                    for (; k < cnt; k += kCodeGroup) {
                        const int kn = min(kCodeGroup, cnt - k);
                        uint32_t cq[kCodeGroup];
                        bool all = true;
#pragma unroll
                        for (int q = 0; q < kCodeGroup; ++q) {
                            const int u = __shfl_sync(0xffffffffu, mycol, (k + q) & 31);
                            cq[q] = q < kn ? static_cast<uint32_t>(__ldg(sin + static_cast<int64_t>(u) * a.sgn_ld)) : 0xFFu;
                        }
#pragma unroll
                        for (int q = 0; q < kCodeGroup; ++q) all = all && sat_code<T>(cq[q]);
                        if (__all_sync(0xffffffffu, all)) {
#pragma unroll
                            for (int q = 0; q < kCodeGroup; ++q)
                                if (q < kn) add_code(acc[0], cq[q]);
                            continue;
                        }
                        int kk = 0;
                        for (; kk + 4 <= kn; kk += 4) {
                            V v[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const int u = __shfl_sync(0xffffffffu, mycol, k + kk + q);
                                v[q] = ldg_vec(reinterpret_cast<const V*>(xin + static_cast<int64_t>(u) * a.ld));
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q)
#pragma unroll
                                for (int e = 0; e < E; ++e) el(acc[0], e) = radd(el(acc[0], e), el(v[q], e));
                        }
                        for (; kk < kn; ++kk) {
                            const int u = __shfl_sync(0xffffffffu, mycol, k + kk);
                            const V v = ldg_vec(reinterpret_cast<const V*>(xin + static_cast<int64_t>(u) * a.ld));
#pragma unroll
                            for (int e = 0; e < E; ++e) el(acc[0], e) = radd(el(acc[0], e), el(v, e));
                        }
                    }
                    continue;
                }
            }
            for (; k + 4 <= cnt; k += 4) {
                V v[4][S];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int u = __shfl_sync(0xffffffffu, mycol, k + q);
                    const V* p = reinterpret_cast<const V*>(xin + static_cast<int64_t>(u) * a.ld);
#pragma unroll
                    for (int s = 0; s < S; ++s) v[q][s] = ldg_vec(p + s * 32);
                }
                // sequential CSR order per element (graph.cpp:118)
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int s = 0; s < S; ++s)
#pragma unroll
                        for (int e = 0; e < E; ++e) el(acc[s], e) = radd(el(acc[s], e), el(v[q][s], e));
            }
            for (; k < cnt; ++k) {
                const int u = __shfl_sync(0xffffffffu, mycol, k);
                const V* p = reinterpret_cast<const V*>(xin + static_cast<int64_t>(u) * a.ld);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const V v = ldg_vec(p + s * 32);
#pragma unroll
                    for (int e = 0; e < E; ++e) el(acc[s], e) = radd(el(acc[s], e), el(v, e));
                }
            }
        }

        const T dg = __ldg(a.deg + row);
        const int64_t rb = static_cast<int64_t>(row) * a.ld + c0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int64_t off = rb + s * 32 * E;
#if LCB_REC_EARLY
            V xv = REC ? xv_early : *reinterpret_cast<const V*>(a.x_in + off);
#else
            V xv = *reinterpret_cast<const V*>(a.x_in + off);
#endif
            if constexpr (MODE == MODE_LAPLACE) {
                V y;
#pragma unroll
                for (int e = 0; e < E; ++e) el(y, e) = rsub(rmul(dg, el(xv, e)), el(acc[s], e));
                *reinterpret_cast<V*>(a.x_out + off) = y;
                continue;
            } else {
#if LCB_REC_EARLY
                V vv = REC ? vv_early : *reinterpret_cast<const V*>(a.vel + off);
#else
                V vv = *reinterpret_cast<const V*>(a.vel + off);
#endif
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
                            m = (a.col_base + colx) / a.l;
                            if (a.tlim) act = a.it < __ldg(a.tlim + m);
                            if constexpr (EE) {
                                if (act && a.it > 0) act = ex_continue(__ldcg(a.flags_prev + m));
                            }
                            if (a.alpha) alpha = __ldg(a.alpha + m);
                        }
                    } else {
                        m = (a.col_base + colx) / a.l;
                    }
                    if (act) {
                        T v = el(vv, e);
                        const T raw = pga_raw(x, el(acc[s], e), v, alpha, a.mu, dg);  // ascent.cpp:66-69
                        if (!isfinite(raw))                                // ascent.cpp:70-72
                            atomicMin(a.err + (a.err_seg ? m / a.err_seg : 0), (static_cast<unsigned long long>(m) << 32) |
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
                if constexpr (REC) {
                    uint32_t code = 0;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        if (el(xo, e) == T(1)) code |= 1u << e;
                        else if (el(xo, e) == T(-1)) code |= 16u << e;
                    }
                    a.sgn_out[static_cast<int64_t>(row) * a.sgn_ld + group * 32 + lane] = static_cast<uint8_t>(code);
                }
            }
        }
    }

    if constexpr (EE) {
        __syncthreads();
        for (int i = threadIdx.x; i < SPAN; i += blockDim.x) {
            const uint32_t b = sbits[i];
            const int colx = group * SPAN + i;
            if (b && colx < a.W) {
                const int m = (a.col_base + colx) / a.l;
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
    if (forced == 1 || forced == 2 || forced == 4) return forced;
    constexpr int E = Vec<T>::E;
    (void)E;
    (void)W;
    return 1;  // measured best on B200 for W in {1024, 2048} (profiles/)
}

template <typename T, bool GEN, bool EE, int MODE>
void dispatch_s(const StepArgs<T>& a, int S, cudaStream_t st) {
    constexpr int E = Vec<T>::E;
    const int rows_blocks = (a.n + kWarps - 1) / kWarps;
    auto go = [&](auto sconst) {
        constexpr int SS = decltype(sconst)::value;
        constexpr int SPAN = 32 * SS * E;
        const int groups = (a.W + SPAN - 1) / SPAN;  // slabs covering the live columns
        const dim3 grid(static_cast<unsigned>(rows_blocks) * groups);
        count_launch();
        if constexpr (SS == 1 && MODE == MODE_STEP) {
            if (a.sgn_out) {
                k_step<T, SS, GEN, EE, MODE, true><<<grid, kWarps * 32, 0, st>>>(a, groups);
                return;
            }
        }
        k_step<T, SS, GEN, EE, MODE, false><<<grid, kWarps * 32, 0, st>>>(a, groups);
    };
    if (S == 1)
        go(std::integral_constant<int, 1>{});
    else if (S == 2)
        go(std::integral_constant<int, 2>{});
    else
        go(std::integral_constant<int, 4>{});
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
