// lcb_narrow.cu — K1n: L2-panel PGA step for graphs whose iterate is far larger
// than L2 (config 4: ER n=1M, W=512 -> 2 GB per buffer).
//
// The batch is processed one narrow column panel at a time: the panel's columns are
// copied into a contiguous [n][P] buffer (P = 8 columns, 32 B per row; 32 MB at
// n = 1M), all T iterations run on it, and the result is copied back.  The panel's
// iterate (read deg times per iteration by the neighbour gathers) stays L2-resident,
// so DRAM only streams the compulsory x / v traffic.  Members are independent
// (ascent.cpp:52), so panels can run sequentially.
//
// Kernel: fp32 2 lanes x float4 per row (16 rows per warp), fp64 4 lanes x double2,
// neighbours in CSR order per element (fp64: bit-exact, graph.cpp:118), fused
// heavy-ball / clamp / finite check (ascent.cpp:66-77).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "lcb_internal.h"

namespace lcb {

namespace {

__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }

#ifndef LCB_NARROW_NB
#define LCB_NARROW_NB 4  // measured: 8 -> 91 regs, 3 blocks/SM, 7.8 ms vs 5.5 ms per C4 iteration
#endif
#ifndef LCB_NARROW_LATE
#define LCB_NARROW_LATE 0
#endif
#ifndef LCB_NARROW_MINB
#define LCB_NARROW_MINB 1
#endif

// Per-lane slice of a panel row: fp32 = 2 lanes x float4, fp64 = 4 lanes x double2.
// NB = neighbours whose gathers are in flight at once per lane.
template <typename T, int COLS>
struct Lane;
template <int COLS>
struct Lane<float, COLS> {
    static constexpr int LPR = COLS / 4;
    static constexpr int NB = LCB_NARROW_NB;
    using VT = float4;
};
template <int COLS>
struct Lane<double, COLS> {
    static constexpr int LPR = COLS / 2;
    static constexpr int NB = 16;
    using VT = double2;
};

// elementwise acc += g, round-to-nearest per element (packed FADD2 for fp32: two
// independent __fadd_rn, so the per-element sum order is the CSR order)
__device__ __forceinline__ void acc_add(float4& a, const float4& g) {
    unsigned long long lo, hi;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(lo)
        : "l"((static_cast<unsigned long long>(__float_as_uint(a.y)) << 32) | __float_as_uint(a.x)),
          "l"((static_cast<unsigned long long>(__float_as_uint(g.y)) << 32) | __float_as_uint(g.x)));
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(hi)
        : "l"((static_cast<unsigned long long>(__float_as_uint(a.w)) << 32) | __float_as_uint(a.z)),
          "l"((static_cast<unsigned long long>(__float_as_uint(g.w)) << 32) | __float_as_uint(g.z)));
    a.x = __uint_as_float(static_cast<unsigned>(lo));
    a.y = __uint_as_float(static_cast<unsigned>(lo >> 32));
    a.z = __uint_as_float(static_cast<unsigned>(hi));
    a.w = __uint_as_float(static_cast<unsigned>(hi >> 32));
}
__device__ __forceinline__ void acc_add(double2& a, const double2& g) {
    a.x = __dadd_rn(a.x, g.x);
    a.y = __dadd_rn(a.y, g.y);
}

// One block of NB neighbours per row: the column loads and all NB gathers are issued
// before the first add, so each warp keeps (32 / LPR) x NB L2 requests in flight (the
// kernel is latency-bound otherwise: row_ptr -> col -> gather).
template <typename T, int COLS, bool GEN>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? LCB_NARROW_MINB : 1) k_narrow(StepArgs<T> a) {
    constexpr int LPR = Lane<T, COLS>::LPR;
    constexpr int NB = Lane<T, COLS>::NB;
    constexpr int VW = COLS / LPR;
    using VT = typename Lane<T, COLS>::VT;
    const int lane = threadIdx.x & 31;
    const int sub = lane & (LPR - 1);
    const int slot = (blockIdx.x * blockDim.x + threadIdx.x) / LPR;
    const bool live = slot < a.n;
    const int row = live ? (a.order ? __ldg(a.order + slot) : slot) : 0;
    const int64_t off = static_cast<int64_t>(row) * LPR + sub;
    const VT* X = reinterpret_cast<const VT*>(a.x_in);  // panel, ld = COLS
    VT* Vel = reinterpret_cast<VT*>(a.vel);
    VT xv{}, vv{};
    T dg = T(0);
    int beg = 0, len = 0;
    if (live) {
        beg = __ldg(a.row_ptr + row);
        len = __ldg(a.row_ptr + row + 1) - beg;
        if (!LCB_NARROW_LATE) {
            xv = X[off];
            vv = __ldcs(Vel + off);  // touched once per iteration: evict first, keep the x panels in L2
            dg = __ldg(a.deg + row);
        }
    }
    int wmax = len;  // warp-wide trip count
#pragma unroll
    for (int o = 16; o >= LPR; o >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    VT acc{};
    for (int base = 0; base < wmax; base += NB) {
        int c[NB / LPR];
#pragma unroll
        for (int k = 0; k < NB / LPR; ++k) {
            const int idx = base + LPR * k + sub;
            c[k] = idx < len ? __ldg(a.col + beg + idx) : -1;
        }
        VT g[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const int u = __shfl_sync(0xffffffffu, c[q / LPR], q % LPR, LPR);
            if (u >= 0) g[q] = __ldg(X + static_cast<int64_t>(u) * LPR + sub);
        }
#pragma unroll
        for (int q = 0; q < NB; ++q)
            if (base + q < len) acc_add(acc, g[q]);  // CSR order per element
    }
    if (!live) return;
    if (LCB_NARROW_LATE) {
        xv = X[off];
        vv = __ldcs(Vel + off);
        dg = __ldg(a.deg + row);
    }
    T* xe = reinterpret_cast<T*>(&xv);
    T* ve = reinterpret_cast<T*>(&vv);
    const T* ae = reinterpret_cast<const T*>(&acc);
    VT xo = xv;
    T* oe = reinterpret_cast<T*>(&xo);
#pragma unroll
    for (int e = 0; e < VW; ++e) {
        const int colx = sub * VW + e;
        if (colx >= a.W) continue;
        const int m = (a.col_base + colx) / a.l;
        bool act = true;
        T alpha = a.alpha_uniform;
        if constexpr (GEN) {
            if (a.tlim) act = a.it < __ldg(a.tlim + m);
            if (a.alpha) alpha = __ldg(a.alpha + m);
        }
        if (!act) continue;
        const T x = xe[e];
        T v = ve[e];
        const T raw = pga_raw(x, ae[e], v, alpha, a.mu, dg);  // ascent.cpp:66-69
        if (!isfinite(raw))
            atomicMin(a.err + (a.err_seg ? m / a.err_seg : 0),
                      (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned>(a.it));
        oe[e] = raw < T(-1) ? T(-1) : (raw > T(1) ? T(1) : raw);  // ascent.cpp:73
        ve[e] = v;
    }
    reinterpret_cast<VT*>(a.x_out)[off] = xo;
    __stcs(Vel + off, vv);
}

// panel in/out: X[v][c0 .. c0+w) <-> P[v][0 .. cols), velocity zeroed on the way in
template <typename T>
__global__ void k_panel_in(const T* __restrict__ X, int64_t ld, int n, int cols, int c0, int w, T* __restrict__ P,
                           T* __restrict__ PV) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(n) * cols) return;
    const int64_t v = i / cols;
    const int c = static_cast<int>(i % cols);
    P[i] = c < w ? X[v * ld + c0 + c] : T(0);
    PV[i] = T(0);
}

template <typename T>
__global__ void k_panel_out(const T* __restrict__ P, int n, int cols, int c0, int w, T* __restrict__ X, int64_t ld) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(n) * cols) return;
    const int64_t v = i / cols;
    const int c = static_cast<int>(i % cols);
    if (c < w) X[v * ld + c0 + c] = P[i];
}

template <typename T, int COLS>
void launch_narrow(const StepArgs<T>& a, cudaStream_t s) {
    const unsigned blocks =
        static_cast<unsigned>((static_cast<int64_t>(a.n) * Lane<T, COLS>::LPR + 255) / 256);
    count_launch();
    if (a.alpha || a.tlim)
        k_narrow<T, COLS, true><<<blocks, 256, 0, s>>>(a);
    else
        k_narrow<T, COLS, false><<<blocks, 256, 0, s>>>(a);
}

}  // namespace

// Panel width: 8 columns (32 B fp32 rows: x_in + x_out panels = 64 MB at n = 1M, well
// inside L2); LCB_PANEL=16 selects 16 for fp32 (tuning hook).
int narrow_panel_cols(int elem_bytes) {
    static const int env = [] {
        const char* e = std::getenv("LCB_PANEL");
        return e ? std::atoi(e) : 8;
    }();
    return elem_bytes == 4 && env == 16 ? 16 : 8;
}

// All T iterations for columns [c0, c0 + w) (w <= cols) of the node-major batch in
// X_in (ld), result written to X_out; P0/P1/PV are [n][cols] panel buffers.
template <typename T>
void run_narrow_panel(const StepArgs<T>& base, const T* X_in, T* X_out, int64_t ld, int c0, int w,
                      int64_t iters, T* P0, T* P1, T* PV, cudaStream_t s) {
    const int n = base.n;
    const int cols = narrow_panel_cols(static_cast<int>(sizeof(T)));
    const int64_t cells = static_cast<int64_t>(n) * cols;
    const unsigned pb = static_cast<unsigned>((cells + 255) / 256);
    count_launch();
    k_panel_in<T><<<pb, 256, 0, s>>>(X_in, ld, n, cols, c0, w, P0, PV);
    StepArgs<T> a = base;
    a.W = w;
    a.col_base = c0;
    a.vel = PV;
    a.ld = cols;
    T* P[2] = {P0, P1};
    for (int64_t it = 0; it < iters; ++it) {
        a.x_in = P[it & 1];
        a.x_out = P[(it + 1) & 1];
        a.it = static_cast<int>(it);
        if (cols == 16)
            launch_narrow<T, 16>(a, s);
        else
            launch_narrow<T, 8>(a, s);
    }
    count_launch();
    k_panel_out<T><<<pb, 256, 0, s>>>(P[iters & 1], n, cols, c0, w, X_out, ld);
}

template void run_narrow_panel<float>(const StepArgs<float>&, const float*, float*, int64_t, int, int, int64_t,
                                      float*, float*, float*, cudaStream_t);
template void run_narrow_panel<double>(const StepArgs<double>&, const double*, double*, int64_t, int, int,
                                       int64_t, double*, double*, double*, cudaStream_t);

}  // namespace lcb
