// lcb_init.cu — K5: device-side initialisation of a batch.
//
//   DUI   init.cpp:20-30   x_v = (2u - 1)(1 - d_v / Δ)
//   IDI   init.cpp:32-62   random signs on d_v > d̄ + βσ, neighbour vote elsewhere
//   mean  init.cpp:89-101 + solver.cpp:210-223 (carry column 0, scale_down)
//   batch init.cpp:69-87   mean + sqrt(η)·N(0,1) per member stream, clamped;
//         around pm1_scaled(z) (solver.cpp:92-101) for every batch after the first.
//
// The integer parts (stream keys, sign bits, votes) are exact.  Box–Muller uses
// CUDA's double log / cos (≤ 2 ulp) where the reference calls glibc, so the
// normals agree to a few ulp; the runtime can instead upload host-drawn normals
// when a bitwise-identical batch is required (lcb_run_opts.host_init).
#include <cuda_runtime.h>

#include <cstdint>

#include "lcb_internal.h"

namespace lcb {

namespace {

__device__ __forceinline__ double dev_normal(uint64_t key, uint64_t k) {
    double u1 = rng_unit(rng_at(key, 2 * k));
    const double u2 = rng_unit(rng_at(key, 2 * k + 1));
    if (u1 <= 0.0) u1 = 0x1p-53;
    return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))),
                     cos(__dmul_rn(6.283185307179586476925286766559, u2)));
}

__device__ __forceinline__ double carry_or(const uint32_t* carry, int c, int v, double x) {
    if (carry && c == 0) return ((carry[v >> 5] >> (v & 31)) & 1u) ? 1.0 : -1.0;
    return x;
}

__global__ void k_dui(const int* __restrict__ row_ptr, int n, double maxdeg,
                      const uint64_t* __restrict__ col_keys, int l, double scale,
                      const uint32_t* __restrict__ carry, double* __restrict__ mean) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(n) * l) return;
    const int c = static_cast<int>(i / n), v = static_cast<int>(i % n);
    const double d = static_cast<double>(row_ptr[v + 1] - row_ptr[v]);
    const double bound = __dsub_rn(1.0, __ddiv_rn(d, maxdeg));
    const double u = rng_unit(rng_at(col_keys[c], static_cast<uint64_t>(v)));
    double x = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0), bound);
    x = carry_or(carry, c, v, x);
    mean[i] = __ddiv_rn(x, scale);
}

__global__ void k_idi_sign(const int* __restrict__ row_ptr, int n, double thr,
                           const uint64_t* __restrict__ col_keys, int l, int8_t* __restrict__ sign) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(n) * l) return;
    const int c = static_cast<int>(i / n), v = static_cast<int>(i % n);
    const double d = static_cast<double>(row_ptr[v + 1] - row_ptr[v]);
    int8_t s = 0;
    if (d > thr) s = (rng_at(col_keys[c], static_cast<uint64_t>(v)) & 1u) ? 1 : -1;
    sign[i] = s;
}

__global__ void k_idi_vote(const int* __restrict__ row_ptr, const int* __restrict__ col, int n,
                           const uint64_t* __restrict__ col_keys, int l, double scale,
                           const uint32_t* __restrict__ carry, const int8_t* __restrict__ sign,
                           double* __restrict__ mean) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(n) * l) return;
    const int c = static_cast<int>(i / n), v = static_cast<int>(i % n);
    const int8_t* sc = sign + static_cast<int64_t>(c) * n;
    double x;
    if (sc[v] != 0) {
        x = static_cast<double>(sc[v]);
    } else {
        int plus = 0, minus = 0;
        for (int k = row_ptr[v]; k < row_ptr[v + 1]; ++k) {
            const int8_t t = sc[col[k]];
            plus += t > 0;
            minus += t < 0;
        }
        if (plus == minus) {
            const uint64_t tie = combine(col_keys[c], 0x7469u);  // split({"ti"})
            x = (rng_at(tie, static_cast<uint64_t>(v)) & 1u) ? 1.0 : -1.0;
        } else {
            x = plus < minus ? 1.0 : -1.0;
        }
    }
    x = carry_or(carry, c, v, x);
    mean[i] = __ddiv_rn(x, scale);
}

// The same vote with one warp per (column, node), the lanes striding over the neighbours
// (dense graphs: a 10k-neighbour row is not one thread's dependent load chain).  The
// counts are integers, so the result equals the sequential vote.
__global__ void k_idi_vote_warp(const int* __restrict__ row_ptr, const int* __restrict__ col, int n,
                                const uint64_t* __restrict__ col_keys, int l, double scale,
                                const uint32_t* __restrict__ carry, const int8_t* __restrict__ sign,
                                double* __restrict__ mean) {
    const int lane = threadIdx.x & 31;
    const int64_t total = static_cast<int64_t>(n) * l;
    const int64_t stride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < total; i += stride) {
        const int c = static_cast<int>(i / n), v = static_cast<int>(i % n);
        const int8_t* sc = sign + static_cast<int64_t>(c) * n;
        double x;
        if (sc[v] != 0) {
            x = static_cast<double>(sc[v]);
        } else {
            int plus = 0, minus = 0;
            for (int k = row_ptr[v] + lane; k < row_ptr[v + 1]; k += 32) {
                const int8_t t = sc[col[k]];
                plus += t > 0;
                minus += t < 0;
            }
            plus = __reduce_add_sync(0xffffffffu, plus);
            minus = __reduce_add_sync(0xffffffffu, minus);
            if (plus == minus) {
                const uint64_t tie = combine(col_keys[c], 0x7469u);  // split({"ti"})
                x = (rng_at(tie, static_cast<uint64_t>(v)) & 1u) ? 1.0 : -1.0;
            } else {
                x = plus < minus ? 1.0 : -1.0;
            }
        }
        x = carry_or(carry, c, v, x);
        if (lane == 0) mean[i] = __ddiv_rn(x, scale);
    }
}

// X[v][m*l+c] = clamp(mean(c,v) + noise * N(member_key(m), c*n + v)); V = 0.
// Columns past W (row padding) are zeroed.
template <typename T>
__global__ void k_gaussian(T* __restrict__ X, T* __restrict__ V, int64_t ld, int n, int members,
                           int l, const uint64_t* __restrict__ mkeys, const double* __restrict__ mean,
                           const uint32_t* __restrict__ bits, double scale, double noise) {
    const int W = members * l;
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= ld) return;
    for (int v = blockIdx.y; v < n; v += gridDim.y) {
        const int64_t i = static_cast<int64_t>(v) * ld + col;
        double val = 0.0;
        if (col < W) {
            const int m = col / l, c = col - m * l;
            double mu;
            if (mean)
                mu = mean[static_cast<int64_t>(c) * n + v];
            else
                mu = __ddiv_rn(((bits[v >> 5] >> (v & 31)) & 1u) ? 1.0 : -1.0, scale);
            const double z = dev_normal(mkeys[m], static_cast<uint64_t>(c) * n + v);
            val = __dadd_rn(mu, __dmul_rn(noise, z));
            val = val < -1.0 ? -1.0 : (val > 1.0 ? 1.0 : val);  // project_box (init.cpp:84)
        }
        X[i] = static_cast<T>(val);
        V[i] = T(0);
    }
}

}  // namespace

void launch_dui(const DevGraph& g, const uint64_t* col_keys, int l, double init_scale,
                const uint32_t* carry_bits, double* mean, cudaStream_t s) {
    const int64_t total = static_cast<int64_t>(g.n) * l;
    count_launch();
    k_dui<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
        g.row_ptr, g.n, static_cast<double>(g.max_degree), col_keys, l, init_scale, carry_bits, mean);
}

void launch_idi(const DevGraph& g, double threshold, const uint64_t* col_keys, int l,
                double init_scale, const uint32_t* carry_bits, int8_t* sign_scratch, double* mean,
                cudaStream_t s) {
    const int64_t total = static_cast<int64_t>(g.n) * l;
    const unsigned blocks = static_cast<unsigned>((total + 255) / 256);
    count_launch();
    k_idi_sign<<<blocks, 256, 0, s>>>(g.row_ptr, g.n, threshold, col_keys, l, sign_scratch);
    count_launch();
    if (g.deg_mean > 64.0)
        k_idi_vote_warp<<<static_cast<unsigned>(std::min<int64_t>((total + 7) / 8, 148 * 32)), 256, 0, s>>>(
            g.row_ptr, g.col, g.n, col_keys, l, init_scale, carry_bits, sign_scratch, mean);
    else
        k_idi_vote<<<blocks, 256, 0, s>>>(g.row_ptr, g.col, g.n, col_keys, l, init_scale, carry_bits,
                                          sign_scratch, mean);
}

template <typename T>
void launch_gaussian(T* X, T* V, int64_t ld, int n, int members, int l, const uint64_t* mkeys,
                     const double* mean, const uint32_t* bits, double scale, double noise,
                     cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((ld + 127) / 128), static_cast<unsigned>(n < 4096 ? n : 4096));
    count_launch();
    k_gaussian<T><<<grid, 128, 0, s>>>(X, V, ld, n, members, l, mkeys, mean, bits, scale, noise);
}

template void launch_gaussian<float>(float*, float*, int64_t, int, int, int, const uint64_t*,
                                     const double*, const uint32_t*, double, double, cudaStream_t);
template void launch_gaussian<double>(double*, double*, int64_t, int, int, int, const uint64_t*,
                                      const double*, const uint32_t*, double, double, cudaStream_t);

}  // namespace lcb
