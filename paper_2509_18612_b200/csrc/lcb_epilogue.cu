// lcb_epilogue.cu — K4: threshold rounding -> bit-packed assignments ->
// bit-sliced integer cut counts -> first-max argmax -> winner bits, plus the
// boundary transposes between DenseState's [B][l][n] and the node-major device
// layout.
//
// Reference lines: round_unlifted / round_lifted objectives.cpp:81-96,
// cut_value :26-35, argmax solver.cpp:125-138, pm1_scaled :92-101.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "lcb_internal.h"

#ifndef LCB_EPI_UNROLL
#define LCB_EPI_UNROLL 4
#endif

namespace lcb {

namespace {

// ---------------------------------------------------------------------------
// transposes: DenseState [W][n] (double) <-> device [n][ld] (T)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_transpose_in(const double* __restrict__ src, T* __restrict__ dst, int n, int W,
                               int64_t ld) {
    __shared__ double tile[32][33];
    const int v0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, v = v0 + threadIdx.x;
        tile[i][threadIdx.x] = (c < W && v < n) ? src[static_cast<int64_t>(c) * n + v] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int v = v0 + i, c = c0 + threadIdx.x;
        if (v < n && c < ld) dst[static_cast<int64_t>(v) * ld + c] = static_cast<T>(tile[threadIdx.x][i]);
    }
}

template <typename T>
__global__ void k_transpose_out(const T* __restrict__ src, double* __restrict__ dst, int n, int W,
                                int64_t ld) {
    __shared__ double tile[32][33];
    const int v0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int v = v0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (v < n && c < W) ? static_cast<double>(src[static_cast<int64_t>(v) * ld + c]) : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, v = v0 + threadIdx.x;
        if (c < W && v < n) dst[static_cast<int64_t>(c) * n + v] = tile[threadIdx.x][i];
    }
}

// ---------------------------------------------------------------------------
// trace objective: out[m] += sum_v sum_c X[v][m*l+c] * Y[v][m*l+c]
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_member_dot(const T* X, const T* Y, int n, int W, int l, int64_t ld, double* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= W) return;
    double acc = 0.0;
    for (int v = blockIdx.y; v < n; v += gridDim.y) {
        const int64_t i = static_cast<int64_t>(v) * ld + c;
        acc += static_cast<double>(X[i]) * static_cast<double>(Y[i]);
    }
    atomicAdd(out + c / l, acc);
}

// ---------------------------------------------------------------------------
// round + pack: one warp per (row, 32-member word); lane = member in the word
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_round_pack(const T* __restrict__ X, int64_t ld, int n, int members, int l,
                             int lifted, uint32_t* __restrict__ Z, int words) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t total = static_cast<int64_t>(n) * words;
    const int64_t stride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t t = gw; t < total; t += stride) {
        const int row = static_cast<int>(t / words);
        const int w = static_cast<int>(t % words);
        const int m = w * 32 + lane;
        bool z = false;
        if (m < members) {
            const T* p = X + static_cast<int64_t>(row) * ld + static_cast<int64_t>(m) * l;
            if (lifted) {
                double s = 0.0;  // fp64 row sum in column order
                for (int c = 0; c < l; ++c) s = __dadd_rn(s, static_cast<double>(p[c]));
                z = s >= 0.0;                  // inclusive (objectives.cpp:94)
            } else {
                z = static_cast<double>(p[0]) > 0.0;  // strict (objectives.cpp:83)
            }
        }
        const uint32_t bits = __ballot_sync(0xffffffffu, z);
        if (lane == 0) Z[static_cast<int64_t>(w) * n + row] = bits;
    }
}

// z bytes [count][n] -> Z[w][v]
__global__ void k_pack_bytes(const uint8_t* __restrict__ z, int n, int count, uint32_t* __restrict__ Z,
                             int words) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    const int w = blockIdx.y;
    if (v >= n) return;
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
        const int m = w * 32 + b;
        if (m < count && z[static_cast<int64_t>(m) * n + v]) bits |= 1u << b;
    }
    Z[static_cast<int64_t>(w) * n + v] = bits;
}

// ---------------------------------------------------------------------------
// bit-sliced cut counting.  For every edge (u < v) and 32-member word w the
// XOR of the two assignment words marks the members that cut the edge; 16 bit
// planes per lane form vertical counters (ripple-carry add), flushed into 32
// per-member integers, warp-reduced with redux.sync and added with one atomic
// per member per warp.  Integer-exact by construction.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void planes_add(uint32_t (&p)[16], uint32_t d) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint32_t t = p[k] & d;
        p[k] ^= d;
        d = t;
    }
}

__device__ __forceinline__ void planes_flush(uint32_t (&p)[16], uint32_t (&cnt)[32]) {
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) c |= ((p[k] >> b) & 1u) << k;
        cnt[b] += c;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) p[k] = 0;
}

// Accumulate the cut edges (u < v) of rows [first, n) with the given stride into the
// thread's bit planes.  Sparse graphs: one row per thread.  Dense graphs (average degree
// above 64): one row per warp, the lanes striding over its neighbours, so a 10k-neighbour
// row is not one thread's dependent load chain.
template <bool COHERENT>
__device__ __forceinline__ void cut_rows(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                         const uint32_t* __restrict__ zw, int n, int part, int parts, bool warp_rows,
                                         uint32_t (&planes)[16], uint32_t (&cnt)[32]) {
    auto zload = [&](int i) { return COHERENT ? __ldcg(zw + i) : __ldg(zw + i); };
    uint32_t adds = 0;
    auto add = [&](uint32_t d) {
        planes_add(planes, d);
        if (++adds == 0xffffu) {
            planes_flush(planes, cnt);
            adds = 0;
        }
    };
    if (!warp_rows) {
        for (int r = part * blockDim.x + threadIdx.x; r < n; r += parts * blockDim.x) {
            const uint32_t zu = zload(r);
            const int beg = __ldg(row_ptr + r), end = __ldg(row_ptr + r + 1);
            int k = beg;
            for (; k + 4 <= end; k += 4) {  // four independent column / Z loads in flight
                int v[4];
                uint32_t zv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(col + k + u);
#pragma unroll
                for (int u = 0; u < 4; ++u) zv[u] = v[u] > r ? zload(v[u]) : zu;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (v[u] > r) add(zu ^ zv[u]);  // each undirected edge once (objectives.cpp:33)
            }
            for (; k < end; ++k) {
                const int v = __ldg(col + k);
                if (v > r) add(zu ^ zload(v));
            }
        }
    } else {
        const int wpb = blockDim.x >> 5, lane = threadIdx.x & 31;
        for (int r = part * wpb + (threadIdx.x >> 5); r < n; r += parts * wpb) {
            const uint32_t zu = zload(r);
            const int beg = __ldg(row_ptr + r), end = __ldg(row_ptr + r + 1);
            for (int k = beg + lane; k < end; k += 32) {
                const int v = __ldg(col + k);
                if (v > r) add(zu ^ zload(v));
            }
        }
    }
}

// first-max argmax over `members` cuts in segments of seg_size, by one block
__device__ void block_argmax(const unsigned long long* cuts, int members, int seg_size, int64_t member_base,
                             unsigned long long* seg_keys) {
    __shared__ unsigned long long red[32];
    const int segs = (members + seg_size - 1) / seg_size;
    for (int s = 0; s < segs; ++s) {
        const int lo = s * seg_size, hi = min(members, lo + seg_size);
        unsigned long long best = 0;
        for (int m = lo + threadIdx.x; m < hi; m += blockDim.x) {
            const unsigned long long gm = static_cast<unsigned long long>(member_base + (m - lo));
            const unsigned long long key = (__ldcg(cuts + m) << 32) | (0xffffffffull - gm);
            best = key > best ? key : best;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
            best = t > best ? t : best;
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x < 32) {
            best = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
                best = t > best ? t : best;
            }
            if (threadIdx.x == 0) seg_keys[s] = best;
        }
        __syncthreads();
    }
}

// Fused epilogue: bit-sliced cut counts, then -- in the last block to finish -- the
// first-max argmax of every segment (one launch instead of two; seg_keys null: counts only).
__global__ void __launch_bounds__(256) k_cut_count(const int* __restrict__ row_ptr,
                                                   const int* __restrict__ col,
                                                   const uint32_t* __restrict__ Z, int n,
                                                   unsigned long long* __restrict__ cuts,
                                                   unsigned long long* __restrict__ done, int members, int seg_size,
                                                   int64_t member_base, unsigned long long* __restrict__ seg_keys,
                                                   int warp_rows) {
    const int w = blockIdx.y;
    const uint32_t* zw = Z + static_cast<int64_t>(w) * n;
    uint32_t planes[16];
    uint32_t cnt[32];
#pragma unroll
    for (int k = 0; k < 16; ++k) planes[k] = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) cnt[b] = 0;
    cut_rows<false>(row_ptr, col, zw, n, blockIdx.x, gridDim.x, warp_rows != 0, planes, cnt);
    planes_flush(planes, cnt);
    const int lane = threadIdx.x & 31;
    uint32_t mine = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        const uint32_t t = __reduce_add_sync(0xffffffffu, cnt[b]);
        if (lane == b) mine = t;
    }
    if (mine) atomicAdd(cuts + w * 32 + lane, static_cast<unsigned long long>(mine));
    if (seg_keys == nullptr) return;
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
        last = atomicAdd(done, 1ull) == static_cast<unsigned long long>(gridDim.x) * gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    block_argmax(cuts, members, seg_size, member_base, seg_keys);
}

// ---------------------------------------------------------------------------
// K4 as ONE kernel (north star 4): round + pack, grid barrier, bit-sliced cut counts,
// then the last block to finish takes the first-max argmax of every segment and, when
// no cross-rank reduction of the key is needed, extracts the winner's bits.  Launched
// cooperatively (every block resident, so the grid barrier cannot deadlock); block b
// counts the edges of assignment word b % words over its share of the rows.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_epilogue(const T* __restrict__ X, int64_t ld, int n, int members, int l,
                                                  int lifted, uint32_t* __restrict__ Z, int words,
                                                  const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                  unsigned long long* __restrict__ cuts,
                                                  unsigned long long* __restrict__ done, int seg_size,
                                                  int64_t member_base, unsigned long long* __restrict__ seg_keys,
                                                  uint32_t* __restrict__ win_bits, int warp_rows,
                                                  uint32_t* __restrict__ Zt, int skip_cut) {
    namespace cg = cooperative_groups;
    // ---- round + pack (objectives.cpp:81-96).  Unlifted: one warp per row, eight words'
    // loads in flight per lane (a 2 KB row of config 4 is 16 coalesced 128-byte loads).
    if (!lifted) {
        const int lane = threadIdx.x & 31;
        const int64_t stride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
        for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < n;
             row += stride) {
            const T* p = X + row * ld;
            for (int w0 = 0; w0 < words; w0 += 8) {
                T v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int m = (w0 + q) * 32 + lane;
                    v[q] = (w0 + q < words && m < members) ? p[m] : T(0);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (w0 + q < words) {
                        const uint32_t bits = __ballot_sync(0xffffffffu, static_cast<double>(v[q]) > 0.0);  // strict
                        if (lane == 0) {
                            Z[static_cast<int64_t>(w0 + q) * n + row] = bits;
                            if (Zt) Zt[row * 8 + w0 + q] = bits;
                        }
                    }
                }
            }
        }
    } else {
        // lifted: one warp per (row, 32-member word), the row sum in column order
        const int lane = threadIdx.x & 31;
        const int64_t total = static_cast<int64_t>(n) * words;
        const int64_t stride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
        for (int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; t < total; t += stride) {
            const int row = static_cast<int>(t / words);
            const int w = static_cast<int>(t % words);
            const int m = w * 32 + lane;
            bool z = false;
            if (m < members) {
                const T* p = X + static_cast<int64_t>(row) * ld + static_cast<int64_t>(m) * l;
                if (lifted) {
                    double s = 0.0;
                    for (int c = 0; c < l; ++c) s = __dadd_rn(s, static_cast<double>(p[c]));
                    z = s >= 0.0;
                } else {
                    z = static_cast<double>(p[0]) > 0.0;
                }
            }
            const uint32_t bits = __ballot_sync(0xffffffffu, z);
            if (lane == 0) {
                Z[static_cast<int64_t>(w) * n + row] = bits;
                if (Zt) Zt[static_cast<int64_t>(row) * 8 + w] = bits;
            }
        }
    }
    cg::this_grid().sync();
    // ---- cut counts (objectives.cpp:26-35); skip_cut: already in `cuts` (dense cut pass)
    if (skip_cut) {
    } else if (Zt) {
        // dense graphs, <= 8 words: warp j of every block counts word j over the block's rows;
        // the 8 warps read the same column runs and the same 32-byte node-major Zt lines, so
        // those loads hit L1 after the first warp
        const int j = static_cast<int>(threadIdx.x >> 5);
        if (j < words) {
            const int lane = threadIdx.x & 31;
            uint32_t planes[16];
            uint32_t cnt[32];
#pragma unroll
            for (int k = 0; k < 16; ++k) planes[k] = 0;
#pragma unroll
            for (int b = 0; b < 32; ++b) cnt[b] = 0;
            uint32_t adds = 0;
            for (int r = blockIdx.x; r < n; r += gridDim.x) {
                const uint32_t zu = Zt[static_cast<int64_t>(r) * 8 + j];
                const int beg = __ldg(row_ptr + r), end = __ldg(row_ptr + r + 1);
                // kU neighbours per lane in flight (the column and Zt loads are independent)
                constexpr int kU = LCB_EPI_UNROLL;
                for (int k = beg + lane; k < end; k += 32 * kU) {
                    int v[kU];
                    uint32_t zv[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) v[u] = k + 32 * u < end ? __ldg(col + k + 32 * u) : -1;
#pragma unroll
                    for (int u = 0; u < kU; ++u) zv[u] = v[u] > r ? Zt[static_cast<int64_t>(v[u]) * 8 + j] : zu;
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        if (v[u] > r) {  // each undirected edge once (objectives.cpp:33)
                            planes_add(planes, zu ^ zv[u]);
                            if (++adds == 0xffffu) {
                                planes_flush(planes, cnt);
                                adds = 0;
                            }
                        }
                    }
                }
            }
            planes_flush(planes, cnt);
            uint32_t mine = 0;
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                const uint32_t t = __reduce_add_sync(0xffffffffu, cnt[b]);
                if (lane == b) mine = t;
            }
            if (mine) atomicAdd(cuts + j * 32 + lane, static_cast<unsigned long long>(mine));
        }
    } else {
        const int w = static_cast<int>(blockIdx.x % words);
        const int parts = static_cast<int>(gridDim.x / words);
        const int part = static_cast<int>(blockIdx.x / words);
        const uint32_t* zw = Z + static_cast<int64_t>(w) * n;
        uint32_t planes[16];
        uint32_t cnt[32];
#pragma unroll
        for (int k = 0; k < 16; ++k) planes[k] = 0;
#pragma unroll
        for (int b = 0; b < 32; ++b) cnt[b] = 0;
        cut_rows<true>(row_ptr, col, zw, n, part, parts, warp_rows != 0, planes, cnt);
        planes_flush(planes, cnt);
        const int lane = threadIdx.x & 31;
        uint32_t mine = 0;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const uint32_t t = __reduce_add_sync(0xffffffffu, cnt[b]);
            if (lane == b) mine = t;
        }
        if (mine) atomicAdd(cuts + w * 32 + lane, static_cast<unsigned long long>(mine));
    }
    // ---- the last block: argmax (solver.cpp:132-134), winner bits (solver.cpp:138)
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1ull) == static_cast<unsigned long long>(gridDim.x) - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    block_argmax(cuts, members, seg_size, member_base, seg_keys);
    if (win_bits == nullptr) return;
    const unsigned long long key = *reinterpret_cast<volatile unsigned long long*>(seg_keys);
    const int64_t m = static_cast<int64_t>(0xffffffffull - (key & 0xffffffffull)) - member_base;
    const int wsel = static_cast<int>(m >> 5), bsel = static_cast<int>(m & 31);
    const int nwords = (n + 31) / 32;
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x >> 5; i < nwords; i += blockDim.x >> 5) {
        const int v = i * 32 + lane;
        const bool z = v < n && ((__ldcg(Z + static_cast<int64_t>(wsel) * n + v) >> bsel) & 1u);
        const uint32_t word = __ballot_sync(0xffffffffu, z);
        if (lane == 0) win_bits[i] = word;
    }
}

// ---------------------------------------------------------------------------
// first-max argmax: key = cut << 32 | (0xffffffff - member) so that the max
// key is the largest cut at the smallest member index (solver.cpp:132-134).
// One block per segment (a batch; several when search candidates are batched).
// ---------------------------------------------------------------------------
__global__ void k_argmax(const unsigned long long* __restrict__ cuts, int members, int seg_size,
                         int64_t member_base, unsigned long long* __restrict__ seg_keys) {
    __shared__ unsigned long long red[32];
    const int s = blockIdx.x;
    const int lo = s * seg_size, hi = min(members, lo + seg_size);
    unsigned long long best = 0;
    for (int m = lo + threadIdx.x; m < hi; m += blockDim.x) {
        const unsigned long long gm = static_cast<unsigned long long>(member_base + (m - lo));
        const unsigned long long key = (cuts[m] << 32) | (0xffffffffull - gm);
        best = key > best ? key : best;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
        best = t > best ? t : best;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        best = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
            best = t > best ? t : best;
        }
        if (threadIdx.x == 0) seg_keys[s] = best;
    }
}

// winner bits for key_src[0]: member (global) -> local word/bit of Z
__global__ void k_extract_winner(const uint32_t* __restrict__ Z, int n,
                                 const unsigned long long* __restrict__ key_src,
                                 int64_t member_base, int members, uint32_t* __restrict__ bits,
                                 int member_offset) {
    const unsigned long long key = *key_src;
    const int64_t gm = static_cast<int64_t>(0xffffffffull - (key & 0xffffffffull));
    const int64_t m = gm - member_base + member_offset;
    const bool local = m >= member_offset && m < members;
    const int w = local ? static_cast<int>(m >> 5) : 0;
    const int b = local ? static_cast<int>(m & 31) : 0;
    const int words = (n + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t stride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = gw; i < words; i += stride) {
        const int v = static_cast<int>(i * 32 + lane);
        bool z = false;
        if (local && v < n) z = (Z[static_cast<int64_t>(w) * n + v] >> b) & 1u;
        const uint32_t word = __ballot_sync(0xffffffffu, z);
        if (lane == 0) bits[i] = word;
    }
}

__global__ void k_unpack_bits(const uint32_t* __restrict__ bits, int n, uint8_t* __restrict__ z) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) z[v] = static_cast<uint8_t>((bits[v >> 5] >> (v & 31)) & 1u);
}

}  // namespace

template <typename T>
void launch_transpose_in(const double* src, T* dst, int n, int W, int64_t ld, cudaStream_t s) {
    const dim3 grid((n + 31) / 32, static_cast<unsigned>((ld + 31) / 32));
    count_launch();
    k_transpose_in<T><<<grid, dim3(32, 8), 0, s>>>(src, dst, n, W, ld);
}

template <typename T>
void launch_transpose_out(const T* src, double* dst, int n, int W, int64_t ld, cudaStream_t s) {
    const dim3 grid((n + 31) / 32, (W + 31) / 32);
    count_launch();
    k_transpose_out<T><<<grid, dim3(32, 8), 0, s>>>(src, dst, n, W, ld);
}

template <typename T>
void launch_member_dot(const T* X, const T* Y, int n, int W, int l, int64_t ld, double* out,
                       cudaStream_t s) {
    const dim3 grid((W + 127) / 128, std::min(n, 256));
    count_launch();
    k_member_dot<T><<<grid, 128, 0, s>>>(X, Y, n, W, l, ld, out);
}

template <typename T>
void launch_round_pack(const T* X, int64_t ld, int n, int members, int l, int lifted, uint32_t* Z,
                       cudaStream_t s) {
    const int words = (members + 31) / 32;
    const int64_t warps = static_cast<int64_t>(n) * words;
    const int blocks = static_cast<int>(std::min<int64_t>((warps + 7) / 8, 148 * 64));
    count_launch();
    k_round_pack<T><<<blocks, 256, 0, s>>>(X, ld, n, members, l, lifted, Z, words);
}

// largest entry of a uint32 array (graph ingest: adjacency range check on the device)
__global__ void k_max_u32(const uint32_t* __restrict__ a, int64_t count, unsigned* __restrict__ out) {
    unsigned m = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * 4;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < count; i += stride) {
        if (i + 3 < count && (reinterpret_cast<uintptr_t>(a + i) & 15) == 0) {
            const uint4 v = *reinterpret_cast<const uint4*>(a + i);
            m = max(m, max(max(v.x, v.y), max(v.z, v.w)));
        } else {
            for (int64_t j = i; j < i + 4 && j < count; ++j) m = max(m, a[j]);
        }
    }
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

void launch_max_u32(const uint32_t* a, int64_t count, unsigned* out, cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof(unsigned), s);
    count_launch();
    k_max_u32<<<148 * 8, 256, 0, s>>>(a, count, out);
}

void launch_pack_bytes(const uint8_t* z, int n, int count, uint32_t* Z, cudaStream_t s) {
    const int words = (count + 31) / 32;
    count_launch();
    k_pack_bytes<<<dim3((n + 255) / 256, words), 256, 0, s>>>(z, n, count, Z, words);
}

void launch_cut_count(const DevGraph& g, const uint32_t* Z, int words, unsigned long long* cuts,
                      cudaStream_t s) {
    cudaMemsetAsync(cuts, 0, sizeof(unsigned long long) * static_cast<size_t>(words) * 32, s);
    const int per_word = std::max(1, std::min((g.n + 255) / 256, (8 * num_sms(g.device)) / words + 1));
    count_launch();
    k_cut_count<<<dim3(per_word, words), 256, 0, s>>>(g.row_ptr, g.col, Z, g.n, cuts, nullptr, 0, 1, 0, nullptr,
                                                       g.deg_mean > 64.0 ? 1 : 0);
}

void launch_cut_argmax(const DevGraph& g, const uint32_t* Z, int words, unsigned long long* cuts, int members,
                       int seg_size, int64_t member_base, unsigned long long* seg_keys, cudaStream_t s) {
    // cuts [words * 32] followed by the block-completion counter, zeroed together
    cudaMemsetAsync(cuts, 0, sizeof(unsigned long long) * (static_cast<size_t>(words) * 32 + 1), s);
    const int per_word = std::max(1, std::min((g.n + 255) / 256, (8 * num_sms(g.device)) / words + 1));
    count_launch();
    k_cut_count<<<dim3(per_word, words), 256, 0, s>>>(g.row_ptr, g.col, Z, g.n, cuts, cuts + words * 32, members,
                                                       seg_size, member_base, seg_keys, g.deg_mean > 64.0 ? 1 : 0);
}

// cut(m) = (nnz - sum_v s_v (A s)_v) / 4 for s = +-1 (each undirected edge appears twice in
// the CSR: sum over edges of s_u s_v = uncut - cut = nnz / 2 - 2 cut); done counter zeroed
__global__ void k_cuts_from_sums(const unsigned long long* __restrict__ sums, int members, int64_t nnz,
                                 unsigned long long* __restrict__ cuts, int slots) {
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m <= slots; m += gridDim.x * blockDim.x)
        cuts[m] = m < members ? static_cast<unsigned long long>((nnz - static_cast<long long>(sums[m])) / 4) : 0ull;
}

template <typename T>
void launch_epilogue(const DevGraph& g, const T* X, int64_t ld, int members, int l, int lifted, uint32_t* Z,
                     unsigned long long* cuts, int seg_size, int64_t member_base, unsigned long long* seg_keys,
                     uint32_t* win_bits, cudaStream_t s, const unsigned long long* cut_sums) {
    const int words = (members + 31) / 32;
    int skip_cut = cut_sums ? 1 : 0;
    if (cut_sums) {
        count_launch();
        k_cuts_from_sums<<<(words * 32 + 256) / 256, 256, 0, s>>>(cut_sums, members, g.nnz, cuts, words * 32);
    } else {
        cudaMemsetAsync(cuts, 0, sizeof(unsigned long long) * (static_cast<size_t>(words) * 32 + 1), s);
    }
    static std::atomic<int> per_sm[64];
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    const int slot = dev >= 0 && dev < 64 ? dev : 0;
    int occ = per_sm[slot].load(std::memory_order_relaxed);
    if (!occ) {
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_epilogue<T>, 256, 0), "occupancy(k_epilogue)");
        occ = std::max(1, occ);
        per_sm[slot].store(occ, std::memory_order_relaxed);
    }
    // every block resident (grid barrier); a multiple of `words` blocks, <= one per 256 rows per word
    const int resident = occ * num_sms(dev);
    // dense graphs with <= 8 words: every block counts all words (warp j = word j) over its
    // rows, sharing the column and Zt loads in L1; Zt = node-major copy of Z [n][8]
    const bool dense_block = !skip_cut && g.deg_mean > 64.0 && words <= 8;
    int parts = std::max(1, std::min((g.n + 255) / 256, resident / words));
    int grid = parts * words;
    uint32_t* Zt = nullptr;
    if (dense_block) {
        grid = std::max(1, std::min(g.n, resident));
        Zt = static_cast<uint32_t*>(pool_alloc(sizeof(uint32_t) * 8 * static_cast<size_t>(g.n), s));
    } else if (parts * words > resident)  // more words than resident blocks: the unfused kernels
    {
        launch_round_pack<T>(X, ld, g.n, members, l, lifted, Z, s);
        if (skip_cut)
            launch_argmax(cuts, members, seg_size, member_base, seg_keys, s);
        else
            launch_cut_argmax(g, Z, words, cuts, members, seg_size, member_base, seg_keys, s);
        if (win_bits) launch_extract_winner(Z, g.n, seg_keys, member_base, members, win_bits, s, 0);
        return;
    }
    unsigned long long* done = cuts + static_cast<size_t>(words) * 32;
    int n = g.n, nw = words;
    const int* rp = g.row_ptr;
    const int* cl = g.col;
    int warp_rows = g.deg_mean > 64.0 ? 1 : 0;
    void* args[] = {&X, &ld, &n, &members, &l, &lifted, &Z, &nw, &rp, &cl, &cuts, &done, &seg_size,
                    &member_base, &seg_keys, &win_bits, &warp_rows, &Zt, &skip_cut};
    count_launch();
    const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_epilogue<T>), dim3(grid),
                                                      dim3(256), args, 0, s);
    if (Zt) pool_free(Zt, s);
    if (e == cudaErrorCooperativeLaunchTooLarge) {
        // other work holds part of the device (the grid barrier needs every block resident):
        // the same epilogue as separate launches
        (void)cudaGetLastError();
        launch_round_pack<T>(X, ld, g.n, members, l, lifted, Z, s);
        if (skip_cut)
            launch_argmax(cuts, members, seg_size, member_base, seg_keys, s);
        else
            launch_cut_argmax(g, Z, words, cuts, members, seg_size, member_base, seg_keys, s);
        if (win_bits) launch_extract_winner(Z, g.n, seg_keys, member_base, members, win_bits, s, 0);
        return;
    }
    cuda_check(e, "cudaLaunchCooperativeKernel(k_epilogue)");
}
template void launch_epilogue<float>(const DevGraph&, const float*, int64_t, int, int, int, uint32_t*,
                                     unsigned long long*, int, int64_t, unsigned long long*, uint32_t*, cudaStream_t,
                                     const unsigned long long*);
template void launch_epilogue<double>(const DevGraph&, const double*, int64_t, int, int, int, uint32_t*,
                                      unsigned long long*, int, int64_t, unsigned long long*, uint32_t*,
                                      cudaStream_t, const unsigned long long*);

void launch_argmax(const unsigned long long* cuts, int members, int seg_size, int64_t member_base,
                   unsigned long long* seg_keys, cudaStream_t s) {
    const int segs = (members + seg_size - 1) / seg_size;
    count_launch();
    k_argmax<<<segs, 256, 0, s>>>(cuts, members, seg_size, member_base, seg_keys);
}

void launch_extract_winner(const uint32_t* Z, int n, const unsigned long long* key_src,
                           int64_t member_base, int members, uint32_t* bits, cudaStream_t s,
                           int member_offset) {
    const int words = (n + 31) / 32;
    const int blocks = std::min((words + 7) / 8, 1024);
    count_launch();
    k_extract_winner<<<blocks, 256, 0, s>>>(Z, n, key_src, member_base, members, bits, member_offset);
}

void launch_unpack_bits(const uint32_t* bits, int n, uint8_t* z, cudaStream_t s) {
    count_launch();
    k_unpack_bits<<<(n + 255) / 256, 256, 0, s>>>(bits, n, z);
}

// member-major bytes z[j][v] from the member-packed bits Z[j / 32][v] (bit j % 32)
__global__ void k_unpack_members(const uint32_t* Z, int n, int members, uint8_t* z) {
    const int64_t total = static_cast<int64_t>(members) * n;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i / n), v = static_cast<int>(i - static_cast<int64_t>(j) * n);
        z[i] = static_cast<uint8_t>((Z[static_cast<int64_t>(j >> 5) * n + v] >> (j & 31)) & 1u);
    }
}

void launch_unpack_members(const uint32_t* Z, int n, int members, uint8_t* z, cudaStream_t s) {
    const int64_t total = static_cast<int64_t>(members) * n;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 4096));
    count_launch();
    k_unpack_members<<<blocks, 256, 0, s>>>(Z, n, members, z);
}

// loopback exchange: out[i] = op over rows r of rows[r][i] (u32 / u64, max / min)
template <typename U, bool MAX>
__global__ void k_reduce_rows(const U* rows, int nrows, size_t count, U* out) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        U v = rows[i];
        for (int r = 1; r < nrows; ++r) {
            const U w = rows[static_cast<size_t>(r) * count + i];
            v = MAX ? (w > v ? w : v) : (w < v ? w : v);
        }
        out[i] = v;
    }
}

void launch_reduce_rows(const void* rows, int nrows, size_t count, int bytes, bool is_max, void* out, cudaStream_t s) {
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((count + 255) / 256, 1024));
    count_launch();
    if (bytes == 8) {
        if (is_max)
            k_reduce_rows<unsigned long long, true><<<blocks, 256, 0, s>>>(static_cast<const unsigned long long*>(rows),
                                                                            nrows, count, static_cast<unsigned long long*>(out));
        else
            k_reduce_rows<unsigned long long, false><<<blocks, 256, 0, s>>>(
                static_cast<const unsigned long long*>(rows), nrows, count, static_cast<unsigned long long*>(out));
    } else {
        if (is_max)
            k_reduce_rows<uint32_t, true><<<blocks, 256, 0, s>>>(static_cast<const uint32_t*>(rows), nrows, count,
                                                                 static_cast<uint32_t*>(out));
        else
            k_reduce_rows<uint32_t, false><<<blocks, 256, 0, s>>>(static_cast<const uint32_t*>(rows), nrows, count,
                                                                  static_cast<uint32_t*>(out));
    }
}

// per-member bit flags <-> one 0/1 word array per bit (an OR across ranks is then a MAX)
__global__ void k_bits_split(const uint32_t* f, int count, int nbits, uint32_t* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        for (int k = 0; k < nbits; ++k) out[static_cast<size_t>(k) * count + i] = (f[i] >> k) & 1u;
}
__global__ void k_bits_merge(const uint32_t* in, int count, int nbits, uint32_t* f) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int k = 0; k < nbits; ++k) v |= (in[static_cast<size_t>(k) * count + i] ? 1u : 0u) << k;
        f[i] = v;
    }
}

void launch_bits_split(const uint32_t* f, int count, int nbits, uint32_t* out, cudaStream_t s) {
    if (count <= 0) return;
    count_launch();
    k_bits_split<<<std::min((count + 255) / 256, 1024), 256, 0, s>>>(f, count, nbits, out);
}
void launch_bits_merge(const uint32_t* in, int count, int nbits, uint32_t* f, cudaStream_t s) {
    if (count <= 0) return;
    count_launch();
    k_bits_merge<<<std::min((count + 255) / 256, 1024), 256, 0, s>>>(in, count, nbits, f);
}

template void launch_transpose_in<float>(const double*, float*, int, int, int64_t, cudaStream_t);
template void launch_transpose_in<double>(const double*, double*, int, int, int64_t, cudaStream_t);
template void launch_transpose_out<float>(const float*, double*, int, int, int64_t, cudaStream_t);
template void launch_transpose_out<double>(const double*, double*, int, int, int64_t, cudaStream_t);
template void launch_member_dot<float>(const float*, const float*, int, int, int, int64_t, double*, cudaStream_t);
template void launch_member_dot<double>(const double*, const double*, int, int, int, int64_t, double*, cudaStream_t);
template void launch_round_pack<float>(const float*, int64_t, int, int, int, int, uint32_t*, cudaStream_t);
template void launch_round_pack<double>(const double*, int64_t, int, int, int, int, uint32_t*, cudaStream_t);

}  // namespace lcb
