// lcb_oracle.cu — exhaustive MaxCut on the GPU (oracle.cpp:50-99).
//
// The reference semantics:
// - The scan covers 2^(n-1) assignments. Node 0 stays on side 0, and code c encodes
//   z = gray(c) << 1.
// - The cut is updated incrementally as deg(f) - 2 * crossing(f) when node f flips.
// - Each visited z also stands for its complement (count += 2).
// - Ties go to the smallest encoding of min(z, ~z).
// All three are independent of how the code range is partitioned, so the range is
// split evenly over a full grid.
//
// Adjacency is held as 64-bit neighbour masks in SMEM. Multi-edges, which a raw CSR
// can carry, become extra mask layers: layer k holds the neighbours whose multiplicity
// is > k. `upper` masks keep only v > u and give the initial cut of a chunk (the
// u < v scan of cut_of_encoding, oracle.cpp:23-31).
#include <cuda_runtime.h>

#include <cstdint>

#include "lcb_internal.h"

namespace lcb {

namespace {

struct BFRec {
    long long cut;
    unsigned long long count;
    unsigned long long minenc;
};

__device__ __forceinline__ void bf_merge(BFRec& a, long long cut, unsigned long long count, unsigned long long enc) {
    if (cut > a.cut) {
        a.cut = cut;
        a.count = count;
        a.minenc = enc;
    } else if (cut == a.cut) {
        a.count += count;
        a.minenc = enc < a.minenc ? enc : a.minenc;
    }
}

__device__ __forceinline__ void bf_consider(BFRec& b, long long cut, uint64_t enc, uint64_t full) {
    const uint64_t cand = enc < (full ^ enc) ? enc : (full ^ enc);  // oracle.cpp:33-46
    bf_merge(b, cut, 2ull, cand);
}

__device__ __forceinline__ void bf_warp_reduce(BFRec& r) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long c = __shfl_xor_sync(0xffffffffu, r.cut, o);
        const unsigned long long k = __shfl_xor_sync(0xffffffffu, r.count, o);
        const unsigned long long e = __shfl_xor_sync(0xffffffffu, r.minenc, o);
        bf_merge(r, c, k, e);
    }
}

constexpr int kMaxLayers = 4;
constexpr int kMaxNodes = 64;

__global__ void __launch_bounds__(256) k_brute(const uint64_t* __restrict__ masks_g,
                                               const uint64_t* __restrict__ upper_g,
                                               const int* __restrict__ deg_g, int n, int layers,
                                               unsigned long long total, unsigned long long per_thread,
                                               BFRec* __restrict__ out) {
    __shared__ uint64_t masks[kMaxLayers * kMaxNodes];
    __shared__ uint64_t upper[kMaxLayers * kMaxNodes];
    __shared__ int deg[kMaxNodes];
    __shared__ BFRec warp_rec[8];
    for (int i = threadIdx.x; i < layers * n; i += blockDim.x) {
        masks[i] = masks_g[i];
        upper[i] = upper_g[i];
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) deg[i] = deg_g[i];
    __syncthreads();
    const uint64_t full = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    BFRec rec{-1, 0ull, ~0ull};
    const unsigned long long t = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const unsigned long long lo = t * per_thread;
    if (lo < total) {
        const unsigned long long hi = lo + per_thread < total ? lo + per_thread : total;
        uint64_t enc = (lo ^ (lo >> 1)) << 1;  // gray(lo) over nodes 1..n-1
        long long cut = 0;
        for (int u = 0; u < n; ++u) {
            const uint64_t other = ((enc >> u) & 1ull) ? ~enc : enc;
            for (int k = 0; k < layers; ++k) cut += __popcll(upper[k * n + u] & other);
        }
        bf_consider(rec, cut, enc, full);
        for (unsigned long long c = lo + 1; c < hi; ++c) {
            const int f = __ffsll(static_cast<long long>(c));  // countr_zero(c) + 1
            const uint64_t other = ((enc >> f) & 1ull) ? ~enc : enc;
            int crossing = 0;
            for (int k = 0; k < layers; ++k) crossing += __popcll(masks[k * n + f] & other);
            cut += deg[f] - 2 * crossing;
            enc ^= 1ull << f;
            bf_consider(rec, cut, enc, full);
        }
    }
    bf_warp_reduce(rec);
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) warp_rec[warp] = rec;
    __syncthreads();
    if (threadIdx.x == 0) {
        BFRec b = warp_rec[0];
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
            bf_merge(b, warp_rec[w].cut, warp_rec[w].count, warp_rec[w].minenc);
        out[blockIdx.x] = b;
    }
}

__global__ void __launch_bounds__(1024) k_brute_final(const BFRec* __restrict__ recs, int nrec,
                                                      BFRec* __restrict__ out) {
    __shared__ BFRec warp_rec[32];
    BFRec r{-1, 0ull, ~0ull};
    for (int i = threadIdx.x; i < nrec; i += blockDim.x) bf_merge(r, recs[i].cut, recs[i].count, recs[i].minenc);
    bf_warp_reduce(r);
    if ((threadIdx.x & 31) == 0) warp_rec[threadIdx.x >> 5] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
        BFRec b = warp_rec[0];
        for (int w = 1; w < 32; ++w) bf_merge(b, warp_rec[w].cut, warp_rec[w].count, warp_rec[w].minenc);
        *out = b;
    }
}

}  // namespace

int brute_force_max_layers() { return kMaxLayers; }

// masks/upper: device [layers][n]; deg: device [n]; scratch: brute_force_scratch_bytes().
// Returns the device address of the final record {int64 optimum, uint64 count (both
// orientations), uint64 min encoding}.
const void* launch_brute_force(const uint64_t* masks, const uint64_t* upper, const int* deg, int n, int layers,
                               void* scratch, cudaStream_t s) {
    const unsigned long long total = n >= 1 ? (1ull << (n - 1)) : 1ull;
    // a full grid of 148 SMs x 8 blocks; fewer threads for small scans
    const unsigned long long max_threads = 148ull * 8ull * 256ull;
    const unsigned long long threads = total < max_threads ? total : max_threads;
    const unsigned long long per_thread = (total + threads - 1) / threads;
    const unsigned blocks = static_cast<unsigned>((((total + per_thread - 1) / per_thread) + 255) / 256);
    BFRec* recs = static_cast<BFRec*>(scratch);
    BFRec* fin = recs + blocks;
    count_launch();
    k_brute<<<blocks, 256, 0, s>>>(masks, upper, deg, n, layers, total, per_thread, recs);
    count_launch();
    k_brute_final<<<1, 1024, 0, s>>>(recs, static_cast<int>(blocks), fin);
    return fin;
}

size_t brute_force_scratch_bytes() { return sizeof(BFRec) * (148 * 8 + 1); }

}  // namespace lcb
