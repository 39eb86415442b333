// lcb_ingest.cu — graph ingest on the device: the Graph(n, edges)
// constructor (graph.cpp:15-50) as radix sorts instead of a host std::sort.
//
//   validate        the first offending edge in input order decides the error, range
//                   before self-loop, with the reference's messages (graph.cpp:18-25);
//   normalise       key = (min(u,v) << 32) | max(u,v);
//   sort + unique   cub radix sort over the 32 + bits(n) key bits, DeviceSelect::Unique
//                   (std::sort + std::unique, graph.cpp:27-28);
//   symmetrise      both directions of every unique edge, sorted again by (row, col):
//                   the reference's rows come out ascending (graph.cpp:36-47), so a
//                   (row, col) sort gives the same adjacency order;
//   CSR             row boundaries of the sorted directed keys -> offsets, low words ->
//                   adjacency, written straight into the device graph.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <limits>
#include <string>
#include <vector>

#include "lcb_internal.h"
#include "liftcut_b200.h"

namespace lcb {

namespace {

__global__ void k_edge_scan(const uint32_t* __restrict__ u, const uint32_t* __restrict__ v, int64_t m, uint32_t n,
                            unsigned long long* __restrict__ first_bad) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t a = u[i], b = v[i];
        if (a >= n || b >= n || a == b) atomicMin(first_bad, static_cast<unsigned long long>(i));
    }
}

__global__ void k_edge_keys(const uint32_t* __restrict__ u, const uint32_t* __restrict__ v, int64_t m,
                            uint64_t* __restrict__ keys) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t a = u[i], b = v[i];
        const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
        keys[i] = (static_cast<uint64_t>(lo) << 32) | hi;
    }
}

__global__ void k_directed(const uint64_t* __restrict__ uk, int64_t mu, uint64_t* __restrict__ d) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < mu;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t k = uk[i];
        d[2 * i] = k;
        d[2 * i + 1] = (k << 32) | (k >> 32);
    }
}

// sorted (row << 32 | col) keys -> col[] and off[0..n] (empty rows filled)
__global__ void k_csr_from_sorted(const uint64_t* __restrict__ d, int64_t nnz, uint32_t n, int* __restrict__ col,
                                  int64_t* __restrict__ off) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= nnz;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t rc = i < nnz ? static_cast<int64_t>(d[i] >> 32) : static_cast<int64_t>(n);
        const int64_t rp = i == 0 ? -1 : static_cast<int64_t>(d[i - 1] >> 32);
        for (int64_t r = rp + 1; r <= rc; ++r) off[r] = i;
        if (i < nnz) col[i] = static_cast<int>(d[i] & 0xffffffffu);
    }
}

template <class T>
struct DevMem {
    T* p = nullptr;
    explicit DevMem(size_t count) { p = static_cast<T*>(pool_alloc(sizeof(T) * (count ? count : 1), 0)); }
    ~DevMem() { pool_free(p, 0); }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
};

int key_bits(uint32_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return 32 + b;
}

}  // namespace

IngestResult ingest_edges(uint32_t n, const uint32_t* eu, const uint32_t* ev, int64_t m, cudaStream_t s) {
    if (n == 0) throw Failure{LCB_VALIDATION, "graph must have at least one node"};
    IngestResult res;
    res.off.assign(static_cast<size_t>(n) + 1, 0);
    const unsigned grid = 148 * 8;
    if (m == 0) {
        res.col = static_cast<int*>(graph_alloc(sizeof(int) * 4));  // + K1s bulk-copy pad
        res.nnz = 0;
        return res;
    }
    DevMem<uint32_t> du(static_cast<size_t>(m)), dv(static_cast<size_t>(m));
    cuda_check(cudaMemcpyAsync(du.p, eu, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, s), "h2d(eu)");
    cuda_check(cudaMemcpyAsync(dv.p, ev, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, s), "h2d(ev)");
    count_h2d(2 * sizeof(uint32_t) * static_cast<size_t>(m));
    // validation: the first offending edge in input order (graph.cpp:17-25)
    DevMem<unsigned long long> bad(1);
    cuda_check(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s), "memset(bad)");
    count_launch();
    k_edge_scan<<<grid, 256, 0, s>>>(du.p, dv.p, m, n, bad.p);
    unsigned long long first = 0;
    cuda_check(cudaMemcpyAsync(&first, bad.p, sizeof(first), cudaMemcpyDeviceToHost, s), "d2h(bad)");
    cuda_check(cudaStreamSynchronize(s), "sync(ingest)");
    if (first != ~0ull) {
        const uint32_t a = eu[first], b = ev[first];
        if (a >= n || b >= n)
            throw Failure{LCB_VALIDATION, "edge endpoint out of range: (" + std::to_string(a) + ", " +
                                              std::to_string(b) + ") with n=" + std::to_string(n)};
        throw Failure{LCB_VALIDATION, "self-loop at node " + std::to_string(a)};
    }
    return ingest_edges_device(n, du.p, dv.p, m, s);
}

IngestResult ingest_edges_device(uint32_t n, const uint32_t* du, const uint32_t* dv, int64_t m, cudaStream_t s) {
    if (n == 0) throw Failure{LCB_VALIDATION, "graph must have at least one node"};
    IngestResult res;
    res.off.assign(static_cast<size_t>(n) + 1, 0);
    const unsigned grid = 148 * 8;
    if (m == 0) {
        res.col = static_cast<int*>(graph_alloc(sizeof(int) * 4));  // + K1s bulk-copy pad
        res.nnz = 0;
        return res;
    }
    const int bits = key_bits(n);
    // normalise, sort, unique
    DevMem<uint64_t> k0(static_cast<size_t>(m)), k1(static_cast<size_t>(m));
    count_launch();
    k_edge_keys<<<grid, 256, 0, s>>>(du, dv, m, k0.p);
    size_t tb_sort = 0, tb_uniq = 0, tb_sort2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, k0.p, k1.p, m, 0, bits, s);
    cub::DeviceSelect::Unique(nullptr, tb_uniq, k1.p, k0.p, static_cast<int64_t*>(nullptr), m, s);
    cub::DeviceRadixSort::SortKeys(nullptr, tb_sort2, k0.p, k1.p, 2 * m, 0, bits, s);
    DevMem<uint8_t> tmp(std::max(tb_sort, std::max(tb_uniq, tb_sort2)));
    DevMem<int64_t> dnu(1);
    cuda_check(cub::DeviceRadixSort::SortKeys(tmp.p, tb_sort, k0.p, k1.p, m, 0, bits, s), "sort(edges)");
    cuda_check(cub::DeviceSelect::Unique(tmp.p, tb_uniq, k1.p, k0.p, dnu.p, m, s), "unique(edges)");
    count_launch(2);
    int64_t mu = 0;
    cuda_check(cudaMemcpyAsync(&mu, dnu.p, sizeof(mu), cudaMemcpyDeviceToHost, s), "d2h(m)");
    cuda_check(cudaStreamSynchronize(s), "sync(unique)");
    const int64_t nnz = 2 * mu;
    if (nnz > std::numeric_limits<int>::max()) throw Failure{LCB_VALIDATION, "graph exceeds 2^31 adjacency entries"};
    // symmetrise and sort by (row, col)
    DevMem<uint64_t> d0(static_cast<size_t>(nnz)), d1(static_cast<size_t>(nnz));
    count_launch();
    k_directed<<<grid, 256, 0, s>>>(k0.p, mu, d0.p);
    cuda_check(cub::DeviceRadixSort::SortKeys(tmp.p, tb_sort2, d0.p, d1.p, nnz, 0, bits, s), "sort(adjacency)");
    count_launch();
    // CSR
    DevMem<int64_t> doff(static_cast<size_t>(n) + 1);
    int* col = nullptr;
    col = static_cast<int*>(graph_alloc(sizeof(int) * (static_cast<size_t>(nnz) + 4)));  // K1s copies 16-byte runs
    count_launch();
    k_csr_from_sorted<<<grid, 256, 0, s>>>(d1.p, nnz, n, col, doff.p);
    cuda_check(cudaMemcpyAsync(res.off.data(), doff.p, sizeof(int64_t) * (static_cast<size_t>(n) + 1),
                               cudaMemcpyDeviceToHost, s),
               "d2h(offsets)");
    count_d2h(sizeof(int64_t) * (static_cast<size_t>(n) + 1));
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        graph_free(col);
        cuda_check(e, "sync(csr)");
    }
    res.col = col;
    res.nnz = nnz;
    return res;
}

}  // namespace lcb
