// lcb_parse.cu — Gset / edge-list text parsed on the device (the
// reader half of graph ingest): parse_edge_list (graph.cpp:136-172) for a whole file at
// once instead of a std::getline / istringstream loop.
//
//   lines       a line starts at 0 and after every '\n' (std::getline: a trailing '\n'
//               ends the last line, it does not open an empty one); starts compacted
//               with cub::DeviceSelect::Flagged;
//   per line    one thread: blank / comment exactly as is_comment_or_blank (only ' ',
//               '\t', '\r' skipped; '%' or '#' first), else `ls >> u >> v` with the
//               istream rules for long long (leading isspace skipped, optional sign,
//               >= 1 digit, stop at the first non-digit, overflow fails) and `ls >> w`
//               for the weight warning;
//   header      the first data line ("n m", n > 0, m >= 0);
//   errors      the first offending data line after the header decides, with the
//               reference's messages: parse failure -> "expected edge", then the id range
//               [1, n], then self-loop (ValidationError);
//   edges       data lines after the header compacted to 0-based (u, v) and handed to
//               the device Graph(n, edges) ingest (lcb_ingest.cu).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <string>

#include "lcb_internal.h"
#include "liftcut_b200.h"

namespace lcb {

namespace {

enum : uint8_t { L_SKIP = 0, L_DATA = 1, L_FAIL = 2 };  // blank/comment, two integers, parse failure

__device__ __forceinline__ bool is_space(char c) {  // std::isspace in the "C" locale
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// istream >> long long: skip isspace, optional sign, at least one digit, stop at the first
// non-digit; false on no digits or overflow
__device__ bool parse_ll(const char* t, int64_t& p, int64_t end, long long& out) {
    while (p < end && is_space(t[p])) ++p;
    bool neg = false;
    if (p < end && (t[p] == '+' || t[p] == '-')) {
        neg = t[p] == '-';
        ++p;
    }
    unsigned long long acc = 0;
    int digits = 0;
    bool over = false;
    const unsigned long long lim = neg ? static_cast<unsigned long long>(LLONG_MAX) + 1ull
                                       : static_cast<unsigned long long>(LLONG_MAX);
    while (p < end && t[p] >= '0' && t[p] <= '9') {
        const unsigned d = static_cast<unsigned>(t[p] - '0');
        if (acc > (lim - d) / 10ull) over = true;
        else acc = acc * 10ull + d;
        ++digits;
        ++p;
    }
    if (!digits || over) return false;
    out = neg ? static_cast<long long>(0ull - acc) : static_cast<long long>(acc);
    return true;
}

// istream >> double would succeed: a mantissa with at least one digit
__device__ bool has_number(const char* t, int64_t p, int64_t end) {
    while (p < end && is_space(t[p])) ++p;
    if (p < end && (t[p] == '+' || t[p] == '-')) ++p;
    if (p < end && t[p] >= '0' && t[p] <= '9') return true;
    return p + 1 < end && t[p] == '.' && t[p + 1] >= '0' && t[p + 1] <= '9';
}

__global__ void k_line_flags(const char* __restrict__ t, int64_t len, uint8_t* __restrict__ flag,
                             unsigned long long* __restrict__ count) {
    unsigned c = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool f = i == 0 || t[i - 1] == '\n';
        flag[i] = f ? 1 : 0;
        c += f ? 1u : 0u;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, static_cast<unsigned long long>(c));
}

// one thread per line: kind, the two integers, weight present
__global__ void k_parse_lines(const char* __restrict__ t, int64_t len, const int64_t* __restrict__ start,
                              int64_t lines, uint8_t* __restrict__ kind, long long* __restrict__ a,
                              long long* __restrict__ b, uint8_t* __restrict__ wt,
                              unsigned long long* __restrict__ first_data) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < lines;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t p = start[i];
        const int64_t end = i + 1 < lines ? start[i + 1] - 1 : (len > 0 && t[len - 1] == '\n' ? len - 1 : len);
        int64_t q = p;
        while (q < end && (t[q] == ' ' || t[q] == '\t' || t[q] == '\r')) ++q;
        uint8_t k = L_SKIP;
        long long x = 0, y = 0;
        uint8_t w = 0;
        if (q < end && t[q] != '%' && t[q] != '#') {
            k = (parse_ll(t, p, end, x) && parse_ll(t, p, end, y)) ? L_DATA : L_FAIL;
            if (k == L_DATA) w = has_number(t, p, end) ? 1 : 0;
            atomicMin(first_data, static_cast<unsigned long long>(i));
        }
        kind[i] = k;
        a[i] = x;
        b[i] = y;
        wt[i] = w;
    }
}

// data lines after the header: first error (line << 2 | code), weights, edge flags
__global__ void k_check_edges(const uint8_t* __restrict__ kind, const long long* __restrict__ a,
                              const long long* __restrict__ b, const uint8_t* __restrict__ wt, int64_t lines,
                              int64_t header, long long n, unsigned long long* __restrict__ first_err,
                              unsigned* __restrict__ weights, uint8_t* __restrict__ is_edge,
                              uint32_t* __restrict__ eu, uint32_t* __restrict__ ev) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < lines;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint8_t k = kind[i];
        const bool edge = i > header && k != L_SKIP;
        uint8_t ok = 0;
        if (edge) {
            unsigned code = 0;
            const long long u = a[i], v = b[i];
            if (k == L_FAIL)
                code = 1;
            else if (u < 1 || u > n || v < 1 || v > n)
                code = 2;
            else if (u == v)
                code = 3;
            if (code)
                atomicMin(first_err, (static_cast<unsigned long long>(i) << 2) | code);
            else {
                ok = 1;
                eu[i] = static_cast<uint32_t>(u - 1);
                ev[i] = static_cast<uint32_t>(v - 1);
                if (wt[i]) *weights = 1u;
            }
        }
        is_edge[i] = ok;
    }
}

template <class T>
struct Buf {
    T* p = nullptr;
    explicit Buf(size_t count) { p = static_cast<T*>(pool_alloc(sizeof(T) * (count ? count : 1), 0)); }
    ~Buf() { pool_free(p, 0); }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
};

}  // namespace

IngestResult parse_edge_text(const char* text, int64_t len, uint32_t& n_out, bool& saw_weights, cudaStream_t s) {
    if (len < 0) throw Failure{LCB_VALIDATION, "negative text length"};
    const unsigned grid = 148 * 8;
    if (len == 0) throw Failure{LCB_PARSE, "empty input: missing \"n m\" header"};
    Buf<char> t(static_cast<size_t>(len));
    cuda_check(cudaMemcpyAsync(t.p, text, static_cast<size_t>(len), cudaMemcpyHostToDevice, s), "h2d(text)");
    count_h2d(static_cast<size_t>(len));
    // line starts
    Buf<uint8_t> flag(static_cast<size_t>(len));
    Buf<int64_t> nsel(1);
    int64_t lines = 0;
    cuda_check(cudaMemsetAsync(nsel.p, 0, sizeof(int64_t), s), "memset(lines)");
    count_launch();
    k_line_flags<<<grid, 256, 0, s>>>(t.p, len, flag.p, reinterpret_cast<unsigned long long*>(nsel.p));
    cuda_check(cudaMemcpyAsync(&lines, nsel.p, sizeof(lines), cudaMemcpyDeviceToHost, s), "d2h(line count)");
    cuda_check(cudaStreamSynchronize(s), "sync(line count)");
    size_t tb = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, cub::CountingInputIterator<int64_t>(0), flag.p,
                               static_cast<int64_t*>(nullptr), nsel.p, len, s);
    Buf<int64_t> start(static_cast<size_t>(lines));  // exactly the line starts
    {
        Buf<uint8_t> tmp(tb);
        cuda_check(cub::DeviceSelect::Flagged(tmp.p, tb, cub::CountingInputIterator<int64_t>(0), flag.p, start.p,
                                              nsel.p, len, s),
                   "select(lines)");
        count_launch();
        cuda_check(cudaMemcpyAsync(&lines, nsel.p, sizeof(lines), cudaMemcpyDeviceToHost, s), "d2h(lines)");
        cuda_check(cudaStreamSynchronize(s), "sync(lines)");
    }
    // per-line parse
    Buf<uint8_t> kind(static_cast<size_t>(lines)), wt(static_cast<size_t>(lines));
    Buf<long long> a(static_cast<size_t>(lines)), b(static_cast<size_t>(lines));
    Buf<unsigned long long> first(2);
    cuda_check(cudaMemsetAsync(first.p, 0xff, 2 * sizeof(unsigned long long), s), "memset(first)");
    count_launch();
    k_parse_lines<<<grid, 256, 0, s>>>(t.p, len, start.p, lines, kind.p, a.p, b.p, wt.p, first.p);
    unsigned long long header = 0;
    cuda_check(cudaMemcpyAsync(&header, first.p, sizeof(header), cudaMemcpyDeviceToHost, s), "d2h(header)");
    cuda_check(cudaStreamSynchronize(s), "sync(parse)");
    if (header == ~0ull) throw Failure{LCB_PARSE, "empty input: missing \"n m\" header"};
    const int64_t h = static_cast<int64_t>(header);
    uint8_t hk = 0;
    long long n = 0, m = 0;
    cuda_check(cudaMemcpy(&hk, kind.p + h, 1, cudaMemcpyDeviceToHost), "d2h(header kind)");
    cuda_check(cudaMemcpy(&n, a.p + h, sizeof(n), cudaMemcpyDeviceToHost), "d2h(n)");
    cuda_check(cudaMemcpy(&m, b.p + h, sizeof(m), cudaMemcpyDeviceToHost), "d2h(m)");
    if (hk != L_DATA || n <= 0 || m < 0)
        throw Failure{LCB_PARSE, "line " + std::to_string(h + 1) + ": expected header \"n m\""};
    if (n > static_cast<long long>(INT_MAX)) throw Failure{LCB_VALIDATION, "graph exceeds 2^31 nodes"};
    // edges
    Buf<uint8_t> is_edge(static_cast<size_t>(lines));
    Buf<uint32_t> eu(static_cast<size_t>(lines)), ev(static_cast<size_t>(lines));
    Buf<unsigned> weights(1);
    cuda_check(cudaMemsetAsync(weights.p, 0, sizeof(unsigned), s), "memset(weights)");
    count_launch();
    k_check_edges<<<grid, 256, 0, s>>>(kind.p, a.p, b.p, wt.p, lines, h, n, first.p + 1, weights.p, is_edge.p, eu.p,
                                       ev.p);
    unsigned long long err = 0;
    unsigned wflag = 0;
    cuda_check(cudaMemcpyAsync(&err, first.p + 1, sizeof(err), cudaMemcpyDeviceToHost, s), "d2h(err)");
    cuda_check(cudaMemcpyAsync(&wflag, weights.p, sizeof(wflag), cudaMemcpyDeviceToHost, s), "d2h(weights)");
    cuda_check(cudaStreamSynchronize(s), "sync(check)");
    if (err != ~0ull) {
        const int64_t line = static_cast<int64_t>(err >> 2) + 1;
        const unsigned code = static_cast<unsigned>(err & 3u);
        if (code == 1) throw Failure{LCB_PARSE, "line " + std::to_string(line) + ": expected edge \"u v [w]\""};
        if (code == 2)
            throw Failure{LCB_PARSE, "line " + std::to_string(line) + ": node id out of range [1, " +
                                         std::to_string(n) + "]"};
        long long u = 0;
        cuda_check(cudaMemcpy(&u, a.p + (line - 1), sizeof(u), cudaMemcpyDeviceToHost), "d2h(u)");
        throw Failure{LCB_VALIDATION, "line " + std::to_string(line) + ": self-loop at node " + std::to_string(u)};
    }
    // compact the edge lines, then Graph(n, edges) on the device
    Buf<uint32_t> cu(static_cast<size_t>(lines)), cv(static_cast<size_t>(lines));
    int64_t me = 0;
    {
        size_t tb2 = 0;
        cub::DeviceSelect::Flagged(nullptr, tb2, eu.p, is_edge.p, cu.p, nsel.p, lines, s);
        Buf<uint8_t> tmp(tb2);
        cuda_check(cub::DeviceSelect::Flagged(tmp.p, tb2, eu.p, is_edge.p, cu.p, nsel.p, lines, s), "select(u)");
        cuda_check(cub::DeviceSelect::Flagged(tmp.p, tb2, ev.p, is_edge.p, cv.p, nsel.p, lines, s), "select(v)");
        count_launch(2);
        cuda_check(cudaMemcpyAsync(&me, nsel.p, sizeof(me), cudaMemcpyDeviceToHost, s), "d2h(m)");
        cuda_check(cudaStreamSynchronize(s), "sync(select)");
    }
    n_out = static_cast<uint32_t>(n);
    saw_weights = wflag != 0;
    return ingest_edges_device(n_out, cu.p, cv.p, me, s);
}

}  // namespace lcb
