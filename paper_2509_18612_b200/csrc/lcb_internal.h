// lcb_internal.h — shared between the kernels (lcb_kernels.cu) and the host
// runtime (lcb_runtime.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace lcb {

// ---------------------------------------------------------------------------
// counter RNG — the integer part of rng.hpp:14-43,73-75, usable on both sides
// ---------------------------------------------------------------------------
__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t combine(uint64_t key, uint64_t word) {
    return mix64(key ^ (word + 0x9e3779b97f4a7c15ULL + (key << 6) + (key >> 2)));
}
__host__ __device__ inline uint64_t rng_at(uint64_t key, uint64_t counter) {
    return mix64(key ^ (counter * 0xd6e8feb86659fd93ULL));
}
__host__ __device__ inline double rng_unit(uint64_t bits) {
    return static_cast<double>(bits >> 11) * 0x1p-53;
}

// Early-exit bits per member per iteration (ascent.cpp:74-75,91-93).
enum : uint32_t { EX_BIG = 1u, EX_NZ = 2u, EX_NOTB = 4u };
__host__ __device__ inline bool ex_continue(uint32_t b) {
    // stop iff boundary ? max_change == 0 : max_change <= 1e-12
    return (b & EX_BIG) || ((b & EX_NZ) && !(b & EX_NOTB));
}

#ifdef __CUDACC__
// The element update of ascent.cpp:66-69: y = deg*x - (Ax)_v, v = mu*v + y, raw = x + alpha*v.
// fp64: separately rounded operations, bit-identical to the reference's FMA-free scalar
// code.  fp32: ONE fused sequence shared by every kernel (K1, K1s, K2, K1n,
// K3), so an fp32 member's trajectory does not depend on which kernel ran it, i.e. on
// the batch width, the rank count or the early-exit flag.
__device__ __forceinline__ float pga_raw(float x, float ax, float& v, float alpha, float mu, float dg) {
    const float y = __fmaf_rn(dg, x, -ax);
    v = __fmaf_rn(mu, v, y);
    return __fmaf_rn(alpha, v, x);
}
__device__ __forceinline__ double pga_raw(double x, double ax, double& v, double alpha, double mu, double dg) {
    const double y = __dsub_rn(__dmul_rn(dg, x), ax);  // Lx   graph.cpp:120
    v = __dadd_rn(__dmul_rn(mu, v), y);                // v    ascent.cpp:68
    return __dadd_rn(x, __dmul_rn(alpha, v));          // raw  ascent.cpp:69
}
#endif

// ---------------------------------------------------------------------------
// device graph
// ---------------------------------------------------------------------------
struct DevGraph {
    int device = 0;
    int n = 0;
    int64_t m = 0;
    int64_t nnz = 0;
    int64_t max_degree = 0;
    double deg_mean = 0, deg_var = 0, deg_sd = 0;  // degree_stats, host-exact
    int* row_ptr = nullptr;   // [n+1]
    int* col = nullptr;       // [nnz]
    double* deg64 = nullptr;  // [n]
    float* deg32 = nullptr;   // [n]
    int* order = nullptr;     // [n] rows by degree descending (ties by index)
    // relabelled copy for the member-resident kernel (rows in `order`, uint16 columns)
    uint32_t* res_info = nullptr; // [n - heavy] light rows: (offset-in-chunk words << 16) | degree
    int* res_chunk = nullptr;     // [ceil((n-heavy)/1024)] chunk base (4-col words)
    int* res_heavy = nullptr;     // [heavy][2] absolute word offset, degree
    int res_nheavy = 0;
    int64_t res_len = 0;          // entries of res_col / res_col_fast
    uint16_t* res_col = nullptr;  // [padded nnz]
    uint16_t* res_col_fast = nullptr;  // fp32 copy, light rows in bank-balanced order (or null)
    void* dense_A = nullptr;      // bf16 [n][roundup(n,8)] adjacency for the tensor-core path (dense graphs)
    int* res_perm = nullptr;      // [n] new row -> original row (== order)
};

// ---------------------------------------------------------------------------
// PGA step (fused SpMM + heavy ball + clamp + finite check + exit flags)
// ---------------------------------------------------------------------------
template <typename T>
struct StepArgs {
    const int* row_ptr;
    const int* col;
    const T* deg;
    const int* order;
    const T* x_in;
    T* x_out;
    T* vel;
    int64_t ld;                 // row stride in elements (multiple of the warp span)
    int n;
    int W;                      // live columns (members * l)
    int l;                      // lift dimension
    const T* alpha;             // [members] or nullptr (uniform)
    const int* tlim;            // [members] iteration count per member, or nullptr
    const uint32_t* flags_prev; // [members] exit bits of it-1
    uint32_t* flags_cur;        // [members] exit bits of it (zeroed beforehand)
    uint32_t* flags_zero;       // [members] buffer to clear for it+1
    int members;
    unsigned long long* err;    // min over (member << 32 | iteration)
    int err_seg;                // members per error slot (0: one slot) — batched search
    int col_base;               // batch column of x_in[0] (L2-panel column chunks)
    T mu;
    T alpha_uniform;            // used when alpha == nullptr
    int it;
    // saturation codes of the iterate (K1, S = 1): one byte per (row, slab, lane), bit e set
    // when the lane's element e is +1, bit 4+e when it is -1.  A neighbour slab whose lane
    // elements are all on the box corners is rebuilt from its code byte (one 32-byte sector
    // per warp) instead of gathering its 512-byte slab; the values are exactly +-1, so the
    // CSR-order sums are unchanged bit for bit.
    const uint8_t* sgn_in;      // codes of x_in, or nullptr (first iteration of a loop)
    uint8_t* sgn_out;           // codes of x_out, or nullptr (not recorded)
    int64_t sgn_ld;             // bytes per row: (ld / span) * 32
    int64_t flag_off;           // K1s: byte offset of the per-row slab flags after the sign codes
    unsigned* tile_ctr;         // K1s: [2] dynamic tile counters (this launch: [launch_seq & 1])
    int64_t launch_seq;         // K1s: launches since the counters were zeroed
    int xskip;                  // K1s: a row slab whose flag is 0 keeps x only in its sign code
};

enum StepMode { MODE_STEP = 0, MODE_LAPLACE = 1 };

// member-resident persistent kernel (lcb_resident.cu), fp32 and fp64
constexpr int64_t kResidentSmemMax = 220 * 1024;
constexpr int kResidentMaxRows = 14 * 1024;
struct ResidentArgs {
    const uint32_t* rowinfo; // light row i (= relabelled row heavy+i): word offset within chunk i/1024 << 16 | degree
    const int* chunk_base;   // first 4-col word of each 1024-light-row chunk
    const int* heavy_info;   // [heavy][2]: absolute 4-col word offset, degree
    int heavy;               // rows 0..heavy-1 (degree > split) are heavy
    const uint16_t* col;     // relabelled; pad entries point at the zero row n
    const int* perm;         // new -> original row
    void* X;                 // [n][ld] (float or double), original row order, in/out
    int64_t ld;
    int n;
    int W;
    int l;
    int T;
    float alpha_uniform;
    float mu;
    double alpha_uniform64;
    double mu64;
    const void* alpha;       // [members] (float or double) or null
    const int* tlim;         // [members] or null
    unsigned long long* err;
    int err_seg;             // members per error slot (0: one slot)
    int c_base;              // first column of this launch (0 unless the wave tail is split off)
    int c_end;               // one past the last column of this launch (0: W)
};
bool resident_fits(int n, int W, int l, bool ee, int elem_bytes, int& K);

// dense tensor-core path (lcb_dense.cu), fp32 iterate, W <= 256
size_t dense_adjacency_bytes(int n);
int dense_ldp(int n);
void build_dense_adjacency(const DevGraph& g, void* A, cudaStream_t s);
void run_dense_iterations(const DevGraph& g, const void* A, const float* X_nodemajor_in, float* X_nodemajor_out,
                          int64_t ld, int W, int l, int64_t iters, float alpha_u, const float* alpha_arr,
                          const int* tlim_arr, float mu, unsigned long long* err, int err_seg, float* Xm, float* Vm,
                          void* planes, cudaStream_t s, int col_base, float* partial,
                          unsigned long long* cut_sum = nullptr);
size_t dense_partial_floats();
size_t dense_planes_bytes(int n, int W);
// L2-panel path (lcb_narrow.cu): all iterations for one narrow column panel
int narrow_panel_cols(int elem_bytes);
template <typename T>
void run_narrow_panel(const StepArgs<T>& base, const T* X_in, T* X_out, int64_t ld, int c0, int w, int64_t iters,
                      T* P0, T* P1, T* PV, cudaStream_t s);
// exhaustive MaxCut (lcb_oracle.cu)
int brute_force_max_layers();
size_t brute_force_scratch_bytes();
const void* launch_brute_force(const uint64_t* masks, const uint64_t* upper, const int* deg, int n, int layers,
                               void* scratch, cudaStream_t s);
int launch_resident(const ResidentArgs& a, int K, bool ee, int elem_bytes, cudaStream_t s);  // returns launches

template <typename T>
void launch_step(const StepArgs<T>& a, bool early_exit, int mode, cudaStream_t s);
template <typename T>
int step_span(int W);  // columns covered by one warp for this W
// K1s (lcb_stream.cu): warp-specialised streaming step over the 1 KB column slabs
// [slab0, slab0 + nslabs) for one iteration; sgn_in / sgn_out hold the slabs' sign codes
// [nslabs][n][32] bytes followed by their per-row "not saturated" flags [nslabs][n] u32
// (< 4 GB; sgn_ld unused)
template <typename T>
void launch_stream(const StepArgs<T>& a, int slab0, int nslabs, bool early_exit, cudaStream_t s);
int stream_slab_cols(int elem_bytes);  // columns of one K1s slab (1 KB of a row)
// write +-1 from the sign codes into X for every row slab whose flag is 0 (x-code mode:
// those slabs were not stored by K1s); codes/flags [nslabs][n], slab sl at column slab0 + sl
template <typename T>
void launch_xcode_fill(T* X, int64_t ld, int n, const uint8_t* codes, int64_t flag_off, int slab0, int nslabs,
                       cudaStream_t s);

template <typename T>
void launch_transpose_in(const double* src, T* dst, int n, int W, int64_t ld, cudaStream_t s);
// per-member flag words <-> nbits arrays of 0/1 words (OR across ranks as a MAX allreduce)
void launch_bits_split(const uint32_t* f, int count, int nbits, uint32_t* out, cudaStream_t s);
void launch_bits_merge(const uint32_t* in, int count, int nbits, uint32_t* f, cudaStream_t s);
template <typename T>
void launch_transpose_out(const T* src, double* dst, int n, int W, int64_t ld, cudaStream_t s);

// x . (Lx) per member from Y = LX  (trace objective, objectives.cpp:37-58)
template <typename T>
void launch_member_dot(const T* X, const T* Y, int n, int W, int l, int64_t ld, double* out,
                       cudaStream_t s);

// round + bit pack:  Z[w][v] bit b = z_{32w+b}(v)
template <typename T>
void launch_round_pack(const T* X, int64_t ld, int n, int members, int l, int lifted,
                       uint32_t* Z, cudaStream_t s);
void launch_pack_bytes(const uint8_t* z, int n, int count, uint32_t* Z, cudaStream_t s);
void launch_max_u32(const uint32_t* a, int64_t count, unsigned* out, cudaStream_t s);
// bit-sliced cut counts per member (cuts zeroed inside)
void launch_cut_count(const DevGraph& g, const uint32_t* Z, int words, unsigned long long* cuts,
                      cudaStream_t s);
// fused: cut counts + (last block) first-max argmax per segment; cuts needs words*32 + 1 entries
// K4 in one cooperative kernel: round + pack -> grid barrier -> cut counts -> argmax of
// every segment (seg_keys) -> winner bits of seg_keys[0] (win_bits, null: not extracted)
template <typename T>
void launch_epilogue(const DevGraph& g, const T* X, int64_t ld, int members, int l, int lifted, uint32_t* Z,
                     unsigned long long* cuts, int seg_size, int64_t member_base, unsigned long long* seg_keys,
                     uint32_t* win_bits, cudaStream_t s, const unsigned long long* cut_sums = nullptr);
void launch_cut_argmax(const DevGraph& g, const uint32_t* Z, int words, unsigned long long* cuts, int members,
                       int seg_size, int64_t member_base, unsigned long long* seg_keys, cudaStream_t s);
// segment argmax of packed keys; seg_keys[s] = max over members of segment s
void launch_argmax(const unsigned long long* cuts, int members, int seg_size,
                   int64_t member_base, unsigned long long* seg_keys, cudaStream_t s);
// winner assignment bits (node-packed, [ceil(n/32)]) of global key `key_src[seg]`;
// zero when the winner is not local
void launch_extract_winner(const uint32_t* Z, int n, const unsigned long long* key_src,
                           int64_t member_base, int members, uint32_t* bits, cudaStream_t s,
                           int member_offset = 0);
void launch_unpack_bits(const uint32_t* bits, int n, uint8_t* z, cudaStream_t s);
// z[j][v] (bytes, member-major) from the member-packed Z[j / 32][v]
void launch_unpack_members(const uint32_t* Z, int n, int members, uint8_t* z, cudaStream_t s);
// out[i] = max / min over the nrows rows of rows[nrows][count] (bytes = 4 or 8 per element)
void launch_reduce_rows(const void* rows, int nrows, size_t count, int bytes, bool is_max, void* out, cudaStream_t s);

// init kernels (init.cpp:20-101)
void launch_dui(const DevGraph& g, const uint64_t* col_keys, int l, double init_scale,
                const uint32_t* carry_bits, double* mean, cudaStream_t s);
void launch_idi(const DevGraph& g, double threshold, const uint64_t* col_keys, int l,
                double init_scale, const uint32_t* carry_bits, int8_t* sign_scratch,
                double* mean, cudaStream_t s);
// gaussian batch around mean ([l][n]) or around pm1(bits)/scale; member keys [members]
template <typename T>
void launch_gaussian(T* X, T* V, int64_t ld, int n, int members, int l, const uint64_t* mkeys,
                     const double* mean, const uint32_t* bits, double scale, double noise,
                     cudaStream_t s);

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct Failure {
    int status;
    std::string msg;
};
void cuda_check(cudaError_t e, const char* what);  // throws Failure{LCB_CUDA}

int num_sms(int device);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, current device),
// thread-safe, error-checked (function attributes are per device context)
void ensure_smem_attr(const void* kernel, int bytes, const char* what);

// Kernel-selection knobs: defaults, overridden by the LCB_* environment
// variable at first use and at run time by lcb_set_option (tests, A/B runs).
enum Opt : int {
    OPT_RESIDENT = 0,  // K2: -1 auto, 0 never, 1 whenever the slab fits
    OPT_STREAM,        // K1s for the HBM-streaming step: -1 auto, 1 on, 0 K1
    OPT_SIGNREC,       // K1 saturation codes: -1 auto (iterate > L2), 0 off, 1 on
    OPT_CHUNK,         // K1n L2 panels: 0 off, 1 always, -1 auto
    OPT_RES_SPLIT,     // K2 wave-tail split into a K=1 launch
    OPT_BANK_ORDER,    // K2 fp32 neighbour order at graph creation: 0 CSR, 1 warp, 2 half-warp
    OPT_BANK_REFINE,   // refinement passes of that order
    OPT_DENSE,         // K3 adjacency at graph creation: -1 auto, 0 never, 1 always
    OPT_SLAB_OUTER,    // K1s order: -1 auto (codes beyond L2), 0 iteration-major, 1 slab-major
    OPT_XCODE,         // K1s: saturated row slabs keep x in the sign code only (1 on, 0 off)
    OPT_DENSE_CUT,     // K3 graphs: unlifted cut counts as a tensor-core pass (1 on, 0 bit-sliced)
    OPT_COUNT
};
int64_t option(Opt o);

// graph arrays: the device's stream-ordered pool, cached (lcb_runtime.cu)
void* graph_alloc(size_t bytes);
void graph_free(void* p);
// stream-ordered temporaries from the same cached pool (ingest / parse scratch)
void* pool_alloc(size_t bytes, cudaStream_t st);
void pool_free(void* p, cudaStream_t st);

// graph ingest from an edge list on the device (lcb_ingest.cu): adjacency `col` [nnz]
// stays on the device (caller owns it), offsets come back to the host
struct IngestResult {
    int* col = nullptr;
    std::vector<int64_t> off;
    int64_t nnz = 0;
};
IngestResult ingest_edges(uint32_t n, const uint32_t* eu, const uint32_t* ev, int64_t m, cudaStream_t s);
// the same from device endpoint arrays already validated (ids < n, no self-loops)
IngestResult ingest_edges_device(uint32_t n, const uint32_t* du, const uint32_t* dv, int64_t m, cudaStream_t s);
// parse_edge_list (graph.cpp:136-172) of a whole text on the device, then ingest; n of the
// header out, saw_weights = some edge line carried a weight (the reference warns)
IngestResult parse_edge_text(const char* text, int64_t len, uint32_t& n_out, bool& saw_weights, cudaStream_t s);

// process-wide counters (bench evidence: launches and host<->device bytes)
void count_launch(int k = 1);
void count_h2d(size_t bytes);
void count_d2h(size_t bytes);

}  // namespace lcb
