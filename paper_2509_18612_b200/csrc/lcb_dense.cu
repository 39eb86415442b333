// lcb_dense.cu — K3: dense-graph PGA step on the 5th-generation tensor cores.
//
// For dense graphs (config 3: ER n=20k p=0.5) the Laplacian product is a GEMM
//   D[v][c] = sum_u A[v][u] X[u][c]      (M = n nodes, N = W columns, K = n)
// with A the 0/1 adjacency — exact in bf16.  X (fp32) is split exactly into three
// bf16 planes hi + mid + lo (8 significand bits each = all 24 of fp32); the three
// products accumulate into ONE fp32 accumulator in tensor memory, so the sum is an
// fp32-faithful A·X (executed flops = 3x algorithmic).
//
// One CTA per 128-row tile of A (M=128), all N = W (<= 256) columns:
//   warp 0  TMA producer: A tile [128 x 32] + plane tiles [N x 32] per K step,
//           64-byte swizzle, L2 evict-first for A / evict-last for the planes;
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer (kind::f16, bf16 x bf16
//           -> fp32, 2 MMAs of K=16 per plane and K step), tcgen05.commit frees ring
//           slots and finally signals the epilogue;
//   warps 2-9 epilogue (two warps per TMEM lane quarter, half the columns each):
//           tcgen05.ld 32 columns at a time, fused y = deg*x - Ax; v = mu v + y;
//           raw = x + alpha v; finite check; clamp (ascent.cpp:66-77), writes x' / v'
//           (fp32, member-major [W][n]) and the three bf16 planes of x' for the next
//           iteration (planes double-buffered: every CTA reads all of them).
// Both operands are stored blocked (one contiguous 8 / 16 KB run per TMA box).
//
// Zero-plane skipping: once x' sits on the box corners (x = +-1 exactly, after a few
// iterations on config 3) its mid / lo planes are exactly zero.  The epilogue records,
// per 32-node K step, whether any mid / lo entry is nonzero; the next launch loads and
// multiplies only the hi plane for the other K steps (adding A*0 changes nothing), and
// when at least half the K steps skip it switches the ring to 8 narrower slots.
// e4m3 units: an aligned pair of such K steps (64 nodes, all x = +-1 or 0) runs as
// kind::f8f6f4 MMAs on an e4m3 copy of A (0/1) and of the hi plane (+-1): both exact in
// e4m3, the products and their sums are integers, so the fp32 accumulator sees the same
// values at half the operand bytes and twice the MMA rate.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "lcb_internal.h"

namespace lcb {

namespace {

constexpr int kBM = 128;                          // rows of A per CTA (UMMA M)
constexpr int kBK = 32;                           // K per stage (32 bf16 = one 64-byte swizzle row)
constexpr int kStages = 4;                        // full mode: 4 x 56 KB slots (A + 3 planes)
constexpr int kSkipStages = 8;                    // skip mode: 8 x 24 KB slots (A + hi) + 1 low slot (mid + lo)
constexpr int kATileBytes = kBM * kBK * 2;        // 8 KB
constexpr int kMaxFlagWords = 64;
#ifndef LCB_DENSE_EPI_WARPS
#define LCB_DENSE_EPI_WARPS 16
#endif
// epilogue warps: 4 (one per TMEM lane quarter), 8 or 16 (2 / 4 warps per quarter split the
// columns); config 3: 96.6 ms/step at 8, 89.9 ms at 16
constexpr int kEpiWarps = LCB_DENSE_EPI_WARPS;
constexpr int kThreadsDense = 64 + 32 * kEpiWarps;                 // K-step flags held in SMEM (n <= 65536)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// long waits (the epilogue waits for the whole main loop): back off between probes so the
// spinning warps leave the issue slots to the producer / MMA threads
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    for (;;) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(256);
    }
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand, 64-byte swizzle: rows of 64 B (kBK bf16), 8-row atoms 512 B apart.
__device__ __forceinline__ uint64_t umma_desc_k_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3fffu);       // start address
    d |= static_cast<uint64_t>(1u) << 16;                      // LBO (unused for swizzled K-major) = 16 B
    d |= static_cast<uint64_t>(512u >> 4) << 32;               // SBO = 512 B between 8-row groups
    d |= static_cast<uint64_t>(1u) << 46;                      // descriptor version (sm_100)
    d |= static_cast<uint64_t>(4u) << 61;                      // SWIZZLE_64B
    return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4)                                   // D format F32
           | (1u << 7)                                 // A BF16
           | (1u << 10)                                // B BF16
           | (static_cast<uint32_t>(N >> 3) << 17)     // N >> 3
           | (static_cast<uint32_t>(M >> 4) << 24);    // M >> 4
}

// kind::f8f6f4 instruction descriptor: e4m3 x e4m3 -> fp32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_e4m3(int M, int N) {
    return (1u << 4)                                   // D format F32
           | (0u << 7)                                 // A E4M3
           | (0u << 10)                                // B E4M3
           | (static_cast<uint32_t>(N >> 3) << 17)     // N >> 3
           | (static_cast<uint32_t>(M >> 4) << 24);    // M >> 4
}
__device__ __forceinline__ void umma_e4m3(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// exact split of an fp32 value into three bf16 (truncating each remainder is exact:
// x - bf16(x) is representable in fp32 and has <= 16 significant bits left)
__device__ __forceinline__ void split3(float x, __nv_bfloat16& h, __nv_bfloat16& m, __nv_bfloat16& l) {
    h = __float2bfloat16_rz(x);
    const float r1 = x - __bfloat162float(h);
    m = __float2bfloat16_rz(r1);
    const float r2 = r1 - __bfloat162float(m);
    l = __float2bfloat16_rn(r2);
}

struct DenseArgs {
    const float* deg;        // [n]
    float* X;                // [W][n] member-major fp32 iterate (in place)
    float* V;                // [W][n] velocity (in place)
    __nv_bfloat16* planes_out;  // blocked planes of x' for the next iteration (plane_index)
    int n;
    int ldx;                 // row pitch of X / V (elements)
    int nks;                 // 32-node K steps
    int nks64;               // 64-node steps of the e4m3 operands
    int nb;                  // member rows per plane block (UMMA N: 64 / 128 / 256)
    int W;                   // live columns (<= 256, multiple of 16)
    int l;
    int col_base;            // first batch column of this launch (column chunks of <= 256)
    float mu;
    float alpha_uniform;
    const float* alpha;      // [members] or null
    const int* tlim;         // [members] or null
    unsigned long long* err;
    int err_seg;
    int it;
    int tile_base;           // first M-tile of this launch
    int k_split;             // K pieces per tile (1: whole K, fused epilogue)
    float* partial;          // k_split > 1: fp32 partial sums [block][N][128]
    uint8_t* plane8_out;        // e4m3 copy of the hi plane, blocked [64-node step][nb][64], pre-swizzled
    const uint8_t* plane8_in;   // the same, written by the previous iteration
    const uint8_t* adj8;        // e4m3 adjacency, blocked [tile][64-node step][128][64], pre-swizzled
    int fp8;                    // e4m3 operands available for fully corner-valued 64-node steps
    const uint32_t* kflags_in;  // [K steps] 0: the mid/lo planes of this 32-node K step are all zero
    uint32_t* kflags_out;       // the same for the planes written by this launch
    unsigned long long* cut_sum;  // cut mode: [W] sum_v s_v (A s)_v of the sign planes (no step)
};

// Blocked B operand: plane p, K step ks = node / 32 -> one contiguous [nb][32] bf16 block
// (nb x 64 B), the exact box one TMA load fetches; likewise A is stored as contiguous
// [128][32] blocks per (M tile, K step), so both operands stream as whole 8-16 KB runs.
__host__ __device__ __forceinline__ int64_t plane_index(int p, int row, int c, int nks, int nb) {
    return ((static_cast<int64_t>(p) * nks + (row >> 5)) * nb + c) * 32 + (row & 31);
}
// e4m3 operands are stored pre-swizzled: a block of 64-byte rows holds exactly the
// SWIZZLE_64B shared-memory image (16-byte chunk j of row r at chunk j ^ ((r >> 1) & 3)),
// so one contiguous bulk copy (no tensor map walk over 64-byte rows) lands it ready for
// the UMMA descriptor
__host__ __device__ __forceinline__ int sw64(int r, int b) {
    return r * 64 + ((((b >> 4) ^ ((r >> 1) & 3)) << 4) | (b & 15));
}
__host__ __device__ __forceinline__ int64_t plane8_index(int row, int c, int nb) {
    return (static_cast<int64_t>(row >> 6) * nb << 6) + sw64(c, row & 63);
}
__host__ __device__ __forceinline__ int64_t adj8_index(int v, int u, int nks64) {
    return ((static_cast<int64_t>(v >> 7) * nks64 + (u >> 6)) << 13) + sw64(v & 127, u & 63);
}
__host__ __device__ __forceinline__ int64_t adj_index(int v, int u, int nks) {
    return ((static_cast<int64_t>(v >> 7) * nks + (u >> 5)) * 128 + (v & 127)) * 32 + (u & 31);
}

// Fused heavy-ball step for one (row, column) given Ax (ascent.cpp:66-77) + plane split.
// Returns whether the mid / lo planes of x' are nonzero (x' = +-1 exactly splits to hi only).
__device__ __forceinline__ bool finish_element(const DenseArgs& a, int row, int c, float ax, float dg) {
    const int m = (a.col_base + c) / a.l;
    bool act = true;
    float alpha = a.alpha_uniform;
    if (a.tlim) act = a.it < __ldg(a.tlim + m);
    if (a.alpha) alpha = __ldg(a.alpha + m);
    float* xp = a.X + static_cast<int64_t>(c) * a.ldx + row;
    float* vp = a.V + static_cast<int64_t>(c) * a.ldx + row;
    float x = *xp;
    if (act) {
        float v = *vp;
        const float raw = pga_raw(x, ax, v, alpha, a.mu, dg);  // ascent.cpp:66-69
        if (!isfinite(raw))
            atomicMin(a.err + (a.err_seg ? m / a.err_seg : 0),
                      (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned>(a.it));
        x = raw < -1.f ? -1.f : (raw > 1.f ? 1.f : raw);  // ascent.cpp:73
        *xp = x;
        *vp = v;
    }
    __nv_bfloat16 h, mi, lo;
    split3(x, h, mi, lo);
    const int64_t po = plane_index(0, row, c, a.nks, a.nb);
    const int64_t ps = static_cast<int64_t>(a.nks) * a.nb * 32;
    a.planes_out[po] = h;
    a.planes_out[ps + po] = mi;
    a.planes_out[2 * ps + po] = lo;
    if (a.plane8_out)  // exact where it is used: only steps whose x are all +-1 / 0
        a.plane8_out[plane8_index(row, c, a.nb)] =
            static_cast<uint8_t>(__nv_cvt_float_to_fp8(x, __NV_SATFINITE, __NV_E4M3));
    return ((__bfloat16_as_ushort(mi) | __bfloat16_as_ushort(lo)) & 0x7fffu) != 0;
}

// 8 columns [c0, c0 + 8) of one row from one tcgen05.ld.x8: the x / v loads are all
// issued before the first store, parameters and addresses are hoisted, and the member
// index (a division) is only formed on the per-member paths.  Kept to 8 columns so the
// epilogue loop body stays small: the fully unrolled 32-column version overflowed the
// instruction cache ("no instruction" stalls dominated the epilogue).
__device__ __forceinline__ bool finish_chunk8(const DenseArgs& a, int row, int c0, const uint32_t (&r)[8], float dg) {
    const int64_t ld = a.ldx;
    float* xr = a.X + static_cast<int64_t>(c0) * ld + row;
    float* vr = a.V + static_cast<int64_t>(c0) * ld + row;
    const int cn = a.W - c0 < 8 ? a.W - c0 : 8;
    float xs[8], vs[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (j < cn) {
            xs[j] = xr[j * ld];
            vs[j] = vr[j * ld];
        }
    const bool uniform = !a.alpha && !a.tlim;
    __nv_bfloat16* P = a.planes_out + plane_index(0, row, c0, a.nks, a.nb);
    const int64_t ps = static_cast<int64_t>(a.nks) * a.nb * 32;
    uint8_t* P8 = a.plane8_out ? a.plane8_out + (static_cast<int64_t>(row >> 6) * a.nb << 6) : nullptr;
    const int b8 = row & 63;
    bool low = false;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (j >= cn) continue;
        const int c = c0 + j;
        float alpha = a.alpha_uniform;
        bool act = true;
        if (!uniform) {
            const int m = (a.col_base + c) / a.l;
            if (a.tlim) act = a.it < __ldg(a.tlim + m);
            if (a.alpha) alpha = __ldg(a.alpha + m);
        }
        float x = xs[j];
        if (act) {
            const float ax = __uint_as_float(r[j]);
            float v = vs[j];
            const float raw = pga_raw(x, ax, v, alpha, a.mu, dg);  // ascent.cpp:66-69
            if (!isfinite(raw)) {
                const int m = (a.col_base + c) / a.l;
                atomicMin(a.err + (a.err_seg ? m / a.err_seg : 0),
                          (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned>(a.it));
            }
            x = raw < -1.f ? -1.f : (raw > 1.f ? 1.f : raw);  // ascent.cpp:73
            xr[j * ld] = x;
            vr[j * ld] = v;
        }
        __nv_bfloat16 h, mi, lo;
        split3(x, h, mi, lo);
        P[j * 32] = h;
        P[ps + j * 32] = mi;
        P[2 * ps + j * 32] = lo;
        if (P8) P8[sw64(c, b8)] = static_cast<uint8_t>(__nv_cvt_float_to_fp8(x, __NV_SATFINITE, __NV_E4M3));
        low |= ((__bfloat16_as_ushort(mi) | __bfloat16_as_ushort(lo)) & 0x7fffu) != 0;
    }
    return low;
}

// Cut mode, 8 columns of one row: the accumulator holds (A s)_v for the sign planes
// s = x > 0 ? +1 : -1 (objectives.cpp:81-96), an exact integer in fp32; sum s_v (A s)_v
// over the warp's 32 rows per column and add it to the column's total.
__device__ __forceinline__ void cut_chunk8(const DenseArgs& a, int row, bool live, int c0, const uint32_t (&r)[8]) {
    const int lane = threadIdx.x & 31;
    const float* xr = a.X + static_cast<int64_t>(c0) * a.ldx + row;
    int mine = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        int d = 0;
        if (live && c0 + j < a.W) {
            d = __float2int_rn(__uint_as_float(r[j]));
            if (!(xr[j * a.ldx] > 0.f)) d = -d;
        }
        d = __reduce_add_sync(0xffffffffu, d);
        if (lane == j) mine = d;
    }
    if (lane < 8 && c0 + lane < a.W && mine)
        atomicAdd(a.cut_sum + c0 + lane, static_cast<unsigned long long>(static_cast<long long>(mine)));
}

// Two smem carve-ups of the same ring, chosen per launch from the K-step flags of the
// previous iteration (all CTAs count them, so all agree):
//   full mode  kStages slots of A + hi + mid + lo;
//   skip mode  (>= half of the K steps have all-zero mid / lo planes, i.e. the iterate
//              sits on the box corners): kSkipStages slots of A + hi, so twice as many
//              K steps are in flight, and one extra slot for the mid / lo planes of the
//              few K steps that still need them.
template <int N>
__global__ void __launch_bounds__(kThreadsDense, 1)
    k_dense_step(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmP, DenseArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kPlaneTile = N * kBK * 2;             // bytes of one plane tile (multiple of 512)
    constexpr int kFullSlot = kATileBytes + 3 * kPlaneTile;
    constexpr int kSkipSlot = kATileBytes + kPlaneTile;
    __shared__ __align__(8) uint64_t full_bar[kSkipStages], empty_bar[kSkipStages], low_empty, acc_bar;
    __shared__ uint32_t tmem_base_sh;
    __shared__ int zero_steps;
    __shared__ uint32_t qflag[4];                  // per TMEM lane quarter: nonzero mid / lo planes
    __shared__ uint32_t need_low[kMaxFlagWords];  // bit ks: K step ks needs its mid / lo planes

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int tile = a.tile_base + static_cast<int>(blockIdx.x) / a.k_split;
    const int piece = static_cast<int>(blockIdx.x) % a.k_split;
    const int m0 = tile * kBM;
    const int nk_all = (a.n + kBK - 1) / kBK;
    const int kb = piece * nk_all / a.k_split;
    const int nk = (piece + 1) * nk_all / a.k_split - kb;   // K steps of this block
    // 1024-byte aligned ring
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));

    if (threadIdx.x == 0) zero_steps = 0;
    if (threadIdx.x < 4) qflag[threadIdx.x] = 0u;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kSkipStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        mbar_init(&low_empty, 1);
        mbar_init(&acc_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmP)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    // programmatic dependent launch: the set-up above overlaps the previous launch's tail;
    // its outputs (flags, planes, X / V) are read only after the wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // the flags go to SMEM once: the single producer / MMA threads must not pay a global
    // load latency per K step
    const bool flags = a.kflags_in && nk_all <= 32 * kMaxFlagWords;
    if (flags) {
        int z = 0;
        for (int w0 = warp * 32; w0 < nk_all; w0 += 32 * (blockDim.x >> 5)) {
            const int i = w0 + lane;
            const bool nz = i >= nk_all || a.kflags_in[i] != 0;
            const uint32_t b = __ballot_sync(0xffffffffu, nz);
            if (lane == 0) need_low[w0 >> 5] = b;
            z += 32 - __popc(b);
        }
        if (lane == 0 && z) atomicAdd(&zero_steps, z);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const bool skipmode = flags && 2 * zero_steps >= nk_all;
    const int S = skipmode ? kSkipStages : kStages;
    const int slot_bytes = skipmode ? kSkipSlot : kFullSlot;
    uint8_t* low = ring + kSkipStages * kSkipSlot;  // skip mode only: mid, lo tiles
    // the unit sequence over this block's K steps, derived identically by producer and MMA:
    // an e4m3 unit covers an aligned pair of 32-node steps whose mid / lo planes are zero
    auto need = [&](int ks) { return !flags || ((need_low[ks >> 5] >> (ks & 31)) & 1u) != 0u; };
    auto fp8_unit = [&](int k) {
        const int ks = kb + k;
        return a.fp8 && skipmode && (ks & 1) == 0 && k + 1 < nk && !need(ks) && !need(ks + 1);
    };

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            // A streams once per iteration (evict first); the planes are re-read by every CTA
            uint64_t pol_a, pol_p;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_a));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_p));
            int low_uses = 0;
            for (int k = 0, u = 0; k < nk; ++u) {
                const int s = u % S;
                const int ks = kb + k;
                if (u >= S) mbar_wait(&empty_bar[s], ((u / S) - 1) & 1);
                uint8_t* st = ring + s * slot_bytes;
                if (fp8_unit(k)) {
                    // 64 nodes whose x are all +-1: e4m3 A and hi, same slot bytes as one
                    // bf16 K step (128 x 64 B + N x 64 B)
                    mbar_expect_tx(&full_bar[s], kATileBytes + kPlaneTile);
                    bulk_load_hint(st, a.adj8 + ((static_cast<int64_t>(tile) * a.nks64 + (ks >> 1)) << 13), kATileBytes,
                                   &full_bar[s], pol_a);
                    bulk_load_hint(st + kATileBytes, a.plane8_in + static_cast<int64_t>(ks >> 1) * N * 64, kPlaneTile,
                                   &full_bar[s], pol_p);
                    k += 2;
                    continue;
                }
                // all-zero mid / lo planes (every x of these 32 nodes is +-1): skip them
                const int np = need(ks) ? 3 : 1;
                mbar_expect_tx(&full_bar[s], kATileBytes + np * kPlaneTile);
                tma_load_2d_hint(st, &tmA, &full_bar[s], 0, (tile * a.nks + ks) * kBM, pol_a);
                tma_load_2d_hint(st + kATileBytes, &tmP, &full_bar[s], 0, ks * N, pol_p);
                if (np == 3) {
                    uint8_t* lp = st + kATileBytes + kPlaneTile;
                    if (skipmode) {
                        if (low_uses > 0) mbar_wait(&low_empty, (low_uses - 1) & 1);
                        ++low_uses;
                        lp = low;
                    }
                    tma_load_2d_hint(lp, &tmP, &full_bar[s], 0, (a.nks + ks) * N, pol_p);
                    tma_load_2d_hint(lp + kPlaneTile, &tmP, &full_bar[s], 0, (2 * a.nks + ks) * N, pol_p);
                }
                k += 1;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = idesc_bf16(kBM, N);
        constexpr uint32_t idesc8 = idesc_e4m3(kBM, N);
        if (lane == 0) {
            bool first = true;
            for (int k = 0, u = 0; k < nk; ++u) {
                const int s = u % S;
                mbar_wait(&full_bar[s], (u / S) & 1);
                tc_fence_after();
                const uint32_t st = smem_u32(ring + s * slot_bytes);
                const int ks = kb + k;
                if (fp8_unit(k)) {  // as the producer
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {  // K = 32 e4m3 per MMA = 32 bytes
                        umma_e4m3(tmem, umma_desc_k_sw64(st + kk * 32), umma_desc_k_sw64(st + kATileBytes + kk * 32),
                                  idesc8, first ? 0u : 1u);
                        first = false;
                    }
                    umma_commit(&empty_bar[s]);
                    k += 2;
                    continue;
                }
                const int np = need(ks) ? 3 : 1;
                const uint32_t lp = (skipmode ? smem_u32(low) : st + kATileBytes + kPlaneTile) - kPlaneTile;
                for (int p = 0; p < np; ++p)
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t da = umma_desc_k_sw64(st + kk * 32);
                        const uint32_t pb = p == 0 ? st + kATileBytes : lp + p * kPlaneTile;
                        const uint64_t db = umma_desc_k_sw64(pb + kk * 32);
                        umma_bf16(tmem, da, db, idesc, first ? 0u : 1u);
                        first = false;
                    }
                umma_commit(&empty_bar[s]);  // slot free once these MMAs have read it
                if (skipmode && np == 3) umma_commit(&low_empty);
                k += 1;
            }
            umma_commit(&acc_bar);           // accumulator complete
        }
        __syncwarp();
    } else {
        // ---------------- epilogue (warps 2..): a warp may only touch TMEM lane quarter
        // warp % 4; with 8 epilogue warps two warps share a quarter and split the columns
        const int q = warp & 3;
        constexpr int parts = kEpiWarps / 4;
        const int part = (warp - 2) / 4;
        const int cbeg = part * (N / parts), cend = cbeg + N / parts;
        const int row = m0 + q * 32 + lane;
        // while the main loop runs, pull this warp's x / v lines (one 128-byte line per
        // column and array: 32 rows x fp32) into L2, so the epilogue's loads do not pay
        // DRAM latency one dependent round at a time
        if (a.k_split == 1 && m0 + q * 32 < a.n) {
            for (int c = cbeg + lane; c < cend && c < a.W; c += 32) {
                const int64_t o = static_cast<int64_t>(c) * a.ldx + m0 + q * 32;
                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a.X + o));
                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a.V + o));
            }
        }
        mbar_wait_sleep(&acc_bar, 0);
        tc_fence_after();
        const bool live = row < a.n;
        const float dg = live ? __ldg(a.deg + row) : 0.f;
        bool low_nz = false;  // any nonzero mid / lo plane entry in this warp's 32 nodes
#pragma unroll 1
        for (int c0 = cbeg; c0 < cend; c0 += 8) {
            uint32_t r[8];
            tmem_ld8(tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0), r);
            if (a.k_split > 1) {  // split-K piece: fp32 partial sums, coalesced along rows
                float* pp = a.partial + static_cast<int64_t>(blockIdx.x) * N * kBM + q * 32 + lane;
#pragma unroll
                for (int j = 0; j < 8; ++j) pp[static_cast<int64_t>(c0 + j) * kBM] = __uint_as_float(r[j]);
                continue;
            }
            if (c0 >= a.W) continue;
            if (a.cut_sum) {
                cut_chunk8(a, row, live, c0, r);
                continue;
            }
            if (!live) continue;
            low_nz |= finish_chunk8(a, row, c0, r, dg);
        }
        // one lane quarter = one 32-node K step of the next iteration's B operand; split-K
        // tail tiles: piece 0 clears the flag, k_dense_reduce ORs it in after the pieces
        if (a.kflags_out) {
            if (a.k_split == 1) {
                if (__any_sync(0xffffffffu, low_nz) && lane == 0) atomicOr(&qflag[q], 1u);
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                if (part == 0 && lane == 0 && m0 + q * 32 < a.n) a.kflags_out[(m0 >> 5) + q] = qflag[q];
            } else if (piece == 0 && part == 0 && lane == 0 && m0 + q * 32 < a.n) {
                a.kflags_out[(m0 >> 5) + q] = 0u;
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(N));
    }
}

// split-K tail: sum the pieces of each tail tile in a fixed order, then the fused step
template <int N>
__global__ void k_dense_reduce(DenseArgs a) {
    const int t = blockIdx.y;                         // tail tile index within this launch
    const int row_in = threadIdx.x;                   // 0..127
    const int row = (a.tile_base + t) * kBM + row_in;
    if (a.cut_sum) {  // cut mode (as cut_chunk8), the pieces summed in the same fixed order
        const bool live = row < a.n;
        for (int c = blockIdx.x; c < a.W; c += gridDim.x) {
            int d = 0;
            if (live) {
                float ax = 0.f;
                for (int p = 0; p < a.k_split; ++p)
                    ax += a.partial[(static_cast<int64_t>(t) * a.k_split + p) * N * kBM + static_cast<int64_t>(c) * kBM +
                                    row_in];
                d = __float2int_rn(ax);
                if (!(a.X[static_cast<int64_t>(c) * a.ldx + row] > 0.f)) d = -d;
            }
            d = __reduce_add_sync(0xffffffffu, d);
            if ((threadIdx.x & 31) == 0 && d)
                atomicAdd(a.cut_sum + c, static_cast<unsigned long long>(static_cast<long long>(d)));
        }
        return;
    }
    if (row >= a.n) return;
    const float dg = __ldg(a.deg + row);
    bool low_nz = false;
    for (int c = blockIdx.x; c < a.W; c += gridDim.x) {
        float ax = 0.f;
        for (int p = 0; p < a.k_split; ++p)
            ax += a.partial[(static_cast<int64_t>(t) * a.k_split + p) * N * kBM + static_cast<int64_t>(c) * kBM + row_in];
        low_nz |= finish_element(a, row, c, ax, dg);
    }
    if (a.kflags_out && low_nz) atomicOr(a.kflags_out + (row >> 5), 1u);
}

// fp32 [n][ld] (node-major) -> member-major [W][n] fp32 + three bf16 planes
__global__ void k_to_member_major(const float* __restrict__ X, int64_t ld, int n, int W, float* __restrict__ Xm,
                                  float* __restrict__ Vm, int ldx, __nv_bfloat16* __restrict__ P, int nks, int nb) {
    __shared__ float tile[32][33];
    const int v0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int v = v0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (v < n && c < W) ? X[static_cast<int64_t>(v) * ld + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, v = v0 + threadIdx.x;
        if (c < W && v < n) {
            const float x = tile[threadIdx.x][i];
            Xm[static_cast<int64_t>(c) * ldx + v] = x;
            Vm[static_cast<int64_t>(c) * ldx + v] = 0.f;
            __nv_bfloat16 h, m, l;
            split3(x, h, m, l);
            const int64_t po = plane_index(0, v, c, nks, nb), ps = static_cast<int64_t>(nks) * nb * 32;
            P[po] = h;
            P[ps + po] = m;
            P[2 * ps + po] = l;
        }
    }
}

// cut mode operands: the sign s = x > 0 ? +1 : -1 of the final iterate as the hi plane
// (mid / lo zero) and as its e4m3 copy (0x38 = +1, 0xb8 = -1)
__global__ void k_sign_planes(const float* __restrict__ Xm, int ldx, int n, int W, __nv_bfloat16* __restrict__ P,
                              int nks, int nb, uint8_t* __restrict__ P8) {
    const int64_t total = static_cast<int64_t>(W) * n;
    const int64_t ps = static_cast<int64_t>(nks) * nb * 32;
    const __nv_bfloat16 one = __float2bfloat16(1.f), mone = __float2bfloat16(-1.f), zero = __float2bfloat16(0.f);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i / n), v = static_cast<int>(i % n);
        const bool z = Xm[static_cast<int64_t>(c) * ldx + v] > 0.f;
        const int64_t po = plane_index(0, v, c, nks, nb);
        P[po] = z ? one : mone;
        P[ps + po] = zero;
        P[2 * ps + po] = zero;
        P8[plane8_index(v, c, nb)] = z ? 0x38 : 0xb8;
    }
}

__global__ void k_from_member_major(const float* __restrict__ Xm, int ldx, int n, int W, float* __restrict__ X,
                                    int64_t ld) {
    __shared__ float tile[32][33];
    const int v0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, v = v0 + threadIdx.x;
        tile[i][threadIdx.x] = (c < W && v < n) ? Xm[static_cast<int64_t>(c) * ldx + v] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int v = v0 + i, c = c0 + threadIdx.x;
        if (v < n && c < W) X[static_cast<int64_t>(v) * ld + c] = tile[threadIdx.x][i];
    }
}

// dense adjacency from CSR: A[v][u] = 1 for every stored neighbour, blocked, as bf16 (32-node
// K steps) and as e4m3 (64-node steps; 0x38 = 1.0)
__global__ void k_scatter_adjacency(const int* __restrict__ row_ptr, const int* __restrict__ col, int n,
                                    __nv_bfloat16* __restrict__ A, int nks, uint8_t* __restrict__ A8, int nks64) {
    const __nv_bfloat16 one = __float2bfloat16(1.f);
    for (int v = blockIdx.x; v < n; v += gridDim.x)
        for (int k = row_ptr[v] + threadIdx.x; k < row_ptr[v + 1]; k += blockDim.x) {
            A[adj_index(v, col[k], nks)] = one;
            A8[adj8_index(v, col[k], nks64)] = 0x38;
        }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}

void make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t pitch_elems,
              uint32_t box_inner, uint32_t box_rows, int elem_bytes = 2) {
    EncodeTiled enc = encode_fn();
    if (!enc) throw Failure{5, "cuTensorMapEncodeTiled unavailable"};
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {pitch_elems * static_cast<uint64_t>(elem_bytes)};
    const cuuint32_t box[2] = {box_inner, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    const CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Failure{4, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r))};
}

template <int N>
void launch_dense_n(const CUtensorMap& mA, const CUtensorMap& mP, DenseArgs a, float* partial, cudaStream_t s) {
    constexpr int full_ring = kStages * (kATileBytes + 3 * N * kBK * 2);
    constexpr int skip_ring = kSkipStages * (kATileBytes + N * kBK * 2) + 2 * N * kBK * 2;
    constexpr int smem = (full_ring > skip_ring ? full_ring : skip_ring) + 1024;
    ensure_smem_attr(reinterpret_cast<const void*>(k_dense_step<N>), smem, "cudaFuncSetAttribute(k_dense_step)");
    // Wave quantisation: full tiles fill whole waves of the SMs; the remaining tail tiles are
    // split along K so the tail also fills one wave, reduced in a fixed order afterwards.
    int dev = 0;
    cudaGetDevice(&dev);
    const char* sms_env = std::getenv("LCB_DENSE_SMS");  // test hook: pretend a smaller wave
    const int sms = sms_env ? std::atoi(sms_env) : num_sms(dev);
    const int tiles = (a.n + kBM - 1) / kBM;
    int tail = tiles % sms;
    if (tail * 2 > sms || tiles < sms || partial == nullptr) tail = 0;  // tail already fills >= half a wave
    const int full = tiles - tail;
    a.tile_base = 0;
    a.k_split = 1;
    a.partial = nullptr;
    // programmatic dependent launch (default on; LCB_DENSE_PDL=0 off): a launch's CTAs set
    // up (barriers, TMEM, tensor-map prefetch) while the previous launch drains
    // (config 3: 81.6 -> 80.4 ms per solve)
    static const bool pdl = [] {
        const char* e = std::getenv("LCB_DENSE_PDL");
        return !e || std::atoi(e) != 0;
    }();
    auto launch = [&](int grid, const DenseArgs& args) {
        count_launch();
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(kThreadsDense);
        cfg.dynamicSmemBytes = static_cast<size_t>(smem);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        cuda_check(cudaLaunchKernelEx(&cfg, k_dense_step<N>, mA, mP, args), "cudaLaunchKernelEx(k_dense_step)");
    };
    launch(full, a);
    if (tail > 0) {
        const int split = std::max(2, sms / tail);
        a.tile_base = full;
        a.k_split = split;
        a.partial = partial;
        launch(tail * split, a);
        count_launch();
        k_dense_reduce<N><<<dim3(std::min(a.W, 64), tail), kBM, 0, s>>>(a);
    }
}

}  // namespace

size_t dense_partial_floats() { return static_cast<size_t>(148 * 2) * 256 * kBM; }

int dense_nb(int W) { return W <= 64 ? 64 : (W <= 128 ? 128 : 256); }
int dense_nks(int n) { return (n + kBK - 1) / kBK; }

int dense_nks64(int n) { return (n + 63) / 64; }

// plane workspace: 2 x 3 blocked bf16 planes | 2 x K-step flags | 2 x e4m3 hi planes
size_t dense_flags_offset(int n, int W) {
    return sizeof(__nv_bfloat16) * 6 * static_cast<size_t>(dense_nks(n)) * dense_nb(W) * 32;
}
size_t dense_plane8_offset(int n, int W) {
    const size_t o = dense_flags_offset(n, W) + sizeof(uint32_t) * 2 * static_cast<size_t>(dense_nks(n));
    return (o + 127) & ~size_t(127);
}
size_t dense_planes_bytes(int n, int W) {
    return dense_plane8_offset(n, W) + 2 * static_cast<size_t>(dense_nks64(n)) * dense_nb(W) * 64 + 64;
}

// adjacency workspace: blocked bf16 [tiles][nks][128][32] | blocked e4m3 [tiles][nks64][128][64]
size_t dense_adjacency_bf16_bytes(int n) {
    const size_t tiles = static_cast<size_t>((n + kBM - 1) / kBM);
    return tiles * kBM * static_cast<size_t>(dense_nks(n)) * 32 * 2;
}
size_t dense_adjacency_bytes(int n) {
    const size_t tiles = static_cast<size_t>((n + kBM - 1) / kBM);
    return dense_adjacency_bf16_bytes(n) + tiles * kBM * static_cast<size_t>(dense_nks64(n)) * 64;
}

void build_dense_adjacency(const DevGraph& g, void* A, cudaStream_t s) {
    cuda_check(cudaMemsetAsync(A, 0, dense_adjacency_bytes(g.n), s), "memset(A)");
    count_launch();
    k_scatter_adjacency<<<std::min(g.n, 148 * 16), 256, 0, s>>>(
        g.row_ptr, g.col, g.n, static_cast<__nv_bfloat16*>(A), dense_nks(g.n),
        static_cast<uint8_t*>(A) + dense_adjacency_bf16_bytes(g.n), dense_nks64(g.n));
}

int dense_ldp(int n) { return (n + 7) / 8 * 8; }

// Dense T loop: X0 in node-major [n][ld] (from the batch init), result written back there.
void run_dense_iterations(const DevGraph& g, const void* A, const float* X_nodemajor_in, float* X_nodemajor_out,
                          int64_t ld, int W, int l, int64_t iters, float alpha_u, const float* alpha_arr,
                          const int* tlim_arr, float mu, unsigned long long* err, int err_seg, float* Xm, float* Vm,
                          void* planes, cudaStream_t s, int col_base, float* partial, unsigned long long* cut_sum) {
    const int n = g.n;
    const int ldx = dense_ldp(n);
    const int nks = dense_nks(n);
    // UMMA N (and the plane block height) = W rounded up to 64 / 128 / 256; the extra
    // columns of a block stay zero and their accumulator columns are never written back
    const int NB = dense_nb(W);
    const size_t plane3 = static_cast<size_t>(3) * nks * NB * 32;
    __nv_bfloat16* P = static_cast<__nv_bfloat16*>(planes);
    __nv_bfloat16* Pbuf[2] = {P, P + plane3};
    cuda_check(cudaMemsetAsync(P, 0, sizeof(__nv_bfloat16) * 2 * plane3, s), "memset(planes)");
    // K-step flags (after both plane buffers): the initial planes are never skipped
    uint32_t* F = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(planes) + dense_flags_offset(n, W));
    const int nks64 = dense_nks64(n);
    const size_t plane8 = static_cast<size_t>(nks64) * NB * 64;
    uint8_t* P8 = static_cast<uint8_t*>(planes) + dense_plane8_offset(n, W);
    uint8_t* P8buf[2] = {P8, P8 + plane8};
    cuda_check(cudaMemsetAsync(P8, 0, 2 * plane8, s), "memset(planes8)");
    static const bool fp8 = [] {
        const char* e = std::getenv("LCB_DENSE_FP8");
        return !e || std::atoi(e) != 0;
    }();
    uint32_t* Fbuf[2] = {F, F + nks};
    static const bool skip = [] {
        const char* e = std::getenv("LCB_DENSE_SKIP");
        return !e || std::atoi(e) != 0;
    }();
    cuda_check(cudaMemsetAsync(F, 1, sizeof(uint32_t) * static_cast<size_t>(nks), s), "memset(kflags)");
    const dim3 tg((n + 31) / 32, (W + 31) / 32);
    count_launch();
    k_to_member_major<<<tg, dim3(32, 8), 0, s>>>(X_nodemajor_in, ld, n, W, Xm, Vm, ldx, Pbuf[0], nks, NB);
    const uint64_t tiles = static_cast<uint64_t>((n + kBM - 1) / kBM);
    CUtensorMap mA, mP[2];
    make_map(&mA, A, kBK, tiles * static_cast<uint64_t>(nks) * kBM, kBK, kBK, kBM);
    for (int b = 0; b < 2; ++b)
        make_map(&mP[b], Pbuf[b], kBK, static_cast<uint64_t>(3) * nks * NB, kBK, kBK, static_cast<uint32_t>(NB));
    const uint8_t* A8 = static_cast<const uint8_t*>(A) + dense_adjacency_bf16_bytes(n);
    DenseArgs a{};
    a.deg = g.deg32;
    a.X = Xm;
    a.V = Vm;
    a.n = n;
    a.ldx = ldx;
    a.nks = nks;
    a.nks64 = nks64;
    a.nb = NB;
    a.W = W;
    a.l = l;
    a.mu = mu;
    a.alpha_uniform = alpha_u;
    a.alpha = alpha_arr;
    a.tlim = tlim_arr;
    a.err = err;
    a.err_seg = err_seg;
    a.col_base = col_base;
    for (int64_t it = 0; it < iters; ++it) {
        a.it = static_cast<int>(it);
        a.planes_out = Pbuf[(it + 1) & 1];
        a.kflags_in = skip ? Fbuf[it & 1] : nullptr;
        a.kflags_out = skip ? Fbuf[(it + 1) & 1] : nullptr;
        a.fp8 = skip && fp8 ? 1 : 0;
        a.plane8_out = a.fp8 ? P8buf[(it + 1) & 1] : nullptr;
        a.plane8_in = P8buf[it & 1];
        a.adj8 = A8;
        const CUtensorMap& mp = mP[it & 1];
        if (NB == 64)
            launch_dense_n<64>(mA, mp, a, partial, s);
        else if (NB == 128)
            launch_dense_n<128>(mA, mp, a, partial, s);
        else
            launch_dense_n<256>(mA, mp, a, partial, s);
    }
    if (cut_sum) {
        // the rounding's cut counts as one more tensor-core pass: (A s) for the sign planes
        // of the final iterate, every K step an e4m3 unit (s = +-1 exactly)
        const int b = static_cast<int>(iters & 1);
        count_launch();
        k_sign_planes<<<148 * 8, 256, 0, s>>>(Xm, ldx, n, W, Pbuf[b], nks, NB, P8buf[b]);
        cuda_check(cudaMemsetAsync(Fbuf[b], 0, sizeof(uint32_t) * static_cast<size_t>(nks), s), "memset(kflags)");
        cuda_check(cudaMemsetAsync(cut_sum, 0, sizeof(unsigned long long) * static_cast<size_t>(W), s), "memset(cut)");
        a.it = static_cast<int>(iters);
        a.planes_out = nullptr;
        a.plane8_out = nullptr;
        a.kflags_in = Fbuf[b];
        a.kflags_out = nullptr;
        a.fp8 = fp8 ? 1 : 0;
        a.plane8_in = P8buf[b];
        a.alpha = nullptr;
        a.tlim = nullptr;
        a.cut_sum = cut_sum;
        const CUtensorMap& mp = mP[b];
        if (NB == 64)
            launch_dense_n<64>(mA, mp, a, partial, s);
        else if (NB == 128)
            launch_dense_n<128>(mA, mp, a, partial, s);
        else
            launch_dense_n<256>(mA, mp, a, partial, s);
    }
    count_launch();
    k_from_member_major<<<tg, dim3(32, 8), 0, s>>>(Xm, ldx, n, W, X_nodemajor_out, ld);
    if (std::getenv("LCB_DENSE_STATS")) {
        std::vector<uint32_t> h(static_cast<size_t>(nks), 0);
        cudaMemcpyAsync(h.data(), Fbuf[iters & 1], sizeof(uint32_t) * nks, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        int z = 0;
        for (uint32_t c : h) z += c == 0;
        fprintf(stderr, "dense: %d of %d K steps skippable after %lld iterations\n", z, nks, static_cast<long long>(iters));
    }
}

}  // namespace lcb
