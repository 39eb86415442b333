// lcb_stream.cu — K1s: warp-specialised streaming PGA step for graphs whose iterate does
// not live on chip (config 4: ER n=1M, W=512 -> 2 GB per iterate buffer).
//
// One launch = one iteration of ascent.cpp:58-77 (Jacobi: every row reads the previous
// iterate of its neighbours) over the column slabs [slab0, slab0 + nslabs).  A slab is
// 1 KB of a row: 256 fp32 / 128 fp64 columns.  Work unit = a tile of R consecutive rows x
// one slab.  The runtime runs large batches slab-major (all iterations of one slab, then
// the next: members are independent, ascent.cpp:52), so the slab's saturation codes stay
// in L2 across iterations while the iterate itself streams from HBM once per iteration.
//
//   warp 0 (producer): per tile one 2D TMA box of x and one of v ([R][1 KB], L2
//           evict-first) and the tile's contiguous column run (bulk copy) into a ring of
//           stages, completion on an mbarrier; the row_ptr range of the tile P ahead
//           loads meanwhile.
//   warps 1..R (consumers): one row of the tile each.  Lane l owns 8 fp32 (4 fp64)
//           columns: the 16-byte groups l and 32+l of the slab (coalesced 512-byte
//           halves).  The neighbours' 32-byte code lines (one sign byte per lane) and
//           "row slab not saturated" flags of the NEXT tile's row are copied into the
//           warp's SMEM buffer with cp.async while this row is processed.
//
// Neighbour sums, in CSR order per element (graph.cpp:116-121):
//   * while every neighbour slab of a 32-neighbour batch is fully on the box corners (flag
//     0), every partial sum is a small integer, exact in fp32 and fp64: the +1 counts are
//     accumulated as SWAR bytes from the sign bits (sum = 2 * plus - count);
//   * from the first batch with an interior neighbour the warp continues with sequential
//     fp adds from that exact partial sum: +-1 from the sign bits for saturated
//     neighbours, the neighbour's 32 bytes of x otherwise.
// So fp64 stays bit-exact with the reference and fp32 equals the sequential fp32 sum.
// Epilogue: fused heavy-ball / finite check / clamp (ascent.cpp:66-73; the shared
// pga_raw op sequence, packed f32x2 FMAs), x' and v' written straight from registers
// (evict-first), plus the row's new sign bytes and slab flag.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "../../include/liftcut_b200.h"
#include "lcb_internal.h"

namespace lcb {

namespace {

#ifndef LCB_STREAM_R
#define LCB_STREAM_R 23
#endif
constexpr int kR = LCB_STREAM_R;  // rows per tile = consumer warps per CTA
constexpr int kThreadsS = 32 * (kR + 1);
#ifndef LCB_STREAM_MINB
#define LCB_STREAM_MINB 1  // resident CTAs per SM the register budget is sized for
#endif
#ifndef LCB_STREAM_STAGES
#define LCB_STREAM_STAGES 4
#endif
constexpr int kStages = LCB_STREAM_STAGES;
constexpr int kColBuf = 32 * kR;  // int32 column slots per stage
#ifndef LCB_STREAM_LOOK
#define LCB_STREAM_LOOK 4
#endif
constexpr int kLook = LCB_STREAM_LOOK;  // producer lookahead (tiles) for the CSR ranges
constexpr int kSlab = 1024;             // bytes of one row of a slab
#ifndef LCB_STREAM_FNB32
#define LCB_STREAM_FNB32 1
#endif
#ifndef LCB_STREAM_FNB64
#define LCB_STREAM_FNB64 2
#endif
// interior-neighbour gathers in flight per warp (fp mode, before saturation): one for fp32
// (the leaner code wins over the whole solve: config 4 1382 -> 1351 us/iteration, config 5
// 80.7 -> 78.2), two for fp64 (3151 vs 3247)
template <typename T>
struct Fnb {
    static constexpr int v = sizeof(T) == 4 ? LCB_STREAM_FNB32 : LCB_STREAM_FNB64;
};
#ifndef LCB_STREAM_D
#define LCB_STREAM_D 1
#endif
// tiles whose neighbour code lines are in flight ahead of the one being summed: the code
// gathers are L2 round trips, so one tile of lookahead left the steady state latency-bound
constexpr int kD = LCB_STREAM_D;
constexpr int kCB = kD + 2;             // code buffers per warp: kD + 1 tiles + the hub chunk
static_assert(kD < kStages, "code lookahead needs the tiles' stages");

template <typename T>
struct Lanes {
    static constexpr int E = kSlab / 32 / static_cast<int>(sizeof(T));  // elements per lane
    static constexpr int H = E / 2;                                     // per 16-byte half
    static constexpr int SPAN = 32 * E;                                 // columns per slab
};

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
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) { mbar_arrive(smem_u32(bar)); }
// the suspend-time hint parks a waiting warp in the barrier unit instead of re-issuing the probe
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) { mbar_wait(smem_u32(bar), parity); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// 2D tensor tile (TMA): box [R rows][1 KB] of X / V at (column c0, row r0); rows past n are
// zero-filled and still counted in the transaction bytes
__device__ __forceinline__ void tma_tile(void* dst, const CUtensorMap* map, int c0, int r0, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_n() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 16-byte vectors of a lane's half-slab
__device__ __forceinline__ void ld16(float* v, const void* smem) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                 : "r"(smem_u32(smem)));
}
__device__ __forceinline__ void ld16(float* v, uint32_t a) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
}
__device__ __forceinline__ void ld16(double* v, uint32_t a) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a));
}
__device__ __forceinline__ void ld16(double* v, const void* smem) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(smem_u32(smem)));
}
__device__ __forceinline__ void ldg16(float* v, const float* p) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x;
    v[1] = q.y;
    v[2] = q.z;
    v[3] = q.w;
}
__device__ __forceinline__ void ldg16(double* v, const double* p) {
    const double2 q = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = q.x;
    v[1] = q.y;
}
// streaming (evict-first) 16-byte loads of data read once
__device__ __forceinline__ void ldcs16(float* v, const float* p) {
    const float4 q = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = q.x;
    v[1] = q.y;
    v[2] = q.z;
    v[3] = q.w;
}
__device__ __forceinline__ void ldcs16(double* v, const double* p) {
    const double2 q = __ldcs(reinterpret_cast<const double2*>(p));
    v[0] = q.x;
    v[1] = q.y;
}
__device__ __forceinline__ void stg16(float* p, const float* v) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
}
__device__ __forceinline__ void stg16(double* p, const double* v) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
}

__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }

// packed fp32x2 FMA (FFMA2): round-to-nearest per lane, identical to two __fmaf_rn
__device__ __forceinline__ void fma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0,
                                     float c1) {
    unsigned long long r;
    const unsigned long long A = (static_cast<unsigned long long>(__float_as_uint(a1)) << 32) | __float_as_uint(a0);
    const unsigned long long B = (static_cast<unsigned long long>(__float_as_uint(b1)) << 32) | __float_as_uint(b0);
    const unsigned long long Cc = (static_cast<unsigned long long>(__float_as_uint(c1)) << 32) | __float_as_uint(c0);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(A), "l"(B), "l"(Cc));
    d0 = __uint_as_float(static_cast<unsigned>(r));
    d1 = __uint_as_float(static_cast<unsigned>(r >> 32));
}
// the pga_raw sequence (lcb_internal.h) for two elements at once: fp32 packed, fp64 scalar
__device__ __forceinline__ void pga_raw2(const float* x, const float* ax, float* v, float alpha, float mu, float dg,
                                         float* raw) {
    float y0, y1;
    fma2(y0, y1, dg, dg, x[0], x[1], -ax[0], -ax[1]);
    fma2(v[0], v[1], mu, mu, v[0], v[1], y0, y1);
    fma2(raw[0], raw[1], alpha, alpha, v[0], v[1], x[0], x[1]);
}
__device__ __forceinline__ void pga_raw2(const double* x, const double* ax, double* v, double alpha, double mu,
                                         double dg, double* raw) {
    raw[0] = pga_raw(x[0], ax[0], v[0], alpha, mu, dg);
    raw[1] = pga_raw(x[1], ax[1], v[1], alpha, mu, dg);
}
// the same with the neighbour sum passed negated (nax = -Ax, exact): y = fma(dg, x, nax)
__device__ __forceinline__ void pga_raw_neg2(const float* x, const float* nax, float* v, float alpha, float mu,
                                             float dg, float* raw) {
    float y0, y1;
    fma2(y0, y1, dg, dg, x[0], x[1], nax[0], nax[1]);
    fma2(v[0], v[1], mu, mu, v[0], v[1], y0, y1);
    fma2(raw[0], raw[1], alpha, alpha, v[0], v[1], x[0], x[1]);
}
__device__ __forceinline__ void pga_raw_neg2(const double* x, const double* nax, double* v, double alpha, double mu,
                                             double dg, double* raw) {
    raw[0] = pga_raw(x[0], -nax[0], v[0], alpha, mu, dg);
    raw[1] = pga_raw(x[1], -nax[1], v[1], alpha, mu, dg);
}

#ifndef LCB_STREAM_CLAIM
#define LCB_STREAM_CLAIM 1
#endif
constexpr int kClaim = LCB_STREAM_CLAIM;  // tiles per dynamic claim
#ifndef LCB_STREAM_ILV
#define LCB_STREAM_ILV 1
#endif
constexpr bool kInterleave = LCB_STREAM_ILV != 0;  // tile order: slab-interleaved (1) or slab-major (0)
#ifndef LCB_STREAM_STATIC
#define LCB_STREAM_STATIC 0
#endif
#ifndef LCB_STREAM_EXP
#define LCB_STREAM_EXP 0  // timing experiments only (wrong results): 1 consumers idle, 2 no v box
#endif
#ifndef LCB_STREAM_XBOX
#define LCB_STREAM_XBOX 0
#endif
// 1: the producer stages the tile's x box when every row needs its stored x; 0: consumers
// always load their own stored x (the SMEM goes to deeper v staging)
constexpr bool kXBox = LCB_STREAM_XBOX != 0;

__device__ __forceinline__ uint32_t sign_bit(float v) { return __float_as_uint(v) >> 31; }
__device__ __forceinline__ uint32_t sign_bit(double v) {
    return static_cast<uint32_t>(static_cast<unsigned long long>(__double_as_longlong(v)) >> 63);
}

// every one of the E values finite: the products with zero are +-0 exactly then, NaN otherwise
__device__ __forceinline__ bool finite_all(const float* r) {
    float z0 = 0.f, z1 = 0.f;
#pragma unroll
    for (int e = 0; e < 8; e += 2) fma2(z0, z1, r[e], r[e + 1], 0.f, 0.f, z0, z1);
    return z0 + z1 == 0.f;
}
__device__ __forceinline__ bool finite_all(const double* r) {
    double z = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) z = fma(r[e], 0.0, z);
    return z == 0.0;
}

struct StreamSmem {
    alignas(128) unsigned char x[kXBox ? kStages : 1][kXBox ? kR : 1][kXBox ? kSlab : 128];
    alignas(128) unsigned char v[kStages][kR][kSlab];
    int col[kStages][kColBuf];
    int row[kStages][kR];
    int beg[kStages][kR];
    int deg[kStages][kR];
    int coff[kStages][kR];
    int xfl[kStages][kR];            // x-code mode: 0 = the row slab's x is its sign code
    int xbox[kStages];               // 1: the stage holds the tile's x box
    int slab[kStages];               // launch-relative slab of the tile in the stage
    // per consumer warp: code lines of <= 32 neighbours (this row, the rows of the next kD
    // tiles, and one more buffer that double-buffers the further 32-neighbour chunks of hub rows)
    alignas(16) uint8_t codes[kR][kCB][32][32];
    uint32_t flags[kR][kCB][32];     // and their "slab not saturated" flags
    alignas(16) uint8_t own[kR][kD + 1][32];  // x-code mode: the row's own code line
    uint64_t full[kStages];
    uint64_t empty[kStages];
};

template <typename T, bool GEN, bool EE, int FNB>
__global__ void __launch_bounds__(kThreadsS, LCB_STREAM_MINB)
    k_stream(StepArgs<T> a, int rowtiles, int slab0, int nslabs, const __grid_constant__ CUtensorMap mx,
             const __grid_constant__ CUtensorMap mv) {
    constexpr int E = Lanes<T>::E, H = Lanes<T>::H, SPAN = Lanes<T>::SPAN;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    StreamSmem& sm = *reinterpret_cast<StreamSmem*>(smem_raw);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ntiles = rowtiles * nslabs;
    const uint32_t n32 = static_cast<uint32_t>(a.n);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kR);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mx)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mv)) : "memory");
    }
    // Programmatic dependent launch: everything above overlaps the previous iteration's tail;
    // nothing the previous launch writes (iterate, codes, flags, counters) is touched before
    // this wait for its completion.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if constexpr (EE) {
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < a.members; i += blockDim.x) a.flags_zero[i] = 0;
    }
    // the tile counter of the NEXT launch (this launch uses tile_ctr[seq & 1], zeroed by the
    // previous one)
    if (blockIdx.x == 0 && threadIdx.x == 0) a.tile_ctr[(a.launch_seq + 1) & 1] = 0u;
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer.  Tiles are claimed dynamically from a launch-wide counter
        // (BA hubs make tiles uneven: a static split left config 5 at 62 % SM activity), P
        // claims ahead, so the row_ptr loads of a claimed tile leave the critical path.  After
        // the last tile a sentinel stage (slab = -1) tells the consumers to stop.
        const uint64_t pol = policy_evict_first();
        // claims in flight: 2 for fp32 (config 5 78.3 -> 76.1 us/iteration), 4 for fp64 (3151 vs 3329)
        constexpr int P = sizeof(T) == 4 ? (kLook < 2 ? kLook : 2) : kLook;
        // tile t -> (slab, first row): slab-interleaved, so the hub rows at the front of every
        // slab (BA graphs) are claimed first and the CTAs holding them catch up on the rest
        auto tile_slab = [&](int t) { return kInterleave ? t % nslabs : t / rowtiles; };
        auto tile_row0 = [&](int t) { return (kInterleave ? t / nslabs : t - (t / rowtiles) * rowtiles) * kR; };
        // per claim: lane j <= R: row_ptr[min(r0 + j, n)]; the tile index; lane j < R: the
        // flag of row r0 + j's slab in the input codes (x-code mode; 0 = x is in the code)
        int qrp[P], qt[P], qfl[P];
        unsigned* ctr = a.tile_ctr + (a.launch_seq & 1);
        const uint32_t* const pfin =
            (a.xskip && a.sgn_in) ? reinterpret_cast<const uint32_t*>(a.sgn_in + a.flag_off) : nullptr;
        // tiles are claimed kClaim at a time (one atomic per kClaim tiles: same-address
        // atomics from every SM serialise in one L2 slice)
        int cbase = 0, cleft = 0;  // lane 0's current claim: next tile, tiles left in it
        int sidx = 0;              // static experiment: this CTA's next tile
        auto claim = [&](int& t, int& fl) {
            int v = 0;
#if LCB_STREAM_STATIC
            v = static_cast<int>(blockIdx.x) + sidx * static_cast<int>(gridDim.x);
            ++sidx;
#else
            if (lane == 0) {
                if (cleft == 0) {
                    cbase = static_cast<int>(atomicAdd(ctr, static_cast<unsigned>(kClaim)));
                    cleft = kClaim;
                }
                v = cbase++;
                --cleft;
            }
#endif
            t = __shfl_sync(0xffffffffu, v, 0);
            int rp = 0;
            fl = 1;
            if (t < ntiles && lane <= kR) {
                int sl = tile_slab(t);
                const int row = tile_row0(t) + lane;
                rp = __ldg(a.row_ptr + min(row, a.n));
                if (pfin && lane < kR) {
                    if (a.it & 1) sl = nslabs - 1 - sl;
                    fl = row < a.n ? static_cast<int>(__ldcg(pfin + static_cast<uint32_t>(sl) * n32 + row)) : 0;
                }
            }
            return rp;
        };
#pragma unroll
        for (int q = 0; q < P; ++q) qrp[q] = claim(qt[q], qfl[q]);
        for (int i0 = 0;; i0 += P) {
            bool done = false;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int i = i0 + q;
                const int s = i % kStages;
                if (i >= kStages) mbar_wait(&sm.empty[s], ((i / kStages) & 1) ^ 1);
                const int t = qt[q];
                if (t >= ntiles) {  // sentinel stage: no copies, a plain arrival
                    if (lane == 0) {
                        sm.slab[s] = -1;
                        mbar_arrive(&sm.full[s]);
                        // this CTA claims no more tiles: the next launch may start its prologue
                        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
                    }
                    done = true;
                    break;
                }
                const int beg = qrp[q];
                const int fl = qfl[q];
                qrp[q] = claim(qt[q], qfl[q]);
                const int end = __shfl_down_sync(0xffffffffu, beg, 1);
                const int first = __shfl_sync(0xffffffffu, beg, 0), last = __shfl_sync(0xffffffffu, beg, kR);
                int sl = tile_slab(t);
                const int r0 = tile_row0(t);
                if (a.it & 1) sl = nslabs - 1 - sl;  // snake: reuse the slab just written
                const int abeg = first & ~3;
                const int ncopy = min(((last + 3) & ~3) - abeg, kColBuf);  // staged prefix of the tile's run
                if (lane == 0) sm.slab[s] = sl;
                if (lane < kR) {
                    const int row = r0 + lane;
                    const bool ok = row < a.n;
                    sm.row[s][lane] = ok ? row : -1;
                    sm.beg[s][lane] = beg;
                    sm.deg[s][lane] = ok ? end - beg : 0;
                    sm.coff[s][lane] = (ok && end - abeg <= ncopy) ? beg - abeg : -1;
                    sm.xfl[s][lane] = fl;
                }
                // the x box only when every row slab of the tile needs its stored x; otherwise the
                // rows whose x is not in the codes load it themselves (consumer ldg)
                const bool skipx = !kXBox || !__all_sync(0xffffffffu, lane >= kR || fl != 0);
                if (lane == 0) sm.xbox[s] = skipx ? 0 : 1;
                __syncwarp();
                if (lane == 0) {
#if LCB_STREAM_EXP == 2  // timing experiment: no v box
                    mbar_expect_tx(&sm.full[s], (skipx ? 0u : 1u) * kR * kSlab + static_cast<uint32_t>(ncopy) * 4u);
#else
                    mbar_expect_tx(&sm.full[s], (skipx ? 1u : 2u) * kR * kSlab + static_cast<uint32_t>(ncopy) * 4u);
#endif
                    if (kXBox && !skipx) tma_tile(&sm.x[kXBox ? s : 0][0][0], &mx, (slab0 + sl) * SPAN, r0, &sm.full[s], pol);
#if LCB_STREAM_EXP != 2
                    tma_tile(&sm.v[s][0][0], &mv, (slab0 + sl) * SPAN, r0, &sm.full[s], pol);
#endif
                    if (ncopy > 0)
                        bulk_g2s(&sm.col[s][0], a.col + abeg, static_cast<uint32_t>(ncopy) * 4u, &sm.full[s], pol);
                }
            }
            if (done) break;
        }
        return;
    }

    // ---------------- consumers: warp w owns row w-1 of every tile
    const int j = warp - 1;
    // lane element e: half e / H (16-byte group lane or 32 + lane of the slab), position e % H
    auto col_of = [&](int slab, int e) { return slab * SPAN + (e / H) * (SPAN / 2) + lane * H + (e % H); };
    auto member_of = [&](int slab, int e) { return (a.col_base + col_of(slab, e)) / a.l; };
    int cur_slab = -1;
    uint32_t act_bits = 0;  // which elements step at this iteration (bit e)
    uint32_t valid_bits = 0;  // which elements are batch columns (not padding past W)
    bool all_act = false;
    uint32_t ebits = 0;     // 3 exit bits per element (EE)
    auto flush_bits = [&]() {
        if constexpr (EE) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const uint32_t b = (ebits >> (3 * e)) & 7u;
                if (b) {
                    const int m = member_of(cur_slab, e);
                    const uint32_t f = __ldcg(a.flags_cur + m);
                    if ((f & b) != b) atomicOr(a.flags_cur + m, b);
                }
            }
            ebits = 0;
        }
    };
    auto enter_slab = [&](int slab) {
        if (cur_slab >= 0) flush_bits();
        cur_slab = slab;
        act_bits = 0;
        valid_bits = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            bool act = col_of(slab, e) < a.W;
            valid_bits |= act ? 1u << e : 0u;
            if constexpr (GEN) {
                if (act) {
                    const int m = member_of(slab, e);
                    if (a.tlim) act = a.it < __ldg(a.tlim + m);
                    if constexpr (EE) {
                        if (act && a.it > 0) act = ex_continue(__ldcg(a.flags_prev + m));
                    }
                }
            }
            act_bits |= act ? 1u << e : 0u;
        }
        all_act = __all_sync(0xffffffffu, act_bits == (1u << E) - 1u);
    };
    const uint8_t* const cin = a.sgn_in;  // codes [slabs][n][32], flags [slabs][n] at flag_off
    const uint32_t* const fin = cin ? reinterpret_cast<const uint32_t*>(cin + a.flag_off) : nullptr;
    uint8_t* const cout = a.sgn_out;
    uint32_t* const fout = cout ? reinterpret_cast<uint32_t*>(cout + a.flag_off) : nullptr;

    // 32-bit shared addresses of this warp's / lane's slots (buffer / stage offsets added per use)
    const uint32_t sb = smem_u32(smem_raw);
    const uint32_t a_codes = sb + static_cast<uint32_t>(offsetof(StreamSmem, codes)) + (j * kCB * 32 + lane) * 32u;
    const uint32_t a_flags = sb + static_cast<uint32_t>(offsetof(StreamSmem, flags)) + (j * kCB * 32 + lane) * 4u;
    const uint32_t a_own = sb + static_cast<uint32_t>(offsetof(StreamSmem, own)) + j * (kD + 1) * 32 + 4 * (lane & 7);
    const uint32_t a_v = sb + static_cast<uint32_t>(offsetof(StreamSmem, v)) + j * kSlab + 16 * lane;
    const uint32_t a_x = sb + static_cast<uint32_t>(offsetof(StreamSmem, x)) + j * kSlab + 16 * lane;
    const uint32_t a_full = sb + static_cast<uint32_t>(offsetof(StreamSmem, full));
    const uint32_t a_empty = sb + static_cast<uint32_t>(offsetof(StreamSmem, empty));

    // code lines + flags of neighbours [k0, k0 + 32) of the row in stage st -> buffer buf
    auto stage_codes = [&](int st, int sl, int buf, int k0) {
        const int row = sm.row[st][j];
        if (row >= 0 && cin) {
            const int deg = sm.deg[st][j];
            const int k = k0 + lane;
            if (k < deg) {
                const int coff = sm.coff[st][j];
                const int u = coff >= 0 ? sm.col[st][coff + k] : __ldg(a.col + sm.beg[st][j] + k);
                const uint32_t line = static_cast<uint32_t>(sl) * n32 + static_cast<uint32_t>(u);
                const uint32_t dc = a_codes + static_cast<uint32_t>(buf) * 1024u;
                cp_async16(dc, cin + line * 32u);
                cp_async16(dc + 16u, cin + line * 32u + 16u);
                cp_async4(a_flags + static_cast<uint32_t>(buf) * 128u, fin + line);
            } else if (k0 == 0 && k < deg + 2 && deg <= 30) {  // zero lines up to a multiple of 3 (fast path)
                const uint32_t dc = a_codes + static_cast<uint32_t>(buf) * 1024u;
                asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dc), "r"(0u) : "memory");
                asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dc + 16u), "r"(0u) : "memory");
            }
            if (k0 == 0 && lane >= 24 && a.xskip && sm.xfl[st][j] == 0) {  // own line, 4 bytes per lane
                const uint32_t line = static_cast<uint32_t>(sl) * n32 + static_cast<uint32_t>(row);
                cp_async4(a_own + static_cast<uint32_t>(buf) * 32u, cin + line * 32u + 4u * (lane - 24));
            }
        }
        cp_async_commit();
    };

    // tiles i .. i + kD have their code lines in flight (one cp.async group per tile; an empty
    // group past the end); have[d]: tile i + d exists (slab -1: the producer's sentinel)
    bool have[kD + 1];
#pragma unroll
    for (int d = 0; d <= kD; ++d) have[d] = false;
    mbar_wait(&sm.full[0], 0);
    have[0] = sm.slab[0] >= 0;
    if (have[0]) stage_codes(0, sm.slab[0], 0, 0);
#pragma unroll
    for (int d = 1; d < kD; ++d) {
        if (have[d - 1]) {
            mbar_wait(&sm.full[d % kStages], (d / kStages) & 1);
            have[d] = sm.slab[d % kStages] >= 0;
        }
        if (have[d])
            stage_codes(d % kStages, sm.slab[d % kStages], d, 0);
        else
            cp_async_commit();
    }
    for (int i = 0; have[0]; ++i) {
        const int s = i % kStages;
        const int sl = sm.slab[s];
        const int slab = slab0 + sl;
        if (slab != cur_slab) enter_slab(slab);
        have[kD] = false;
        if (have[kD - 1]) {  // tile i + kD's stage has normally landed (the producer runs ahead)
            const int sn = (i + kD) % kStages;
            mbar_wait(a_full + 8u * static_cast<uint32_t>(sn), ((i + kD) / kStages) & 1);
            have[kD] = sm.slab[sn] >= 0;
        }
        if (have[kD])
            stage_codes((i + kD) % kStages, sm.slab[(i + kD) % kStages], (i + kD) % (kD + 1), 0);
        else
            cp_async_commit();
        cp_async_wait_n<kD>();  // this tile's code lines have landed
        __syncwarp();
        const int row = sm.row[s][j];
        if (row >= 0 && LCB_STREAM_EXP != 1) {
            const int deg = sm.deg[s][j];
            const int coff = sm.coff[s][j];
            // x-code mode: this row slab was not stored last iteration, its x is the sign code
            const bool own_code = a.xskip && cin && sm.xfl[s][j] == 0;
            const int buf = i % (kD + 1);
            const uint32_t own_bits = own_code ? sm.own[j][buf][lane] : 0u;
            // stored x outside a loaded box: issued now, consumed by the epilogue
            const bool own_ld = !own_code && sm.xbox[s] == 0;
            T xg[E];
            if (own_ld) {
                const T* p = a.x_in + static_cast<int64_t>(row) * a.ld + col_of(slab, 0);
                ldcs16(&xg[0], p);
                ldcs16(&xg[H], p + SPAN / 2);
            }
            T nacc[E];
            // Fast path (the saturated steady state): <= 32 neighbours, all on the box corners.
            // Sign bytes are compressed three at a time (full adder: parity = weight 1,
            // majority = weight 2) before the nibble spread into byte counters.
            bool fast = false;
            if (cin != nullptr && deg <= 32) {
                const uint32_t* fb0 = &sm.flags[j][buf][0];
                fast = !__any_sync(0xffffffffu, lane < deg && fb0[lane] != 0u);
            }
            if (fast) {
                const uint8_t* cb = &sm.codes[j][buf][0][lane];
                auto spread = [](uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; };
                uint32_t q0 = 0, q1 = 0;  // +1 counts: byte e of q0 = element e, of q1 = element 4 + e
                // the staged lines past the degree are zero (stage_codes pads up to a multiple of
                // 3 when that fits the 32 slots): zero signs count no +1
                const int kfull = deg <= 30 ? deg : deg - deg % 3;
                int k = 0;
                for (; k < kfull; k += 3) {
                    const uint32_t b0 = cb[32 * k], b1 = cb[32 * (k + 1)], b2 = cb[32 * (k + 2)];
                    const uint32_t par = b0 ^ b1 ^ b2;
                    const uint32_t maj = (b0 & b1) | (b2 & (b0 | b1));
                    q0 += spread(par & 0xFu) + 2u * spread(maj & 0xFu);
                    if constexpr (E == 8) q1 += spread(par >> 4) + 2u * spread(maj >> 4);
                }
                for (; k < deg; ++k) {
                    const uint32_t b = cb[32 * k];
                    q0 += spread(b & 0xFu);
                    if constexpr (E == 8) q1 += spread(b >> 4);
                }
                if constexpr (sizeof(T) == 4) {
                    // fp32: the doubled count byte (2c <= 64) as the low mantissa byte of 2^22
                    // (0x4A8000xx = 2^22 + c, exact), then deg - 2c = fma(-2, 2^22 + c, deg + 2^23)
                    // exactly (deg + 2^23 is representable, the fma rounds once an exact
                    // integer).  Only a zero sum differs from the sequential -(+0.0) (+0.0
                    // here), and only for isolated rows, where y = 0 * x + (+-0) leaves v = +0
                    // and x unchanged either way.
                    const float dbias = static_cast<float>(deg) + 8388608.f;
                    const uint32_t d0 = q0 << 1, d1 = q1 << 1;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const uint32_t cf = __byte_perm(e < 4 ? d0 : d1, 0x4A800000u, 0x7640u + static_cast<uint32_t>(e & 3));
                        nacc[e] = __fmaf_rn(-2.f, __uint_as_float(cf), dbias);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const uint32_t c = __byte_perm(e < 4 ? q0 : q1, 0u, 0x4440u + static_cast<uint32_t>(e & 3));
                        nacc[e] = -static_cast<T>(2 * static_cast<int>(c) - deg);
                    }
                }
            } else {
                int cur = buf;  // buffer holding the current 32-neighbour chunk
                const T* xin0 = a.x_in + col_of(slab, 0);
                const T* xin1 = xin0 + SPAN / 2;
                // integer mode: SWAR byte counters of +1 signs, p0 elements 0..3, p1 elements 4..7
                // (<= 224 neighbours per fold; hub rows fold into wide counters)
                uint32_t p0 = 0, p1 = 0, wide[E];
                int folded = 0, in_bytes = 0;
                bool wide_used = false;
                bool fmode = cin == nullptr;
                T acc[E];  // fp mode: the running sum
#pragma unroll
                for (int e = 0; e < E; ++e) acc[e] = T(0);
                auto unpack = [&](int e) -> uint32_t {
                    return __byte_perm(e < 4 ? p0 : p1, 0u, 0x4440u + static_cast<uint32_t>(e & 3));
                };
                for (int base = 0; base < deg; base += 32) {
                    const int cnt = min(32, deg - base);
                    int nxt = cur;
                    if (cin && base + 32 < deg) {  // hub rows: stage the next chunk while this one is summed
                        nxt = cur == kD + 1 ? buf : kD + 1;
                        __syncwarp();  // every lane is done with buffer nxt (the chunk before this one)
                        stage_codes(s, sl, nxt, base + 32);
                        // chunk 0 landed with the tile's group; later chunks: everything but the copy
                        // just issued (the lookahead tiles' groups are older and complete with it)
                        if (base > 0) cp_async_wait1();
                        __syncwarp();
                    } else if (cin && base > 0) {
                        cp_async_wait0();
                        __syncwarp();
                    }
                    const uint8_t* cb = &sm.codes[j][cur][0][lane];  // neighbour k's sign byte for this lane: cb[32 k]
                    const uint32_t* fb = &sm.flags[j][cur][0];
                    cur = nxt;
                    if (!fmode) {
                        const bool interior = __any_sync(0xffffffffu, lane < cnt && fb[lane] != 0u);
                        if (!interior) {
#pragma unroll 4
                            for (int k = 0; k < cnt; ++k) {
                                const uint32_t b = cb[32 * k];
                                p0 += ((b & 0xFu) * 0x00204081u) & 0x01010101u;  // sign bit e -> byte e
                                if constexpr (E == 8) p1 += ((b >> 4) * 0x00204081u) & 0x01010101u;
                            }
                            folded += cnt;
                            in_bytes += cnt;
                            if (in_bytes > 224) {  // hub rows: keep the byte counters from overflowing
                                if (!wide_used) {
#pragma unroll
                                    for (int e = 0; e < E; ++e) wide[e] = 0;
                                    wide_used = true;
                                }
#pragma unroll
                                for (int e = 0; e < E; ++e) wide[e] += unpack(e);
                                p0 = p1 = 0;
                                in_bytes = 0;
                            }
                            continue;
                        }
                        fmode = true;  // exact partial sum so far: (+1 count) - (-1 count)
#pragma unroll
                        for (int e = 0; e < E; ++e)
                            acc[e] = static_cast<T>(2 * static_cast<int>(unpack(e) + (wide_used ? wide[e] : 0u)) - folded);
                    }
                    // sequential fp adds; the neighbour index is only needed for interior neighbours
                    constexpr int kFNB = FNB;
                    for (int k = 0; k < cnt; k += kFNB) {
                        T g[kFNB][E];
                        uint32_t bq[kFNB];
                        bool in[kFNB];
#pragma unroll
                        for (int q = 0; q < kFNB; ++q) {
                            const int kk = k + q;
                            const bool live = kk < cnt;
                            in[q] = live && (cin == nullptr || fb[kk] != 0u);  // warp-uniform
                            bq[q] = (live && cin) ? cb[32 * kk] : 0u;
                            if (in[q]) {
                                const int u =
                                    coff >= 0 ? sm.col[s][coff + base + kk] : __ldg(a.col + sm.beg[s][j] + base + kk);
                                const int64_t o = static_cast<int64_t>(u) * a.ld;
                                ldg16(&g[q][0], xin0 + o);
                                ldg16(&g[q][H], xin1 + o);
                            }
                        }
                        bool all_in = true;
#pragma unroll
                        for (int q = 0; q < kFNB; ++q) all_in = all_in && (in[q] || k + q >= cnt);
                        if (all_in) {  // before saturation: every neighbour gathered, plain adds
#pragma unroll
                            for (int q = 0; q < kFNB; ++q)
                                if (k + q < cnt)
#pragma unroll
                                    for (int e = 0; e < E; ++e) acc[e] = radd(acc[e], g[q][e]);
                            continue;
                        }
#pragma unroll
                        for (int q = 0; q < kFNB; ++q) {
                            if (k + q < cnt) {
#pragma unroll
                                for (int e = 0; e < E; ++e)
                                    acc[e] = radd(acc[e], in[q] ? g[q][e] : (((bq[q] >> e) & 1u) ? T(1) : T(-1)));
                            }
                        }
                    }
                }
                // -acc, exact: -((count of +1) - (count of -1)); negated after the conversion so a zero
                // sum is -0.0 exactly as -(+0.0) of the sequential sum
                if (!fmode) {
#pragma unroll
                    for (int e = 0; e < E; ++e)
                        nacc[e] = -static_cast<T>(2 * static_cast<int>(unpack(e) + (wide_used ? wide[e] : 0u)) - folded);
                } else {
#pragma unroll
                    for (int e = 0; e < E; ++e) nacc[e] = -acc[e];
                }
            }

            // ---- epilogue (ascent.cpp:66-77)
            T xv[E], vv[E];
            if (own_code) {  // x on the box corners, exactly: +-1 from the sign bits
#pragma unroll
                for (int e = 0; e < E; ++e) xv[e] = ((own_bits >> e) & 1u) ? T(1) : T(-1);
            } else if (own_ld) {
#pragma unroll
                for (int e = 0; e < E; ++e) xv[e] = xg[e];
            } else if constexpr (kXBox) {
                ld16(&xv[0], a_x + static_cast<uint32_t>(s) * (kR * kSlab));
                ld16(&xv[H], a_x + static_cast<uint32_t>(s) * (kR * kSlab) + 512u);
            }
            ld16(&vv[0], a_v + static_cast<uint32_t>(s) * (kR * kSlab));
            ld16(&vv[H], a_v + static_cast<uint32_t>(s) * (kR * kSlab) + 512u);
            const T dg = static_cast<T>(deg);
            T raw[E], xo[E];
            uint32_t bad = 0, sign = 0;
            bool interior = false;
            if (all_act && !(GEN && a.alpha)) {
                // every element steps with the uniform alpha (the steady state)
#pragma unroll
                for (int e = 0; e < E; e += 2) pga_raw_neg2(&xv[e], &nacc[e], &vv[e], a.alpha_uniform, a.mu, dg, &raw[e]);
                // finite check (ascent.cpp:70-72) folded: sum of raw * 0 is NaN iff some raw is not
                // finite; the per-element mask only then
                if (!finite_all(raw)) {
#pragma unroll
                    for (int e = 0; e < E; ++e) bad |= isfinite(raw[e]) ? 0u : 1u << e;
                }
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    xo[e] = fmin(fmax(raw[e], T(-1)), T(1));                 // ascent.cpp:73 (raw finite)
                    if constexpr (EE) {
                        const T ch = fabs(xo[e] - xv[e]);
                        uint32_t b = 0;
                        if (ch > T(1e-12)) b |= EX_BIG;
                        if (ch > T(0)) b |= EX_NZ;
                        if (xo[e] != T(1) && xo[e] != T(-1)) b |= EX_NOTB;
                        ebits |= b << (3 * e);
                    }
                    interior |= fabs(xo[e]) != T(1);
                }
                if (!interior) {  // all +-1: the sign bit alone decides x > 0
#pragma unroll
                    for (int e = 0; e < E; ++e) sign |= (sign_bit(xo[e]) ^ 1u) << e;
                } else {
#pragma unroll
                    for (int e = 0; e < E; ++e) sign |= (xo[e] > T(0) ? 1u : 0u) << e;
                }
            } else {
                T vn[E];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    vn[e] = vv[e];
                    const T alpha = (GEN && a.alpha) ? __ldg(a.alpha + member_of(slab, e)) : a.alpha_uniform;
                    raw[e] = pga_raw(xv[e], -nacc[e], vn[e], alpha, a.mu, dg);
                }
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const bool act = (act_bits >> e) & 1u;
                    bad |= (act && !isfinite(raw[e])) ? 1u << e : 0u;
                    const T cl = fmin(fmax(raw[e], T(-1)), T(1));
                    if constexpr (EE) {
                        const T ch = fabs(cl - xv[e]);
                        uint32_t b = 0;
                        if (ch > T(1e-12)) b |= EX_BIG;
                        if (ch > T(0)) b |= EX_NZ;
                        if (cl != T(1) && cl != T(-1)) b |= EX_NOTB;
                        ebits |= (act ? b : 0u) << (3 * e);
                    }
                    xo[e] = act ? cl : xv[e];
                    vv[e] = act ? vn[e] : vv[e];
                    sign |= (xo[e] > T(0) ? 1u : 0u) << e;
                    // padding columns past the batch never reach the corners (they stay 0) and
                    // are never read for a real member: they do not keep the slab interior
                    interior |= ((valid_bits >> e) & 1u) && fabs(xo[e]) != T(1);
                }
            }
            if (bad) {
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if ((bad >> e) & 1u) {
                        const int m = member_of(slab, e);
                        atomicMin(a.err + (a.err_seg ? m / a.err_seg : 0),
                                  (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned>(a.it));
                    }
            }
            T* xo0 = a.x_out + static_cast<int64_t>(row) * a.ld + col_of(slab, 0);
            T* vo0 = a.vel + static_cast<int64_t>(row) * a.ld + col_of(slab, 0);
            const bool any_interior = __any_sync(0xffffffffu, interior);
            // x-code mode: a row slab entirely on the box corners is stored as its sign code only
            // (readers take +-1 from it; launch_xcode_fill writes X after the last iteration)
            if (!(a.xskip && cout) || any_interior) {
                stg16(xo0, &xo[0]);
                stg16(xo0 + SPAN / 2, &xo[H]);
            }
            stg16(vo0, &vv[0]);
            stg16(vo0 + SPAN / 2, &vv[H]);
            if (cout) {
                const uint32_t line = static_cast<uint32_t>(sl) * n32 + static_cast<uint32_t>(row);
                cout[line * 32u + lane] = static_cast<uint8_t>(sign);
                if (lane == 0) fout[line] = any_interior ? 1u : 0u;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(a_empty + 8u * static_cast<uint32_t>(s));
#pragma unroll
        for (int d = 0; d < kD; ++d) have[d] = have[d + 1];
    }
    if (cur_slab >= 0) flush_bits();
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn tiled_encoder() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// X / V [n][ld] as a 2D tensor; box = one 1 KB slab row x R rows, no swizzle (the SMEM
// stage is [R][1 KB] row-major, as the consumers read it)
void slab_map(CUtensorMap* m, const void* base, int64_t ld, int n, int elem_bytes) {
    EncodeTiledFn enc = tiled_encoder();
    if (!enc) throw Failure{LCB_CUDA, "cuTensorMapEncodeTiled unavailable"};
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(n)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * static_cast<cuuint64_t>(elem_bytes)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kSlab / elem_bytes), static_cast<cuuint32_t>(kR)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(m, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                           const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Failure{LCB_CUDA, "cuTensorMapEncodeTiled(slab) failed: " + std::to_string(static_cast<int>(r))};
}

template <typename T, bool GEN, bool EE, int FNB = Fnb<T>::v>
void go_stream(const StepArgs<T>& a, int slab0, int nslabs, cudaStream_t st) {
    const int smem = static_cast<int>(sizeof(StreamSmem));
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    ensure_smem_attr(reinterpret_cast<const void*>(k_stream<T, GEN, EE, FNB>), smem, "cudaFuncSetAttribute(k_stream)");
    static std::atomic<int> grid_per_dev[64];
    const int slot = dev >= 0 && dev < 64 ? dev : 0;
    int gpd = grid_per_dev[slot].load(std::memory_order_relaxed);
    if (!gpd) {
        int occ = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<T, GEN, EE, FNB>, kThreadsS, smem),
                   "occupancy(k_stream)");
        gpd = std::max(1, occ) * num_sms(dev);
        grid_per_dev[slot].store(gpd, std::memory_order_relaxed);
    }
    const int rowtiles = (a.n + kR - 1) / kR;
    const int ntiles = rowtiles * nslabs;
    const int grid = std::min(gpd, ntiles);
    CUtensorMap mx, mv;
    slab_map(&mx, a.x_in, a.ld, a.n, static_cast<int>(sizeof(T)));
    slab_map(&mv, a.vel, a.ld, a.n, static_cast<int>(sizeof(T)));
    count_launch();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreadsS);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, k_stream<T, GEN, EE, FNB>, a, rowtiles, slab0, nslabs, mx, mv),
               "cudaLaunchKernelEx(k_stream)");
}

// one warp per (slab, row): +-1 from the sign byte of each lane for row slabs with flag 0
template <typename T>
__global__ void k_xcode_fill(T* X, int64_t ld, int n, const uint8_t* codes, int64_t flag_off, int slab0,
                             int nslabs) {
    constexpr int E = Lanes<T>::E, H = Lanes<T>::H, SPAN = Lanes<T>::SPAN;
    const uint32_t* flags = reinterpret_cast<const uint32_t*>(codes + flag_off);
    const int lane = threadIdx.x & 31;
    const int64_t lines = static_cast<int64_t>(n) * nslabs;
    for (int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < lines;
         w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        if (flags[w] != 0u) continue;
        const int sl = static_cast<int>(w / n);
        const int row = static_cast<int>(w - static_cast<int64_t>(sl) * n);
        const uint32_t b = codes[w * 32 + lane];
        T xo[E];
#pragma unroll
        for (int e = 0; e < E; ++e) xo[e] = ((b >> e) & 1u) ? T(1) : T(-1);
        T* p = X + static_cast<int64_t>(row) * ld + static_cast<int64_t>(slab0 + sl) * SPAN + lane * H;
        stg16(p, &xo[0]);
        stg16(p + SPAN / 2, &xo[H]);
    }
}

}  // namespace

template <typename T>
void launch_xcode_fill(T* X, int64_t ld, int n, const uint8_t* codes, int64_t flag_off, int slab0, int nslabs,
                       cudaStream_t s) {
    const int64_t lines = static_cast<int64_t>(n) * nslabs;
    if (lines <= 0) return;
    const int grid = static_cast<int>(std::min<int64_t>((lines + 7) / 8, 16 * num_sms(-1)));
    count_launch();
    k_xcode_fill<T><<<grid, 256, 0, s>>>(X, ld, n, codes, flag_off, slab0, nslabs);
    cuda_check(cudaGetLastError(), "k_xcode_fill");
}
template void launch_xcode_fill<float>(float*, int64_t, int, const uint8_t*, int64_t, int, int, cudaStream_t);
template void launch_xcode_fill<double>(double*, int64_t, int, const uint8_t*, int64_t, int, int, cudaStream_t);

int stream_slab_cols(int elem_bytes) { return kSlab / elem_bytes; }

template <typename T>
void launch_stream(const StepArgs<T>& a, int slab0, int nslabs, bool early_exit, cudaStream_t s) {
    if (early_exit)
        go_stream<T, true, true>(a, slab0, nslabs, s);
    else if (a.tlim != nullptr || a.alpha != nullptr)
        go_stream<T, true, false>(a, slab0, nslabs, s);
    else if (sizeof(T) == 4 && a.it < 24)
        // before saturation fp32 gathers every neighbour: two gathers in flight pay there
        // (config 4: 5175 vs 5859 us per iteration over the first 20), the leaner one-gather
        // build wins afterwards; both sum in the same order (bitwise identical)
        go_stream<T, false, false, 2>(a, slab0, nslabs, s);
    else
        go_stream<T, false, false>(a, slab0, nslabs, s);
}

template void launch_stream<float>(const StepArgs<float>&, int, int, bool, cudaStream_t);
template void launch_stream<double>(const StepArgs<double>&, int, int, bool, cudaStream_t);

}  // namespace lcb
