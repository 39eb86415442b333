// lcb_stream.cu — K1s: warp-specialised streaming PGA step for graphs whose iterate
// does not live on chip (configs 4 and 5; config 2's unlifted batches when K2 is off).
//
// One launch = one iteration of ascent.cpp:58-77 over the whole batch (Jacobi: every
// row reads the previous iterate of its neighbours).  Work unit = a tile of R rows x
// one 512-byte column slab (128 fp32 / 64 fp64 columns).  Tiles are visited
// slab-major by a persistent grid, so at any moment all SMs work on one slab and the
// slab's saturation codes (1 byte per lane: 32 bytes per row; 32 MB for n = 1M) stay in
// L2 while the iterate itself (2 GB for config 4) streams from HBM exactly once.
//
//   warp 0 (producer): per tile, the rows' CSR ranges, then cp.async.bulk copies of
//           each row's x slab, v slab (512 B each, L2 evict-first) and its column
//           list into a ring of stages, completion on an mbarrier;
//   warps 1..R (consumers): one row of the tile each: neighbour sums from the codes
//           (+-1 exactly) when a neighbour's lane elements sit on the box corners, else
//           from the neighbour's x slab, in CSR order per element (graph.cpp:116-121,
//           so fp64 stays bit-exact); fused heavy-ball / finite check / clamp
//           (ascent.cpp:66-77); x', v' (evict-first) and the row's new code written
//           straight from registers; then the stage is released.
// The own-row traffic (x, v in; x', v' out) is the 16 B/node-update of the roofline
// model; the gathers cost 32 B per neighbour and slab from L2 once saturated.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "../../include/liftcut_b200.h"
#include "lcb_internal.h"

namespace lcb {

namespace {

#ifndef LCB_STREAM_R
#define LCB_STREAM_R 16
#endif
constexpr int kR = LCB_STREAM_R;  // rows per tile = consumer warps per CTA
constexpr int kThreadsS = 32 * (kR + 1);
#ifndef LCB_STREAM_STAGES
#define LCB_STREAM_STAGES 4
#endif
constexpr int kStages = LCB_STREAM_STAGES;
constexpr int kColBuf = 32 * kR;  // int32 column slots per stage (aligned per-row runs)
#ifndef LCB_STREAM_MINB
#define LCB_STREAM_MINB 2
#endif
#ifndef LCB_STREAM_NB
#define LCB_STREAM_NB 8
#endif
constexpr int kNB = LCB_STREAM_NB;  // neighbour codes in flight per batch
#ifndef LCB_STREAM_LOOK
#define LCB_STREAM_LOOK 4
#endif
constexpr int kLook = LCB_STREAM_LOOK;  // producer lookahead (tiles) for the CSR ranges

template <typename T>
struct SVec;
template <>
struct SVec<float> {
    using type = float4;
    static constexpr int E = 4;
};
template <>
struct SVec<double> {
    using type = double2;
    static constexpr int E = 2;
};
__device__ __forceinline__ float& el(float4& v, int e) { return (&v.x)[e]; }
__device__ __forceinline__ double& el(double2& v, int e) { return (&v.x)[e]; }
__device__ __forceinline__ float el(const float4& v, int e) { return (&v.x)[e]; }
__device__ __forceinline__ double el(const double2& v, int e) { return (&v.x)[e]; }

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    // the suspend-time hint parks the warp in the barrier unit instead of re-issuing the
    // probe (waiting warps otherwise take issue slots from the working ones)
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// 2D tensor tile (TMA): box [R rows][512 bytes] of X / V at (column c0, row r0); rows past
// n are zero-filled and still counted in the transaction bytes
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
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// predicated code load (no branch): `fill` when !pred.  0xF0 = all four elements -1 is the
// neutral filler of the integer path (saturated, no +1 counts)
__device__ __forceinline__ uint32_t ld_code_if(const uint8_t* p, bool pred, uint32_t fill) {
    uint32_t v;
    asm volatile(
        "{\n"
        ".reg .pred q;\n"
        "setp.ne.b32 q, %2, 0;\n"
        "mov.b32 %0, %3;\n"
        "@q ld.global.nc.L1::no_allocate.u8 %0, [%1];\n"
        "}\n"
        : "=r"(v)
        : "l"(p), "r"(static_cast<uint32_t>(pred)), "r"(fill));
    return v;
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ uint32_t lds_u8_if(const uint8_t* p, bool pred, uint32_t fill) {
    uint32_t v;
    asm volatile(
        "{\n"
        ".reg .pred q;\n"
        "setp.ne.b32 q, %2, 0;\n"
        "mov.b32 %0, %3;\n"
        "@q ld.shared.u8 %0, [%1];\n"
        "}\n"
        : "=r"(v)
        : "r"(smem_u32(p)), "r"(static_cast<uint32_t>(pred)), "r"(fill));
    return v;
}

__device__ __forceinline__ float4 lds_v(const float4* p) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ double2 lds_v(const double2* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ void stg_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void stg_stream(double2* p, double2 v) { __stcs(p, v); }

__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }

// a neighbour slab whose lane elements are all on the box corners (+1 bit e / -1 bit 4+e)
template <int E>
__device__ __forceinline__ bool sat_code(uint32_t c) {
    constexpr uint32_t full = (1u << E) - 1u;
    return ((c | (c >> 4)) & full) == full;
}

template <typename T>
struct StreamSmem {
    using V = typename SVec<T>::type;
    V x[kStages][kR][32];
    V v[kStages][kR][32];
    int col[kStages][kColBuf];
    int row[kStages][kR];
    int beg[kStages][kR];
    int deg[kStages][kR];
    int coff[kStages][kR];
    int slab[kStages];             // launch-relative slab index of the tile in the stage
    uint8_t codes[kR][2][32][32];  // per consumer warp: code lines of <= 32 neighbours, two rows
    uint64_t full[kStages];
    uint64_t empty[kStages];
};

template <typename T, bool GEN, bool EE>
__global__ void __launch_bounds__(kThreadsS, LCB_STREAM_MINB) k_stream(StepArgs<T> a, int rowtiles, int slab0, int nslabs,
                                                                      const __grid_constant__ CUtensorMap mx,
                                                                      const __grid_constant__ CUtensorMap mv) {
    using V = typename SVec<T>::type;
    constexpr int E = SVec<T>::E;
    constexpr int SPAN = 32 * E;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    StreamSmem<T>& sm = *reinterpret_cast<StreamSmem<T>*>(smem_raw);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ntiles = rowtiles * nslabs;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kR);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (EE) {
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < a.members; i += blockDim.x) a.flags_zero[i] = 0;
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer.  Rows in natural order: a tile is R consecutive rows, so its
        // x and v slabs are ONE 2D TMA box each ([R][512 B]) and its column lists one contiguous
        // bulk copy.  The row_ptr range of tile i+P loads while tile i's copies are issued.
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mx)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mv)) : "memory");
        }
        const uint64_t pol = policy_evict_first();
        constexpr int P = kLook;
        int qrp[P];  // lane j <= R: row_ptr[min(r0 + j, n)] of the tile P ahead
        // tile t = (row tile rt, slab sl); this CTA's tiles t = blockIdx.x + i * gridDim.x are
        // walked incrementally (no division per tile)
        const int drt = static_cast<int>(gridDim.x) % rowtiles, dsl = static_cast<int>(gridDim.x) / rowtiles;
        int cur_rt = static_cast<int>(blockIdx.x) % rowtiles, cur_sl = static_cast<int>(blockIdx.x) / rowtiles;
        int ah_rt = cur_rt, ah_sl = cur_sl;  // the tile P ahead
        auto adv = [&](int& rt, int& sl) {
            rt += drt;
            sl += dsl;
            if (rt >= rowtiles) {
                rt -= rowtiles;
                ++sl;
            }
        };
        auto fetch = [&]() {
            int v = 0;
            if (ah_sl < nslabs && lane <= kR) v = __ldg(a.row_ptr + min(ah_rt * kR + lane, a.n));
            adv(ah_rt, ah_sl);
            return v;
        };
#pragma unroll
        for (int q = 0; q < P; ++q) qrp[q] = fetch();
        const CUtensorMap* mapx = &mx;
        const CUtensorMap* mapv = &mv;
        for (int i0 = 0;; i0 += P) {
            bool done = false;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int i = i0 + q;
                if (cur_sl >= nslabs) {
                    done = true;
                    break;
                }
                const int beg = qrp[q];
                qrp[q] = fetch();
                const int end = __shfl_down_sync(0xffffffffu, beg, 1);
                const int first = __shfl_sync(0xffffffffu, beg, 0), last = __shfl_sync(0xffffffffu, beg, kR);
                const int s = i % kStages;
                if (i >= kStages) mbar_wait(&sm.empty[s], ((i / kStages) & 1) ^ 1);
                int sl = cur_sl;
                const int r0 = cur_rt * kR;
                adv(cur_rt, cur_sl);
                if (a.it & 1) sl = nslabs - 1 - sl;  // snake: reuse the slab just written
                const int slab = slab0 + sl;
                const int abeg = first & ~3;
                const int need = ((last + 3) & ~3) - abeg;          // whole tile's column run
                const int ncopy = min(need, kColBuf);                 // staged prefix
                if (lane == 0) sm.slab[s] = sl;
                if (lane < kR) {
                    const int row = r0 + lane;
                    const bool ok = row < a.n;
                    sm.row[s][lane] = ok ? row : -1;
                    sm.beg[s][lane] = beg;
                    sm.deg[s][lane] = ok ? end - beg : 0;
                    sm.coff[s][lane] = (ok && end - abeg <= ncopy) ? beg - abeg : -1;
                }
                __syncwarp();
                if (lane == 0) {
                    const uint32_t bytes = 2u * kR * 512u + static_cast<uint32_t>(ncopy) * 4u;
                    mbar_expect_tx(&sm.full[s], bytes);
                    tma_tile(&sm.x[s][0][0], mapx, slab * SPAN, r0, &sm.full[s], pol);
                    tma_tile(&sm.v[s][0][0], mapv, slab * SPAN, r0, &sm.full[s], pol);
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
    const uint64_t pol_keep = policy_evict_last();
    constexpr uint32_t FULL = (1u << E) - 1u;
    // per-slab lane state, fixed for the whole launch (no per-row division / loads): which of
    // the lane's elements step at this iteration (bit e), the member of element e is
    // recomputed only on the rare paths that need it (exit bits, non-finite values)
    int cur_slab = -1;
    uint32_t act_bits = 0;
    uint32_t ebits = 0;  // 3 exit bits per element (EE)
    auto member_of = [&](int slab, int e) { return (a.col_base + slab * SPAN + lane * E + e) / a.l; };
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
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int colx = slab * SPAN + lane * E + e;
            bool act = colx < a.W;
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
    };
    bool float_hint = false;  // the previous row met an unsaturated neighbour

    // The code lines (32 B) of a row's first <= 32 neighbours are copied into this warp's
    // SMEM buffer with cp.async one tile ahead (lane k copies neighbour k), so the
    // neighbour sums read SMEM only and the L2 latency of the gathers is off the critical path.
    auto issue_codes = [&](int st, int sl, int buf) {
        const int row = sm.row[st][j];
        if (row >= 0 && a.sgn_in) {
            const int deg = sm.deg[st][j];
            uint8_t* dst = &sm.codes[j][buf][lane][0];
            if (lane < deg) {
                const int coff = sm.coff[st][j];
                const int u = coff >= 0 ? sm.col[st][coff + lane] : __ldg(a.col + sm.beg[st][j] + lane);
                const uint8_t* src =
                    a.sgn_in + (static_cast<uint32_t>(sl) * static_cast<uint32_t>(a.n) + static_cast<uint32_t>(u)) * 32u;
                cp_async16(dst, src);
                cp_async16(dst + 16, src + 16);
            } else if (lane < ((deg + 3) & ~3)) {
                // neutral filler up to a multiple of 4: every element -1 (saturated, no +1 count),
                // so the integer loop runs without bounds checks
                const uint4 f = make_uint4(0xF0F0F0F0u, 0xF0F0F0F0u, 0xF0F0F0F0u, 0xF0F0F0F0u);
                reinterpret_cast<uint4*>(dst)[0] = f;
                reinterpret_cast<uint4*>(dst)[1] = f;
            }
        }
        cp_async_commit();
    };

    const int my_tiles = (ntiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                         static_cast<int>(gridDim.x);
    if (my_tiles > 0) {
        mbar_wait(&sm.full[0], 0);
        issue_codes(0, sm.slab[0], 0);
    }
    for (int i = 0; i < my_tiles; ++i) {
        const int s = i % kStages;
        const int sl = sm.slab[s];
        const int slab = slab0 + sl;
        if (slab != cur_slab) enter_slab(slab);
        // next tile: its stage is normally landed already (the producer runs ahead)
        if (i + 1 < my_tiles) {
            const int sn = (i + 1) % kStages;
            mbar_wait(&sm.full[sn], ((i + 1) / kStages) & 1);
            issue_codes(sn, sm.slab[sn], (i + 1) & 1);
        } else {
            cp_async_commit();
        }
        cp_async_wait1();  // this tile's code lines have landed
        __syncwarp();
        const int row = sm.row[s][j];
        if (row >= 0) {
            const int deg = sm.deg[s][j];
            const int coff = sm.coff[s][j];
            const int* cl = coff >= 0 ? &sm.col[s][coff] : a.col + sm.beg[s][j];
            const int c0 = slab * SPAN + lane * E;
            const uint8_t* cb = &sm.codes[j][i & 1][0][lane];  // neighbour k's byte for this lane: cb[32 k]
            // codes of this launch's slab sl beyond the staged 32 neighbours: [nslabs][n][32] (< 4 GB)
            const uint8_t* sin =
                a.sgn_in ? a.sgn_in + static_cast<uint32_t>(sl) * static_cast<uint32_t>(a.n) * 32u + lane : nullptr;
            // Neighbour sums in CSR order (graph.cpp:116-121).  While every neighbour element of
            // the lane sits on a box corner the partial sums are small integers, exact in fp32 /
            // fp64, so they are kept as integer counts of +1 (SWAR bytes: code bit e -> byte e);
            // from the first batch with an interior value on ANY lane the warp continues with
            // sequential fp adds starting from that exact partial sum.
            uint32_t pe[E];
#pragma unroll
            for (int e = 0; e < E; ++e) pe[e] = 0;
            int folded = 0;
            bool fmode = sin == nullptr || float_hint;
            V acc;
#pragma unroll
            for (int e = 0; e < E; ++e) el(acc, e) = T(0);
            for (int base = 0; base < deg; base += 32) {
                const int cnt = min(32, deg - base);
                const bool staged = base == 0;
                int mycol = 0;  // neighbour index of this lane's slot (global path / float path only)
                if (!staged) mycol = lane < cnt ? cl[base + lane] : 0;
                if (!fmode) {
                    uint32_t A = 0xFFu, plus = 0;
                    if (staged) {
                        for (int k = 0; k < cnt; k += 4) {  // lines cnt..round4(cnt) hold the filler
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const uint32_t c = cb[32 * (k + q)];
                                A &= c | (c >> 4);
                                plus += ((c & 0xFu) * 0x00204081u) & 0x01010101u;  // bit e -> byte e, no carries
                            }
                        }
                    } else {
                        for (int k = 0; k < cnt; k += kNB) {
                            uint32_t cq[kNB];
#pragma unroll
                            for (int q = 0; q < kNB; ++q) {
                                const uint32_t u = static_cast<uint32_t>(__shfl_sync(0xffffffffu, mycol, (k + q) & 31));
                                cq[q] = ld_code_if(sin + u * 32u, k + q < cnt, 0xF0u);
                            }
#pragma unroll
                            for (int q = 0; q < kNB; ++q) {
                                A &= cq[q] | (cq[q] >> 4);
                                plus += ((cq[q] & 0xFu) * 0x00204081u) & 0x01010101u;
                            }
                        }
                    }
                    if (__all_sync(0xffffffffu, (A & FULL) == FULL)) {
#pragma unroll
                        for (int e = 0; e < E; ++e) pe[e] += (plus >> (8 * e)) & 0xFFu;
                        folded += cnt;
                        continue;
                    }
                    fmode = true;  // exact partial sum so far: (+1 count) - (-1 count)
#pragma unroll
                    for (int e = 0; e < E; ++e) el(acc, e) = static_cast<T>(2 * static_cast<int>(pe[e]) - folded);
                }
                if (staged) mycol = lane < cnt ? cl[base + lane] : 0;
                const T* xin = a.x_in + c0;
                for (int k = 0; k < cnt; k += 4) {
                    uint32_t cq[4];
                    V g[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int u = __shfl_sync(0xffffffffu, mycol, (k + q) & 31);
                        const bool in = sin != nullptr && k + q < cnt;
                        cq[q] = staged ? lds_u8_if(cb + 32 * ((k + q) & 31), in, 0u)
                                       : ld_code_if(sin + static_cast<uint32_t>(u) * 32u, in, 0u);
                        if (k + q < cnt && !sat_code<E>(cq[q]))
                            g[q] = __ldg(reinterpret_cast<const V*>(xin + static_cast<int64_t>(u) * a.ld));
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (k + q < cnt) {
                            const bool sat = sat_code<E>(cq[q]);
#pragma unroll
                            for (int e = 0; e < E; ++e)
                                el(acc, e) = radd(el(acc, e), sat ? (((cq[q] >> e) & 1u) ? T(1) : T(-1)) : el(g[q], e));
                        }
                    }
                }
            }
            if (!fmode) {
#pragma unroll
                for (int e = 0; e < E; ++e) el(acc, e) = static_cast<T>(2 * static_cast<int>(pe[e]) - folded);
            }
            float_hint = fmode && sin != nullptr;

            const V xv = lds_v(&sm.x[s][j][lane]);
            V vv = lds_v(&sm.v[s][j][lane]);
            const T dg = static_cast<T>(deg);
            V xo;
            uint32_t code = 0, bad = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const T x = el(xv, e);
                const bool act = (act_bits >> e) & 1u;
                T alpha = a.alpha_uniform;
                if constexpr (GEN) {
                    if (a.alpha) alpha = __ldg(a.alpha + member_of(slab, e));
                }
                T vel = el(vv, e);
                const T raw = pga_raw(x, el(acc, e), vel, alpha, a.mu, dg);
                bad |= (act && !isfinite(raw)) ? 1u << e : 0u;       // ascent.cpp:70-72
                const T cl = fmin(fmax(raw, T(-1)), T(1));             // ascent.cpp:73 (raw finite)
                const T o = act ? cl : x;
                if constexpr (EE) {
                    const T ch = fabs(cl - x);
                    uint32_t b = 0;
                    if (ch > T(1e-12)) b |= EX_BIG;
                    if (ch > T(0)) b |= EX_NZ;
                    if (cl != T(1) && cl != T(-1)) b |= EX_NOTB;
                    ebits |= (act ? b : 0u) << (3 * e);
                }
                el(vv, e) = act ? vel : el(vv, e);
                el(xo, e) = o;
                code |= (o == T(1) ? 1u : 0u) << e;
                code |= (o == T(-1) ? 16u : 0u) << e;
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
            const int64_t off = static_cast<int64_t>(row) * a.ld + c0;
            stg_stream(reinterpret_cast<V*>(a.x_out + off), xo);
            stg_stream(reinterpret_cast<V*>(a.vel + off), vv);
            if (a.sgn_out)
                a.sgn_out[(static_cast<uint32_t>(sl) * static_cast<uint32_t>(a.n) + static_cast<uint32_t>(row)) * 32u + lane] =
                    static_cast<uint8_t>(code);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
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

// X / V [n][ld] as a 2D tensor; box = one 512-byte slab of R rows, no swizzle (the SMEM
// stage is [R][512 B] row-major, as the consumers read it)
void slab_map(CUtensorMap* m, const void* base, int64_t ld, int n, int elem_bytes) {
    EncodeTiledFn enc = tiled_encoder();
    if (!enc) throw Failure{LCB_CUDA, "cuTensorMapEncodeTiled unavailable"};
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(n)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * static_cast<cuuint64_t>(elem_bytes)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(512 / elem_bytes), static_cast<cuuint32_t>(kR)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(m, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                           const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Failure{LCB_CUDA, "cuTensorMapEncodeTiled(slab) failed: " + std::to_string(static_cast<int>(r))};
}

template <typename T, bool GEN, bool EE>
void go_stream(const StepArgs<T>& a, int slab0, int nslabs, cudaStream_t st) {
    const int smem = static_cast<int>(sizeof(StreamSmem<T>));
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    ensure_smem_attr(reinterpret_cast<const void*>(k_stream<T, GEN, EE>), smem, "cudaFuncSetAttribute(k_stream)");
    static std::atomic<int> grid_per_dev[64];
    const int slot = dev >= 0 && dev < 64 ? dev : 0;
    int gpd = grid_per_dev[slot].load(std::memory_order_relaxed);
    if (!gpd) {
        int occ = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<T, GEN, EE>, kThreadsS, smem),
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
    k_stream<T, GEN, EE><<<grid, kThreadsS, smem, st>>>(a, rowtiles, slab0, nslabs, mx, mv);
}

}  // namespace

template <typename T>
void launch_stream(const StepArgs<T>& a, int slab0, int nslabs, bool early_exit, cudaStream_t s) {
    if (early_exit)
        go_stream<T, true, true>(a, slab0, nslabs, s);
    else if (a.tlim != nullptr || a.alpha != nullptr)
        go_stream<T, true, false>(a, slab0, nslabs, s);
    else
        go_stream<T, false, false>(a, slab0, nslabs, s);
}

template void launch_stream<float>(const StepArgs<float>&, int, int, bool, cudaStream_t);
template void launch_stream<double>(const StepArgs<double>&, int, int, bool, cudaStream_t);

}  // namespace lcb
