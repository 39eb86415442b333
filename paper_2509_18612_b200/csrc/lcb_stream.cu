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
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

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
#define LCB_STREAM_NB 16
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
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
__device__ __forceinline__ uint32_t ld_code(const uint8_t* p, uint64_t pol) {
    uint16_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_code(uint8_t* p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(p), "h"(static_cast<uint16_t>(v)), "l"(pol)
                 : "memory");
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
    uint64_t full[kStages];
    uint64_t empty[kStages];
};

template <typename T, bool GEN, bool EE>
__global__ void __launch_bounds__(kThreadsS, LCB_STREAM_MINB) k_stream(StepArgs<T> a, int rowtiles, int slab0, int nslabs) {
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
        // ---------------- producer: the CSR ranges of tile i+P are loaded while tile i's
        // copies are issued (P tiles of lookahead: the row_ptr loads leave the critical path)
        const uint64_t pol = policy_evict_first();
        constexpr int P = kLook;
        int qrow[P], qbeg[P], qend[P];
        auto fetch = [&](int t, int& row, int& beg, int& end) {
            row = -1;
            beg = end = 0;
            if (t < ntiles && lane < kR) {
                const int slab = t / rowtiles;
                const int idx = (t - slab * rowtiles) * kR + lane;
                if (idx < a.n) {
                    row = a.order ? __ldg(a.order + idx) : idx;
                    beg = __ldg(a.row_ptr + row);
                    end = __ldg(a.row_ptr + row + 1);
                }
            }
        };
#pragma unroll
        for (int q = 0; q < P; ++q) fetch(blockIdx.x + q * gridDim.x, qrow[q], qbeg[q], qend[q]);
        for (int i0 = 0;; i0 += P) {
            bool done = false;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int i = i0 + q;
                const int t = blockIdx.x + i * gridDim.x;
                if (t >= ntiles) {
                    done = true;
                    break;
                }
                const int row = qrow[q], beg = qbeg[q], end = qend[q];
                fetch(t + P * gridDim.x, qrow[q], qbeg[q], qend[q]);
                const int s = i % kStages;
                if (i >= kStages) mbar_wait(&sm.empty[s], ((i / kStages) & 1) ^ 1);
                int sl = t / rowtiles;
                if (a.it & 1) sl = nslabs - 1 - sl;  // snake: reuse the slab just written
                const int slab = slab0 + sl;
                const int abeg = beg & ~3, aend = (end + 3) & ~3;
                const int need = row >= 0 ? aend - abeg : 0;
                int incl = need;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int off = incl - need;
                const bool fits = need > 0 && incl <= kColBuf;
                uint32_t bytes = row >= 0 ? 2u * 512u + (fits ? static_cast<uint32_t>(need) * 4u : 0u) : 0u;
                if (lane < kR) {
                    sm.row[s][lane] = row;
                    sm.beg[s][lane] = beg;
                    sm.deg[s][lane] = end - beg;
                    sm.coff[s][lane] = fits ? off + (beg - abeg) : -1;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
                __syncwarp();
                if (lane == 0) mbar_expect_tx(&sm.full[s], bytes);
                __syncwarp();
                if (row >= 0) {
                    const int64_t o = static_cast<int64_t>(row) * a.ld + static_cast<int64_t>(slab) * SPAN;
                    bulk_g2s(&sm.x[s][lane][0], a.x_in + o, 512u, &sm.full[s], pol);
                    bulk_g2s(&sm.v[s][lane][0], a.vel + o, 512u, &sm.full[s], pol);
                    if (fits)
                        bulk_g2s(&sm.col[s][off], a.col + abeg, static_cast<uint32_t>(need) * 4u, &sm.full[s], pol);
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

    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int s = i % kStages;
        int sl = t / rowtiles;
        if (a.it & 1) sl = nslabs - 1 - sl;
        const int slab = slab0 + sl;
        if (slab != cur_slab) enter_slab(slab);
        mbar_wait(&sm.full[s], (i / kStages) & 1);
        const int row = sm.row[s][j];
        if (row >= 0) {
            const int deg = sm.deg[s][j];
            const int coff = sm.coff[s][j];
            const int* cl = coff >= 0 ? &sm.col[s][coff] : a.col + sm.beg[s][j];
            const int c0 = slab * SPAN + lane * E;
            // codes of this launch's slab sl: [nslabs][n][32] bytes (< 4 GB, launch_stream)
            const uint8_t* sin =
                a.sgn_in ? a.sgn_in + static_cast<uint32_t>(sl) * static_cast<uint32_t>(a.n) * 32u + lane : nullptr;
            // Neighbour sums in CSR order (graph.cpp:116-121).  While every neighbour element of
            // the lane sits on a box corner the partial sums are small integers, exact in fp32 /
            // fp64, so they are kept as integer counts of +1 (SWAR bytes: code bit e -> byte e);
            // from the first batch with an interior value on ANY lane the warp continues with
            // sequential fp adds starting from that exact partial sum.
            uint32_t plus = 0;  // byte e: +1 count of element e (<= 255: folded every 32 neighbours)
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
                const int mycol = lane < cnt ? cl[base + lane] : 0;
                if (!fmode) {
                    uint32_t A = 0xFFu;
                    plus = 0;
                    for (int k = 0; k < cnt; k += kNB) {
                        uint32_t cq[kNB];
#pragma unroll
                        for (int q = 0; q < kNB; ++q) {
                            if (k + q < cnt) {
                                const uint32_t u = static_cast<uint32_t>(__shfl_sync(0xffffffffu, mycol, k + q));
                                cq[q] = ld_code(sin + u * 32u, pol_keep);
                            }
                        }
#pragma unroll
                        for (int q = 0; q < kNB; ++q) {
                            if (k + q < cnt) {
                                A &= cq[q] | (cq[q] >> 4);
                                plus += ((cq[q] & 0xFu) * 0x00204081u) & 0x01010101u;  // bit e -> byte e, no carries
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
                const T* xin = a.x_in + c0;
                for (int k = 0; k < cnt; k += 4) {
                    uint32_t cq[4];
                    V g[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int u = __shfl_sync(0xffffffffu, mycol, (k + q) & 31);
                        cq[q] = (sin && k + q < cnt) ? ld_code(sin + static_cast<uint32_t>(u) * 32u, pol_keep) : 0u;
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
            V xo = xv;
            uint32_t code = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const T x = el(xv, e);
                if (act_bits & (1u << e)) {
                    T vel = el(vv, e);
                    T alpha = a.alpha_uniform;
                    if constexpr (GEN) {
                        if (a.alpha) alpha = __ldg(a.alpha + member_of(slab, e));
                    }
                    const T raw = pga_raw(x, el(acc, e), vel, alpha, a.mu, dg);
                    if (!isfinite(raw)) {  // ascent.cpp:70-72
                        const int m = member_of(slab, e);
                        atomicMin(a.err + (a.err_seg ? m / a.err_seg : 0),
                                  (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned>(a.it));
                    }
                    const T cl = raw < T(-1) ? T(-1) : (raw > T(1) ? T(1) : raw);  // ascent.cpp:73
                    if constexpr (EE) {
                        const T ch = fabs(cl - x);
                        uint32_t b = 0;
                        if (ch > T(1e-12)) b |= EX_BIG;
                        if (ch > T(0)) b |= EX_NZ;
                        if (cl != T(1) && cl != T(-1)) b |= EX_NOTB;
                        ebits |= b << (3 * e);
                    }
                    el(vv, e) = vel;
                    el(xo, e) = cl;
                }
                const T o = el(xo, e);
                code |= (o == T(1) ? 1u : (o == T(-1) ? 16u : 0u)) << e;
            }
            const int64_t off = static_cast<int64_t>(row) * a.ld + c0;
            stg_stream(reinterpret_cast<V*>(a.x_out + off), xo);
            stg_stream(reinterpret_cast<V*>(a.vel + off), vv);
            if (a.sgn_out)
                st_code(a.sgn_out + (static_cast<uint32_t>(sl) * static_cast<uint32_t>(a.n) + static_cast<uint32_t>(row)) * 32u +
                            lane,
                        code, pol_keep);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    if (cur_slab >= 0) flush_bits();
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
    count_launch();
    k_stream<T, GEN, EE><<<grid, kThreadsS, smem, st>>>(a, rowtiles, slab0, nslabs);
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
