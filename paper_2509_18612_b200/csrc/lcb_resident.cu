// lcb_resident.cu — K2: member-resident persistent PGA kernel (fp32).
//
// For graphs whose per-column state fits on chip (n * K * 8 B <= ~220 KB, i.e.
// configs 1 and 2), one CTA owns K columns of the batch for ALL n rows:
//   * the iterate lives in shared memory, double-buffered (Jacobi update:
//     ascent.cpp:58-77 reads the old iterate of every neighbour);
//   * the velocity lives in registers (each row is owned by one lane);
//   * all T iterations run inside one launch with a CTA barrier per iteration —
//     members are independent (ascent.cpp:52), so no grid-wide sync is needed;
//   * the CSR is streamed from L2 every iteration (relabelled rows in
//     degree-descending order, uint16 columns), shared by every CTA.
// HBM is touched only to load the initial slab and write the final one.  The
// per-iteration work is 8 lanes per row over the row's neighbours (coalesced
// column loads, random LDS gathers), a 3-step shuffle reduction, and the fused
// heavy-ball / clamp / finite-check / exit-flag epilogue.
//
// Summation order within a row is a fixed lane-strided tree, not the reference's
// sequential order, so this path is the fp32 fast path (norm-wise tolerance);
// the fp64 bit-exact path is k_step in lcb_kernels.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "lcb_internal.h"

namespace lcb {

namespace {

template <int K>
struct SlabT;
template <>
struct SlabT<1> {
    using type = float;
};
template <>
struct SlabT<2> {
    using type = float2;
};

__device__ __forceinline__ float comp(const float& v, int) { return v; }
__device__ __forceinline__ float comp(const float2& v, int k) { return k ? v.y : v.x; }
__device__ __forceinline__ void setc(float& v, int, float x) { v = x; }
__device__ __forceinline__ void setc(float2& v, int k, float x) {
    if (k)
        v.y = x;
    else
        v.x = x;
}
__device__ __forceinline__ void addto(float& a, const float& b) { a += b; }
__device__ __forceinline__ void addto(float2& a, const float2& b) {
    a.x += b.x;
    a.y += b.y;
}
__device__ __forceinline__ float xor_sum8(float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v;
}
__device__ __forceinline__ float2 xor_sum8(float2 v) {
    v.x = xor_sum8(v.x);
    v.y = xor_sum8(v.y);
    return v;
}
__device__ __forceinline__ void zero(float& v) { v = 0.f; }
__device__ __forceinline__ void zero(float2& v) { v = make_float2(0.f, 0.f); }

constexpr int kThreads = 1024;
constexpr int kSub = kThreads / 8;  // 8-lane subgroups per CTA

template <int K, int SLOTS, bool GEN, bool EE>
__global__ void __launch_bounds__(kThreads, 1) k_resident(ResidentArgs a) {
    using VT = typename SlabT<K>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    VT* xs0 = reinterpret_cast<VT*>(smem_raw);
    VT* xs1 = xs0 + a.n;
    __shared__ uint32_t sflag[3][K];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int l8 = lane & 7;
    const int sg = (tid >> 5) * 4 + (lane >> 3);
    const int c0 = blockIdx.x * K;
    const int n = a.n;

    // per-column parameters
    float alpha_k[K];
    int tl[K];
    bool valid[K];
    int mem[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int c = c0 + k;
        valid[k] = c < a.W;
        mem[k] = valid[k] ? c / a.l : 0;
        alpha_k[k] = a.alpha_uniform;
        tl[k] = a.T;
        if (GEN && valid[k]) {
            if (a.alpha) alpha_k[k] = __ldg(a.alpha + mem[k]);
            if (a.tlim) tl[k] = __ldg(a.tlim + mem[k]);
        }
    }

    // load the slab (new row r <- old row perm[r])
    for (int r = tid; r < n; r += kThreads) {
        const float* src = a.X + static_cast<int64_t>(__ldg(a.perm + r)) * a.ld + c0;
        VT v;
#pragma unroll
        for (int k = 0; k < K; ++k) setc(v, k, valid[k] ? src[k] : 0.f);
        xs0[r] = v;
    }
    if (tid < 3 * K) (&sflag[0][0])[tid] = 0u;

    VT vreg[SLOTS];
#pragma unroll
    for (int q = 0; q < SLOTS; ++q) zero(vreg[q]);
    __syncthreads();

    int it = 0;
    for (; it < a.T; ++it) {
        const VT* cur = (it & 1) ? xs1 : xs0;
        VT* nxt = (it & 1) ? xs0 : xs1;
        bool act[K];
        bool any = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            act[k] = valid[k] && it < tl[k];
            if (EE && act[k] && it > 0) act[k] = ex_continue(sflag[(it + 2) % 3][k]);
            any |= act[k];
        }
        if (!any) break;  // uniform: derived from shared state after a barrier
        if (EE && tid < K) sflag[(it + 1) % 3][tid] = 0u;
        uint32_t bits[K];
#pragma unroll
        for (int k = 0; k < K; ++k) bits[k] = 0u;

        for (int q = 0; q < SLOTS; ++q) {
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                const int r = sg + kSub * (q * 8 + p);
                int beg = 0, end = 0;
                if (r < n) {
                    beg = __ldg(a.row_ptr + r);
                    end = __ldg(a.row_ptr + r + 1);
                }
                VT acc;
                zero(acc);
                for (int e = beg + l8; e < end; e += 8) addto(acc, cur[__ldg(a.col + e)]);
                acc = xor_sum8(acc);
                if (l8 == p && r < n) {
                    const VT xv = cur[r];
                    const float dg = static_cast<float>(end - beg);
                    VT xo = xv;
                    VT vv = vreg[0];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        if (!act[k]) continue;
                        const float x = comp(xv, k);
                        const float y = dg * x - comp(acc, k);        // Lx (graph.cpp:120)
                        const float v = a.mu * comp(vv, k) + y;       // ascent.cpp:68
                        const float raw = x + alpha_k[k] * v;         // ascent.cpp:69
                        if (!isfinite(raw))
                            atomicMin(a.err, (static_cast<unsigned long long>(mem[k]) << 32) |
                                                 static_cast<unsigned>(it));
                        const float cl = raw < -1.f ? -1.f : (raw > 1.f ? 1.f : raw);
                        if (EE) {
                            const float ch = fabsf(cl - x);
                            if (ch > 1e-12f) bits[k] |= EX_BIG;
                            if (ch > 0.f) bits[k] |= EX_NZ;
                            if (cl != 1.f && cl != -1.f) bits[k] |= EX_NOTB;
                        }
                        setc(xo, k, cl);
                        setc(vv, k, v);
                    }
                    nxt[r] = xo;
                    vreg[0] = vv;
                }
            }
            // rotate the velocity queue cyclically: slot q+1 moves to the front;
            // after SLOTS rotations the queue is back in order for the next iteration
            const VT head = vreg[0];
#pragma unroll
            for (int s = 0; s + 1 < SLOTS; ++s) vreg[s] = vreg[s + 1];
            vreg[SLOTS - 1] = head;
        }
        if (EE) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                // members spanning several CTAs never reach here (host gate: K % l == 0)
                const uint32_t b = __reduce_or_sync(0xffffffffu, bits[k]);
                if (lane == 0 && b) atomicOr(&sflag[it % 3][k], b);
            }
        }
        __syncthreads();
    }

    // write back the final slab
    const VT* fin = (it & 1) ? xs1 : xs0;
    for (int r = tid; r < n; r += kThreads) {
        float* dst = a.X + static_cast<int64_t>(__ldg(a.perm + r)) * a.ld + c0;
        const VT v = fin[r];
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (valid[k]) dst[k] = comp(v, k);
    }
}

}  // namespace

int resident_slots(int n) {
    const int per_sub = (n + kSub - 1) / kSub;
    return (per_sub + 7) / 8;
}

bool resident_fits(int n, int W, int l, bool ee, int& K) {
    K = (W / 2 >= 148 && static_cast<int64_t>(n) * 2 * 8 <= kResidentSmemMax) ? 2 : 1;
    if (static_cast<int64_t>(n) * K * 8 > kResidentSmemMax) return false;
    if (n > 65535) return false;
    if (ee && (K % l) != 0) return false;  // a member's columns must share a CTA
    return resident_slots(n) <= 28;
}

template <int K, int SLOTS, bool GEN, bool EE>
static void go(const ResidentArgs& a, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(a.n) * K * 8;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_resident<K, SLOTS, GEN, EE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kResidentSmemMax);
        attr = true;
    }
    const int ctas = (a.W + K - 1) / K;
    count_launch();
    k_resident<K, SLOTS, GEN, EE><<<ctas, kThreads, smem, s>>>(a);
}

template <int K, bool GEN, bool EE>
static void by_slots(const ResidentArgs& a, cudaStream_t s) {
    const int sl = resident_slots(a.n);
    if (sl <= 1)
        go<K, 1, GEN, EE>(a, s);
    else if (sl <= 2)
        go<K, 2, GEN, EE>(a, s);
    else if (sl <= 4)
        go<K, 4, GEN, EE>(a, s);
    else if (sl <= 8)
        go<K, 8, GEN, EE>(a, s);
    else if (sl <= 10)
        go<K, 10, GEN, EE>(a, s);
    else if (sl <= 14)
        go<K, 14, GEN, EE>(a, s);
    else
        go<K, 28, GEN, EE>(a, s);
}

void launch_resident(const ResidentArgs& a, int K, bool ee, cudaStream_t s) {
    const bool gen = ee || a.alpha || a.tlim;
    if (K == 2) {
        if (ee)
            by_slots<2, true, true>(a, s);
        else if (gen)
            by_slots<2, true, false>(a, s);
        else
            by_slots<2, false, false>(a, s);
    } else {
        if (ee)
            by_slots<1, true, true>(a, s);
        else if (gen)
            by_slots<1, true, false>(a, s);
        else
            by_slots<1, false, false>(a, s);
    }
}

}  // namespace lcb
