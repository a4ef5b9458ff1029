// rhseg_device.cuh -- shared device-side definitions for the sm_100a RHSEG path.
//
// Exactness contract (reference _kernels.py:1-12, dissim.py:33-42):
// every dissimilarity is evaluated in fp64 with the reference's operation order and
// no FMA contraction (explicit __d*_rn intrinsics, and the whole library is compiled
// with -fmad=false):
//   coef = (n_i * n_j) / (n_i + n_j);  s = sum_b (mu_i[b] - mu_j[b])^2 (b ascending);
//   d = sqrt(coef * s);   mu[r][b] = sums[r][b] / count[r]  (IEEE div, cached).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

namespace rhseg {

#ifndef RHSEG_KTHREADS
#define RHSEG_KTHREADS 256
#endif
constexpr int kThreads = RHSEG_KTHREADS;  // CTA size of every section kernel (the loop's A/B knob)
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCluster = 16;         // non-portable cluster limit on sm_100a
constexpr int kNoJ = INT_MAX;           // "no partner" sentinel inside reductions
constexpr double kInf = __builtin_huge_val();

// ---------------------------------------------------------------------------
// Exact pair dissimilarity pieces (dissim.py:33-42 op order)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double bsmse_step(double s, double mi, double mj) {
    double t = __dsub_rn(mi, mj);
    return __dadd_rn(s, __dmul_rn(t, t));
}
__device__ __forceinline__ double bsmse_finish(double ni, double nj, double s) {
    double coef = __ddiv_rn(__dmul_rn(ni, nj), __dadd_rn(ni, nj));
    return __dsqrt_rn(__dmul_rn(coef, s));
}

// ---------------------------------------------------------------------------
// Extension measures (BASELINE north star: BSMSE / SAM / Euclidean). The
// reference ships only sqrt-bsmse (dissim.py:45); these follow the same
// conventions (fp64, bands ascending, no FMA) and are pinned only against the
// oracle's restatement (oracle/rhseg_oracle.c), i.e. parity unpinned.
//   euclidean: d = sqrt(sum_b (mu_i[b] - mu_j[b])^2)
//   sam:       d = acos(clamp(dot / sqrt(n2_i * n2_j), -1, 1)),
//              dot = sum_b mu_i[b] * mu_j[b], n2 = sum_b mu[b]^2;
//              a zero vector gives 0 against a zero vector, pi/2 otherwise.
// ---------------------------------------------------------------------------
enum Measure { kBsmse = 0, kEuclid = 1, kSam = 2 };

// fdlibm's e_acos algorithm restated with explicit IEEE operations, so the
// device and the oracle compute the same bits (SAM ties stay ties).
__device__ __forceinline__ double rhseg_acos(double x) {
    const double pi = 3.14159265358979311600e+00, pio2_hi = 1.57079632679489655800e+00,
                 pio2_lo = 6.12323399573676603587e-17, pS0 = 1.66666666666666657415e-01,
                 pS1 = -3.25565818622400915405e-01, pS2 = 2.01212532134862925881e-01,
                 pS3 = -4.00555345006794114027e-02, pS4 = 7.91534994289814532176e-04,
                 pS5 = 3.47933107596021167570e-05, qS1 = -2.40339491173441421878e+00,
                 qS2 = 2.02094576023350569471e+00, qS3 = -6.88283971605453293030e-01,
                 qS4 = 7.70381505559019352791e-02;
    const int hx = __double2hiint(x);
    const int ix = hx & 0x7fffffff;
    if (ix >= 0x3ff00000) {
        if (((ix - 0x3ff00000) | __double2loint(x)) == 0) return hx > 0 ? 0.0 : __dadd_rn(pi, __dmul_rn(2.0, pio2_lo));
        return __longlong_as_double(0x7ff8000000000000LL);
    }
    auto pq = [&](double z) {
        const double p = __dmul_rn(
            z, __dadd_rn(pS0, __dmul_rn(z, __dadd_rn(pS1, __dmul_rn(z, __dadd_rn(pS2, __dmul_rn(z, __dadd_rn(
                                                        pS3, __dmul_rn(z, __dadd_rn(pS4, __dmul_rn(z, pS5)))))))))));
        const double q = __dadd_rn(
            1.0, __dmul_rn(z, __dadd_rn(qS1, __dmul_rn(z, __dadd_rn(qS2, __dmul_rn(z, __dadd_rn(qS3, __dmul_rn(z, qS4))))))));
        return __ddiv_rn(p, q);
    };
    if (ix < 0x3fe00000) {
        if (ix <= 0x3c600000) return __dadd_rn(pio2_hi, pio2_lo);
        const double r = pq(__dmul_rn(x, x));
        return __dsub_rn(pio2_hi, __dsub_rn(x, __dsub_rn(pio2_lo, __dmul_rn(x, r))));
    } else if (hx < 0) {
        const double z = __dmul_rn(__dadd_rn(1.0, x), 0.5);
        const double r = pq(z);
        const double s = __dsqrt_rn(z);
        const double w = __dsub_rn(__dmul_rn(r, s), pio2_lo);
        return __dsub_rn(pi, __dmul_rn(2.0, __dadd_rn(s, w)));
    } else {
        const double z = __dmul_rn(__dsub_rn(1.0, x), 0.5);
        const double s = __dsqrt_rn(z);
        const double df = __hiloint2double(__double2hiint(s), 0);
        const double c = __ddiv_rn(__dsub_rn(z, __dmul_rn(df, df)), __dadd_rn(s, df));
        const double r = pq(z);
        const double w = __dadd_rn(__dmul_rn(r, s), c);
        return __dmul_rn(2.0, __dadd_rn(df, w));
    }
}

template <int M>
__device__ __forceinline__ double acc_step(double s, double mi, double mj) {
    if (M == kSam) return __dadd_rn(s, __dmul_rn(mi, mj));
    return bsmse_step(s, mi, mj);
}
__device__ __forceinline__ double sam_finish(double dot, double n2i, double n2j) {
    if (n2i == 0.0 || n2j == 0.0) return (n2i == n2j) ? 0.0 : 1.57079632679489655800e+00;
    double c = __ddiv_rn(dot, __dsqrt_rn(__dmul_rn(n2i, n2j)));
    c = c > 1.0 ? 1.0 : (c < -1.0 ? -1.0 : c);
    return rhseg_acos(c);
}
// ni/nj: pixel counts, n2i/n2j: squared norms of the means (SAM only).
template <int M>
__device__ __forceinline__ double pair_finish(double ni, double nj, double s, double n2i, double n2j) {
    if (M == kBsmse) return bsmse_finish(ni, nj, s);
    if (M == kEuclid) return __dsqrt_rn(s);
    return sam_finish(s, n2i, n2j);
}
// n2 of one mean vector: sequential ascending sum of squares (oracle order).
__device__ __forceinline__ double norm2_seq(const double* mu, size_t stride, int B) {
    double s = 0.0;
    for (int k = 0; k < B; ++k) {
        const double m = mu[(size_t)k * stride];
        s = __dadd_rn(s, __dmul_rn(m, m));
    }
    return s;
}

// ---------------------------------------------------------------------------
// Lexicographic keys.
//   RowBest (d, j): per-row best partner; strict < over ascending j in the
//     reference (_kernels.py:55, 110) == lexicographic min of (d, j).
//   Pair (d, lo, hi): global stage minimum; np.argmin over ascending rows of
//     per-row bests (engine.py:281-296) == lexicographic min of (d, min, max).
// Candidates with d not < +inf (inf or NaN) are never accepted, matching the
// reference's strict `d < best_d` starting from +inf.
// ---------------------------------------------------------------------------
struct RowBest {
    double d;
    int j;
};
struct Pair {
    double d;
    int lo, hi;
};

__device__ __forceinline__ RowBest rb_none() { return RowBest{kInf, kNoJ}; }
__device__ __forceinline__ Pair pair_none() { return Pair{kInf, kNoJ, kNoJ}; }

__device__ __forceinline__ bool rb_less(double d, int j, const RowBest& b) {
    return d < b.d || (d == b.d && j < b.j);
}
__device__ __forceinline__ void rb_offer(RowBest& b, double d, int j) {
    if (d < kInf && rb_less(d, j, b)) { b.d = d; b.j = j; }
}
__device__ __forceinline__ bool pair_less(const Pair& x, const Pair& y) {
    return x.d < y.d || (x.d == y.d && (x.lo < y.lo || (x.lo == y.lo && x.hi < y.hi)));
}
__device__ __forceinline__ void pair_offer(Pair& b, const Pair& c) {
    if (c.d < kInf && pair_less(c, b)) b = c;
}
__device__ __forceinline__ Pair make_pair(double d, int i, int j) {
    return Pair{d, i < j ? i : j, i < j ? j : i};
}

__device__ __forceinline__ RowBest warp_min_rb(RowBest v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double d = __shfl_xor_sync(0xffffffffu, v.d, o);
        int j = __shfl_xor_sync(0xffffffffu, v.j, o);
        if (d < v.d || (d == v.d && j < v.j)) { v.d = d; v.j = j; }
    }
    return v;
}
__device__ __forceinline__ Pair warp_min_pair(Pair v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Pair c;
        c.d = __shfl_xor_sync(0xffffffffu, v.d, o);
        c.lo = __shfl_xor_sync(0xffffffffu, v.lo, o);
        c.hi = __shfl_xor_sync(0xffffffffu, v.hi, o);
        if (pair_less(c, v)) v = c;
    }
    return v;
}

// Block-wide lexicographic minima through a kWarps-entry shared scratch.
// Every thread returns the block result. Contains two __syncthreads().
__device__ __forceinline__ RowBest block_min_rb(RowBest v, RowBest* scratch) {
    v = warp_min_rb(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    RowBest r = scratch[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) {
        RowBest c = scratch[w];
        if (c.d < r.d || (c.d == r.d && c.j < r.j)) r = c;
    }
    __syncthreads();
    return r;
}
__device__ __forceinline__ Pair block_min_pair(Pair v, Pair* scratch) {
    v = warp_min_pair(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    Pair r = scratch[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w)
        if (pair_less(scratch[w], r)) r = scratch[w];
    __syncthreads();
    return r;
}

// Two block-wide minima with one shared exchange (scratch: 2 * kWarps entries).
__device__ __forceinline__ void block_min_pair2(Pair& a, Pair& b, Pair* scratch) {
    a = warp_min_pair(a);
    b = warp_min_pair(b);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        scratch[warp] = a;
        scratch[kWarps + warp] = b;
    }
    __syncthreads();
    Pair ra = scratch[0], rb = scratch[kWarps];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) {
        if (pair_less(scratch[w], ra)) ra = scratch[w];
        if (pair_less(scratch[kWarps + w], rb)) rb = scratch[kWarps + w];
    }
    __syncthreads();
    a = ra;
    b = rb;
}
__device__ __forceinline__ void block_min_rb2(RowBest& a, RowBest& b, RowBest* scratch) {
    a = warp_min_rb(a);
    b = warp_min_rb(b);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        scratch[warp] = a;
        scratch[kWarps + warp] = b;
    }
    __syncthreads();
    // lanes 0..7 combine the per-warp minima of a, lanes 8..15 those of b
    RowBest r = lane < 2 * kWarps ? scratch[lane] : rb_none();
#pragma unroll
    for (int o = kWarps / 2; o > 0; o >>= 1) {
        const double d = __shfl_xor_sync(0xffffffffu, r.d, o);
        const int j = __shfl_xor_sync(0xffffffffu, r.j, o);
        if (d < r.d || (d == r.d && j < r.j)) { r.d = d; r.j = j; }
    }
    a.d = __shfl_sync(0xffffffffu, r.d, 0);
    a.j = __shfl_sync(0xffffffffu, r.j, 0);
    b.d = __shfl_sync(0xffffffffu, r.d, kWarps);
    b.j = __shfl_sync(0xffffffffu, r.j, kWarps);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Thread-block-cluster helpers (barrier.cluster + DSMEM)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// Full cluster barrier; release/acquire orders global + shared writes at cluster scope.
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of `p` (this CTA's smem) in CTA `rank`'s shared window, as a 32-bit
// shared::cluster address.
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, unsigned rank) {
    uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
    return remote;
}
__device__ __forceinline__ void dsmem_st_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t dsmem_ld_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

// ---------------------------------------------------------------------------
// Bulk async copy (TMA 1D) + mbarrier helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// One arrival that also raises the barrier's expected transaction bytes.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> this CTA's shared memory, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// Order this thread's generic-proxy global writes before later async-proxy reads.
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_shared() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace rhseg
