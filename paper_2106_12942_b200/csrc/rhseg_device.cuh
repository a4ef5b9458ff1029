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

constexpr int kThreads = 256;           // CTA size of every section kernel
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
