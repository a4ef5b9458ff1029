// hseg_kernels.cu -- the HSEG region-growing hot path on sm_100a.
//
// Reference semantics being replaced (rhseg, read-only at /root/reference/pkg/src):
//   engine.py:309-342  hseg_step   (snapshot -> adjacent scan -> spectral scan -> rule -> merge)
//   engine.py:345-371  hseg_run    (loop while live_count > target)
//   _kernels.py:31-115 scan_adjacent / scan_nonadjacent (per-row best partner, fp64)
//   graph.py:229-264   merge_regions (smaller id survives, sums add, adjacency union)
//
// B200 design (not a translation): the reference rebuilds both best-pair tables from
// scratch every step, O(R^2 B). Here every section keeps, resident in HBM/L2,
//   * an exact fp64 dissimilarity matrix D (all live pairs when w > 0, adjacent pairs
//     when w = 0), filled once by the tiled all-pairs kernel `dinit_dense_kernel`;
//   * per-row cached best partners for both stages (shared memory of the owning CTA).
// A merge (a, b) only changes pairs that touch a or b, so each step recomputes the
// single row a (R x B fp64 ops, bit-identical to the reference's op order), offers
// (d(i, a), a) to every row i, and rescans from D only the rows whose cached partner
// was a or b. Because the per-row caches always equal the reference's per-row table
// entries and the global pick is the same lexicographic (d, min id, max id) minimum,
// the merge sequence, dissimilarities and labels are bit-identical to hseg_run.
//
// One thread-block cluster (C CTAs, 1 <= C <= 16) owns one section and loops over all
// of its merges without returning to the host: CTA r owns rows [r*Rs, (r+1)*Rs). The
// single cross-CTA exchange per step is a 64-byte slot per CTA read through DSMEM after
// one barrier.cluster (double-buffered by step parity).
//
// APO variant (the default for w > 0, BSMSE/Euclidean, one CTA per section): row a is
// not recomputed from the means at all. D rows a and b bound every d(a', j) through the
// parallelogram identity (see "APO" below), so D entries and row caches may hold
// rigorous intervals; exact values are formed only where a comparison needs them, and
// the log's values after the loop. Same merge sequence, far fewer bytes per step.
#include <cuda_runtime.h>

#include <cstdlib>

#include <type_traits>

#include "rhseg_batch.h"
#include "rhseg_device.cuh"
#include "apo_device.cuh"

namespace rhseg {

#ifndef RHSEG_DINIT_FMA
#define RHSEG_DINIT_FMA 1  // APO sections: fused-multiply-add all-pairs init into intervals
#endif

// ===========================================================================
// 1. All-pairs D initialisation (the spectral-clustering all-pairs stage).
//    64x64 pair tiles, 256 threads, 4x4 register blocking, bands staged through
//    shared memory in ascending chunks (per-pair accumulation stays sequential in
//    b, so blocking never changes a bit). FP64-pipe bound: 3 DP ops per pair-band.
// ===========================================================================
constexpr int kTile = 64;
constexpr int kKB = 16;

// IV (APO sections, BSMSE/Euclidean): the per-band step is fl(a - b) then one fused
// multiply-add -- 2 FP64 ops instead of 3 -- and D receives an interval around the
// reference's value instead of the value itself. Both sums accumulate the same rounded
// differences t_b: s_ref = sum t_b^2 (1 + th), s_fma = sum t_b^2 (1 + th'), |th|, |th'| <=
// (B + 1) u (nonnegative terms), so d_ref lies within (B + 4) u of the d formed from s_fma;
// the interval is twice that. The loop treats D entries as intervals anyway (exact values
// only where a comparison needs them), so the merge sequence is unchanged.
//
// GRAM (RHSEG_DINIT_GRAM, the default for IV): ||m_i - m_j||^2 = n_i + n_j - 2 <m_i, m_j>
// with n = ||m||^2 -- ONE fused multiply-add per pair-band (half the FP64 instructions).
// Rigorous bound (u = 2^-53, FMA-accumulated sums of length B, gamma_B = B u / (1 - B u)):
//   |g^ - g| <= gamma_B sum |m_ik m_jk| <= gamma_B (n_i + n_j) / 2,  |n^ - n| <= gamma_B n,
//   S = fl(n^_i + n^_j), T^ = fl(S - 2 g^):  |T^ - T| <= (2 gamma_B + u) S + u |T^|,
// taken twice over: T in [T^ - eT, T^ + eT], eT = (4B + 16) u S + 4 u |T^|. The reference
// value then satisfies d_ref^2 = C T (1 + eps), |eps| <= (B + 8) u (apo_device.cuh), so
// d_ref lies in [d(T_lo) (1 - rho), d(T_hi) (1 + rho)], rho = 2 (B + 8) u (+ the rounding of
// d itself). The cancellation makes these intervals ~ (n_i + n_j) / T wider than the
// difference form's -- ~1e-9 relative on the synthetic cubes, far below what the loop's
// comparisons resolve; a pair whose lower bound reaches 0 (near-identical means) is
// evaluated exactly here.
#ifndef RHSEG_DINIT_GRAM
#define RHSEG_DINIT_GRAM 0  // measured: init 83 -> 88 ms (4x4 blocking turns shared-memory bound) and the loop 376 -> 677 ms (1e-9-wide intervals: 11x more exact pairs); off
#endif
constexpr int kDT = 256;  // dinit_dense_kernel's CTA: a 16x16 thread grid over a 64x64 tile
template <int M, bool IV = false>
__global__ void __launch_bounds__(kDT) dinit_dense_kernel(SectionBatch bt) {
    constexpr bool GRAM = IV && RHSEG_DINIT_GRAM;
    const int sec = bt.sec0 + blockIdx.y;
    const int R0 = bt.R0[sec];
    const int nt = (R0 + kTile - 1) / kTile;
    int t = blockIdx.x;
    if (t >= nt * (nt + 1) / 2) return;
    int ti = 0;
    while (t >= nt - ti) { t -= nt - ti; ++ti; }
    const int tj = ti + t;
    const int i0 = ti * kTile, j0 = tj * kTile;
    const int B = bt.B, Rp = bt.Rp;
    const double* __restrict__ mu = bt.mu + sec * bt.mu_stride();
    double* __restrict__ D = bt.D + (sec - bt.sec0) * bt.d_stride();
    const uint32_t* __restrict__ cnt = bt.count + (size_t)sec * Rp;
    const double* __restrict__ n2 = M == kSam ? bt.nrm2 + (size_t)sec * Rp : nullptr;

    // band staging: two buffers of (sA, sB) chunks filled by cp.async while the other
    // is consumed (double buffering); the transpose tile sT aliases the staging area
    // and is only touched after the last chunk's trailing __syncthreads()
    constexpr int kStage = 2 * kKB * kTile;  // doubles per buffer (A then B)
    __shared__ __align__(16) double smraw[(2 * kStage > kTile * (kTile + 1)) ? 2 * kStage : kTile * (kTile + 1)];
    __shared__ double snorm[2 * kTile];  // GRAM: ||m||^2 of the tile's rows, then columns
    double nacc = 0.0;                  // GRAM: threads < 128 accumulate one norm each
    double (*sT)[kTile + 1] = reinterpret_cast<double (*)[kTile + 1]>(smraw);
    // thread (tx, ty) owns rows i0 + 4 ty + p and columns j0 + 4 tx + q: both operand
    // quads are contiguous in shared memory (two 16-byte loads each)
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;

    // one chunk = kKB bands x 64 rows of each operand = 2 x kKB x 32 16-byte pieces;
    // bands past B are zero-filled (src-size 0): +0.0 to every accumulator, an identity
    auto stage = [&](int k0, int buf) {
        double* dst = smraw + buf * kStage;
        for (int e = threadIdx.x; e < 2 * kKB * (kTile / 2); e += kDT) {
            const int op = e / (kKB * (kTile / 2)), r = e % (kKB * (kTile / 2));
            const int kk = r / (kTile / 2), c = r % (kTile / 2);
            const int k = k0 + kk;
            const double* src = mu + (size_t)min(k, B - 1) * Rp + (op ? j0 : i0) + 2 * c;
            const uint32_t d = smem_u32(dst + op * kKB * kTile + kk * kTile + 2 * c);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(k < B ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int nchunk = (B + kKB - 1) / kKB;
    stage(0, 0);
    for (int ch = 0; ch < nchunk; ++ch) {
        if (ch + 1 < nchunk) {
            stage((ch + 1) * kKB, (ch + 1) & 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double (*sA)[kTile] = reinterpret_cast<const double (*)[kTile]>(smraw + (ch & 1) * kStage);
        const double (*sB)[kTile] = reinterpret_cast<const double (*)[kTile]>(smraw + (ch & 1) * kStage + kKB * kTile);
#pragma unroll
        for (int kk = 0; kk < kKB; ++kk) {
            const double2 a01 = *reinterpret_cast<const double2*>(&sA[kk][4 * ty]);
            const double2 a23 = *reinterpret_cast<const double2*>(&sA[kk][4 * ty + 2]);
            const double2 b01 = *reinterpret_cast<const double2*>(&sB[kk][4 * tx]);
            const double2 b23 = *reinterpret_cast<const double2*>(&sB[kk][4 * tx + 2]);
            const double a[4] = {a01.x, a01.y, a23.x, a23.y};
            const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (GRAM) {
                        acc[p][q] = __fma_rn(a[p], b[q], acc[p][q]);
                    } else if (IV) {
                        const double t = __dsub_rn(a[p], b[q]);
                        acc[p][q] = __fma_rn(t, t, acc[p][q]);
                    } else {
                        acc[p][q] = acc_step<M>(acc[p][q], a[p], b[q]);
                    }
                }
        }
        if (GRAM && threadIdx.x < 2 * kTile) {
            const int r = threadIdx.x & (kTile - 1);
            const double (*sX)[kTile] = threadIdx.x < kTile ? sA : sB;
#pragma unroll
            for (int kk = 0; kk < kKB; ++kk) nacc = __fma_rn(sX[kk][r], sX[kk][r], nacc);
        }
        __syncthreads();  // buffer ch & 1 is refilled by the next iteration's stage()
    }
    if (GRAM) {
        if (threadIdx.x < 2 * kTile) snorm[threadIdx.x] = nacc;
        __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int i = i0 + 4 * ty + p;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = j0 + 4 * tx + q;
            double d = 0.0;
            if (GRAM && i < R0 && j < R0) {
                constexpr double u = 1.1102230246251565e-16;
                const double S = __dadd_rn(snorm[4 * ty + p], snorm[kTile + 4 * tx + q]);
                const double T = __dsub_rn(S, 2.0 * acc[p][q]);
                const double eT = __dadd_ru(__dmul_ru(S, (4.0 * bt.B + 16.0) * u), __dmul_ru(fabs(T), 4.0 * u));
                const double Tlo = fmax(0.0, __dsub_rd(T, eT)), Thi = __dadd_ru(T, eT);
                const double ci = (double)cnt[i], cj = (double)cnt[j];
                const double rho = 2.0 * (bt.B + 8) * u;
                const double lo = __dmul_rd(pair_finish<M>(ci, cj, Tlo, 0.0, 0.0), __dsub_rd(1.0, rho));
                const double hi = __dmul_ru(pair_finish<M>(ci, cj, Thi, 0.0, 0.0), __dadd_ru(1.0, rho));
                if (i == j) {
                    d = 0.0;  // (never read: rows skip their own column)
                } else if (!d_pack_interval(lo, hi, d)) {
                    // (near-)identical means: the reference's exact value (rare)
                    double sx = 0.0;
                    for (int k = 0; k < B; ++k) sx = acc_step<M>(sx, mu[(size_t)k * Rp + i], mu[(size_t)k * Rp + j]);
                    d = pair_finish<M>(ci, cj, sx, 0.0, 0.0);
                }
                D[(size_t)i * Rp + j] = d;
            } else if (i < R0 && j < R0) {
                d = pair_finish<M>((double)cnt[i], (double)cnt[j], acc[p][q], M == kSam ? n2[i] : 0.0,
                                   M == kSam ? n2[j] : 0.0);
                if (IV && d > 0.0) {
                    const double rho = 2.0 * (bt.B + 4) * 1.1102230246251565e-16;
                    double v;
                    if (d_pack_interval(__dmul_rd(d, __dsub_rd(1.0, rho)), __dmul_ru(d, __dadd_ru(1.0, rho)), v)) d = v;
                }
                D[(size_t)i * Rp + j] = d;
            }
            sT[4 * ty + p][4 * tx + q] = d;
        }
    }
    if (ti == tj) return;  // diagonal tile already holds both orders (d is bitwise symmetric)
    __syncthreads();
    for (int e = threadIdx.x; e < kTile * kTile; e += kDT) {
        const int r = e / kTile, c = e % kTile;  // output row j0+r, column i0+c
        if (j0 + r < R0 && i0 + c < R0) D[(size_t)(j0 + r) * Rp + i0 + c] = sT[c][r];
    }
}

// w = 0: only adjacent pairs are ever read (engine.py:326 skips the spectral stage),
// so D is filled on the adjacency graph only. One thread per row.
template <int M>
__global__ void __launch_bounds__(kThreads) dinit_sparse_kernel(SectionBatch bt) {
    const int sec = bt.sec0 + blockIdx.y;
    const int R0 = bt.R0[sec];
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= R0) return;
    const int B = bt.B, Rp = bt.Rp, W = bt.W;
    const uint32_t* cnt = bt.count + (size_t)sec * Rp;
    if (cnt[i] == 0u) return;
    const double* mu = bt.mu + sec * bt.mu_stride();
    double* D = bt.D + (sec - bt.sec0) * bt.d_stride();
    const uint32_t* arow = bt.adj + (size_t)sec * bt.C * bt.adj_copy() + (size_t)i * W;
    for (int w = (i + 1) >> 5; w < W; ++w) {
        uint32_t bits = arow[w];
        while (bits) {
            const int j = (w << 5) + __ffs(bits) - 1;
            bits &= bits - 1;
            if (j <= i) continue;
            double s = 0.0;
            for (int k = 0; k < B; ++k) s = acc_step<M>(s, mu[(size_t)k * Rp + i], mu[(size_t)k * Rp + j]);
            const double* n2 = bt.nrm2 + (size_t)sec * Rp;
            const double d = pair_finish<M>((double)cnt[i], (double)cnt[j], s, M == kSam ? n2[i] : 0.0,
                                            M == kSam ? n2[j] : 0.0);
            D[(size_t)i * Rp + j] = d;
            D[(size_t)j * Rp + i] = d;
        }
    }
}

// APO sections' all-pairs init (IV: fl(a - b) then one DFMA per pair-band, D receives the
// interval of dinit_dense_kernel<M, true>, bit for bit): 64x64 pair tiles on 128 threads with
// 8x4 register blocking, so each band step issues 6 shared 16-byte loads per 64 FP64
// instructions (the 4x4 layout: 4 per 32, and the FP64 pipe sat at 72%).
#ifndef RHSEG_DINIT_84
#define RHSEG_DINIT_84 1
#endif
constexpr int kDiThreads = 128;
template <int M>
__global__ void __launch_bounds__(kDiThreads) dinit_iv84_kernel(SectionBatch bt) {
    const int sec = bt.sec0 + blockIdx.y;
    const int R0 = bt.R0[sec];
    const int nt = (R0 + kTile - 1) / kTile;
    int t = blockIdx.x;
    if (t >= nt * (nt + 1) / 2) return;
    int ti = 0;
    while (t >= nt - ti) { t -= nt - ti; ++ti; }
    const int tj = ti + t;
    const int i0 = ti * kTile, j0 = tj * kTile;
    const int B = bt.B, Rp = bt.Rp;
    const double* __restrict__ mu = bt.mu + sec * bt.mu_stride();
    double* __restrict__ D = bt.D + (sec - bt.sec0) * bt.d_stride();
    const uint32_t* __restrict__ cnt = bt.count + (size_t)sec * Rp;
    constexpr int kStage = 2 * kKB * kTile;
    __shared__ __align__(16) double smraw[(2 * kStage > kTile * (kTile + 1)) ? 2 * kStage : kTile * (kTile + 1)];
    double (*sT)[kTile + 1] = reinterpret_cast<double (*)[kTile + 1]>(smraw);
    // thread (tx, ty): rows i0 + 8 ty + p (p < 8), columns j0 + 4 tx + q (q < 4)
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[8][4];
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
    auto stage = [&](int k0, int buf) {
        double* dst = smraw + buf * kStage;
        for (int e = threadIdx.x; e < 2 * kKB * (kTile / 2); e += kDiThreads) {
            const int op = e / (kKB * (kTile / 2)), r = e % (kKB * (kTile / 2));
            const int kk = r / (kTile / 2), c = r % (kTile / 2);
            const int k = k0 + kk;
            const double* src = mu + (size_t)min(k, B - 1) * Rp + (op ? j0 : i0) + 2 * c;
            const uint32_t d = smem_u32(dst + op * kKB * kTile + kk * kTile + 2 * c);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(k < B ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int nchunk = (B + kKB - 1) / kKB;
    stage(0, 0);
    for (int ch = 0; ch < nchunk; ++ch) {
        if (ch + 1 < nchunk) {
            stage((ch + 1) * kKB, (ch + 1) & 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double (*sA)[kTile] = reinterpret_cast<const double (*)[kTile]>(smraw + (ch & 1) * kStage);
        const double (*sB)[kTile] = reinterpret_cast<const double (*)[kTile]>(smraw + (ch & 1) * kStage + kKB * kTile);
#pragma unroll
        for (int kk = 0; kk < kKB; ++kk) {
            double a[8], b[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const double2 v = *reinterpret_cast<const double2*>(&sA[kk][8 * ty + 2 * h]);
                a[2 * h] = v.x;
                a[2 * h + 1] = v.y;
            }
            const double2 b01 = *reinterpret_cast<const double2*>(&sB[kk][4 * tx]);
            const double2 b23 = *reinterpret_cast<const double2*>(&sB[kk][4 * tx + 2]);
            b[0] = b01.x; b[1] = b01.y; b[2] = b23.x; b[3] = b23.y;
#pragma unroll
            for (int p = 0; p < 8; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double d = __dsub_rn(a[p], b[q]);
                    acc[p][q] = __fma_rn(d, d, acc[p][q]);
                }
        }
        __syncthreads();
    }
    const double rho = 2.0 * (bt.B + 4) * 1.1102230246251565e-16;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const int i = i0 + 8 * ty + p;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = j0 + 4 * tx + q;
            double d = 0.0;
            if (i < R0 && j < R0) {
                d = pair_finish<M>((double)cnt[i], (double)cnt[j], acc[p][q], 0.0, 0.0);
                if (d > 0.0) {
                    double v;
                    if (d_pack_interval(__dmul_rd(d, __dsub_rd(1.0, rho)), __dmul_ru(d, __dadd_ru(1.0, rho)), v)) d = v;
                }
                D[(size_t)i * Rp + j] = d;
            }
            sT[8 * ty + p][4 * tx + q] = d;
        }
    }
    if (ti == tj) return;  // diagonal tile already holds both orders (d is bitwise symmetric)
    __syncthreads();
    for (int e = threadIdx.x; e < kTile * kTile; e += kDiThreads) {
        const int r = e / kTile, c = e % kTile;  // output row j0+r, column i0+c
        if (j0 + r < R0 && i0 + c < R0) D[(size_t)(j0 + r) * Rp + i0 + c] = sT[c][r];
    }
}

void launch_dinit(const SectionBatch& b, int nrun, int R0max, cudaStream_t st) {
    if (nrun == 0 || R0max == 0) return;
    if (b.spec) {
        const int nt = (R0max + kTile - 1) / kTile;
        dim3 grid(nt * (nt + 1) / 2, nrun);
        if (b.measure == kSam) dinit_dense_kernel<kSam><<<grid, kDT, 0, st>>>(b);
        else if (b.measure == kEuclid && b.apo && RHSEG_DINIT_FMA && RHSEG_DINIT_84 && !RHSEG_DINIT_GRAM)
            dinit_iv84_kernel<kEuclid><<<grid, kDiThreads, 0, st>>>(b);
        else if (b.apo && RHSEG_DINIT_FMA && RHSEG_DINIT_84 && !RHSEG_DINIT_GRAM && b.measure == kBsmse)
            dinit_iv84_kernel<kBsmse><<<grid, kDiThreads, 0, st>>>(b);
        else if (b.measure == kEuclid && b.apo && RHSEG_DINIT_FMA) dinit_dense_kernel<kEuclid, true><<<grid, kDT, 0, st>>>(b);
        else if (b.measure == kEuclid) dinit_dense_kernel<kEuclid><<<grid, kDT, 0, st>>>(b);
        else if (b.apo && RHSEG_DINIT_FMA) dinit_dense_kernel<kBsmse, true><<<grid, kDT, 0, st>>>(b);
        else dinit_dense_kernel<kBsmse><<<grid, kDT, 0, st>>>(b);
    } else {
        dim3 grid((R0max + kThreads - 1) / kThreads, nrun);
        if (b.measure == kSam) dinit_sparse_kernel<kSam><<<grid, kThreads, 0, st>>>(b);
        else if (b.measure == kEuclid) dinit_sparse_kernel<kEuclid><<<grid, kThreads, 0, st>>>(b);
        else dinit_sparse_kernel<kBsmse><<<grid, kThreads, 0, st>>>(b);
    }
}

// ===========================================================================
// 2. Persistent per-section merge loop.
// ===========================================================================
struct Slot {
    Pair selA, selN;   // this CTA's best adjacent / non-adjacent pair over its own rows
    RowBest rpA, rpN;  // this CTA's partial best for row a_prev over its own columns
};
static_assert(sizeof(Slot) == 64, "slot is copied as 16 u32 words");

// Streaming ring for the spectral row-a pass (w > 0): the live regions' mean
// columns of one CTA are streamed band-chunk by band-chunk from HBM with bulk
// async copies (TMA 1D) into a ring of nstages x stage_bytes of shared memory.
// Measured on C4 (tools/ab_variants.py, profiles/r01_loop_variants.md): 2 x 32 KB
// stages with 2 CTAs/SM beat 4 x 16 KB (-12%), 8 x 8 KB, 3 CTAs/SM with 2 x 16 KB,
// per-warp empty barriers, L2 bulk prefetch and direct (unstaged) loads; the
// per-stage block barrier + wait overhead, not the fetch latency, sets the pace.
#ifndef RHSEG_APO_TOP2
#define RHSEG_APO_TOP2 0  // APO rows keep their two best partners: C4 7.3 -> 4.4 rescans per step but each costs 1.8x (loop 359 -> 425 ms), off
#endif
#ifndef RHSEG_APO_OVERLAP
#define RHSEG_APO_OVERLAP 0  // 1: row a' intervals by each warp right after its rescans (measured slower on C4)
#endif
#ifndef RHSEG_APO
#define RHSEG_APO 1  // bound row a' from D (no mean stream) where possible; host may still disable
#endif
#ifndef RHSEG_COMPACT_K
#define RHSEG_COMPACT_K 16  // compaction threshold: holes^2 >= K * S (K=16: C4 loop 874 -> 864 ms)
#endif
#ifndef RHSEG_RESCAN_PREFETCH
#define RHSEG_RESCAN_PREFETCH 1
#endif
#ifndef RHSEG_RESCAN_STAGE
#define RHSEG_RESCAN_STAGE 0  // APO: first N rescans' D rows bulk-copied to shared memory (C4 loop 319 -> 354/357/367 ms for N = 1/2/3: off)
#endif
#ifndef RHSEG_APO_FUSE_OFFERS
#define RHSEG_APO_FUSE_OFFERS 1  // APO: offers of d(a', j) made in the row-a' interval pass (C4 371.7 -> 369.8 ms)
#endif
constexpr int kRsStage = RHSEG_RESCAN_STAGE;
constexpr bool kFuseOffers = RHSEG_APO_FUSE_OFFERS && !RHSEG_APO_TOP2;
#ifndef RHSEG_RESCAN_HI
#define RHSEG_RESCAN_HI 0  // APO rescans on the high words of D, 2U loads in flight (C4 372.6 -> 411.7 ms: off)
#endif
#ifndef RHSEG_RESCAN_HI_KMAX
#define RHSEG_RESCAN_HI_KMAX 24  // ... while every interval code in D is at most this (else full doubles)
#endif
#ifndef RHSEG_RESCAN_LPT
#define RHSEG_RESCAN_LPT 1  // APO: rescans claimed longest first (full walks, then adjacent-only gathers)
#endif
#ifndef RHSEG_STAGES
#define RHSEG_STAGES 2
#endif
#ifndef RHSEG_STAGE_KB
#define RHSEG_STAGE_KB 32
#endif
constexpr int kMaxStages = 4;  // ring depth for levels with at most one CTA per SM
constexpr int kStageBytes = RHSEG_STAGE_KB * 1024;
// SAM keeps the two best partners per row (TOP2 below) and pays for those
// arrays with a smaller stream ring, so two CTAs still fit one SM.
constexpr int kStageBytesTop2 = 20 * 1024;
constexpr int kMaxSlots = 2048;  // own columns per CTA (cluster grows beyond)
constexpr int kNbList = 256;     // b's neighbours re-pointed in parallel per merge

// one slice of a split APO rescan: per stage the two smallest 32-bit keys, the
// winner's column and D value, and the widest interval code
struct RsSlice {
    unsigned a1, a2, n1, n2;
    int ja, jn, km, pad;
    double va, vn;
};
struct LoopSmem {
    size_t xstg, rbuf, rsp, livew, ver, apk, sdv, slot, rslot, pscr, rscr, spart, misc, rpart, bars, mua, bAd, bNd, bAj, bNj, inv, cnt, col, slot_of, bAd2, bNd2,
        bAj2, bNj2, cx, nbl, sra, ring, total;
};
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline int own_rows(int R, int C) { return (((R + C - 1) / C) + 1) & ~1; }
__host__ __device__ inline LoopSmem loop_smem_layout(int Rp, int C, int B, bool spec, bool top2,
                                                     int stage_bytes, int nstages) {
    const size_t Rs = (size_t)own_rows(Rp, C);
    top2 = top2 || (spec && nstages == 0 && RHSEG_APO_TOP2);  // APO: two partners per row
    LoopSmem L;
    size_t o = 0;
    L.slot = o;  o += 2 * sizeof(Slot);
    L.rslot = o; o += 2 * kMaxCluster * sizeof(Slot);  // [step parity][source CTA]
    L.pscr = o;  o += 2 * kWarps * sizeof(Pair);
    L.rscr = o;  o += 2 * kWarps * sizeof(RowBest);
    L.spart = o; o += kWarps * sizeof(RowBest);
    L.misc = o;  o += 64;
    L.rpart = o; o += 2 * sizeof(RowBest);
    L.bars = o;  o += kMaxStages * 8;  // full[nstages]
    L.bAd = o;   o = align16(o + Rs * 8);
    L.bNd = o;   o = align16(o + Rs * 8);
    L.bAj = o;   o = align16(o + Rs * 4);
    L.bNj = o;   o = align16(o + Rs * 4);
    L.inv = o;   o = align16(o + Rs * 4);
    L.cnt = o;   o = align16(o + (size_t)Rp * 4);
    L.col = o;   o = align16(o + (spec ? Rs * 2 : 0));      // int16: region ids < 16384
    L.slot_of = o; o = align16(o + (spec ? Rs * 2 : 0));
    L.bAd2 = o;  o = align16(o + (top2 ? Rs * 8 : 0));
    L.bNd2 = o;  o = align16(o + (top2 ? Rs * 8 : 0));
    L.bAj2 = o;  o = align16(o + (top2 ? Rs * 4 : 0));
    L.bNj2 = o;  o = align16(o + (top2 ? Rs * 4 : 0));
    L.cx = o;    o = align16(o + (top2 ? Rs : 0));
    L.nbl = o;   o = align16(o + kNbList * 2);  // b's neighbours during a merge
    L.sra = o;   o = align16(o + (size_t)(Rp / 32) * 4);  // a's new adjacency row (row-a pass)
    L.sdv = o;   o = align16(o + (spec && nstages == 0 ? Rs * 16 : 0));  // APO: per-slot D values / bounds
    L.apk = o;   o += 64;                                                  // APO: argmin keys, rule scratch
    L.ver = o;   o = align16(o + (spec && nstages == 0 ? (size_t)Rp * 2 : 0));  // APO: mean version per region
    L.livew = o; o = align16(o + (spec && nstages == 0 ? (size_t)(Rp / 32) * 4 : 0));  // APO: live-region bitset
    L.rsp = o;   o = align16(o + (spec && nstages == 0 ? 2 * kWarps * sizeof(RsSlice) : 0));  // APO: rescan slices
    o = (o + 127) & ~size_t(127);
    L.rbuf = o;  o += spec && nstages == 0 ? (size_t)kRsStage * Rp * 8 : 0;  // APO: staged D rows of rescans
    // the band-sized arrays last: with a compile-time capacity every offset above folds
    L.mua = o;   o = align16(o + (size_t)B * 8);
    L.xstg = o;  o = align16(o + (spec && nstages == 0 ? (size_t)kWarps * B * 8 : 0));  // APO: exact-sum staging rows
    o = (o + 127) & ~size_t(127);
    L.ring = o;
    o += spec && nstages > 0 ? (size_t)nstages * stage_bytes + kThreads * 8 : 0;  // (APO: no ring)
    L.total = o;
    return L;
}
__host__ __device__ inline bool use_top2(bool spec, int C, int measure) { return spec && C == 1 && measure == kSam; }
__host__ __device__ inline bool apo_capable(bool spec, int C, int measure) {
    return RHSEG_APO && spec && C == 1 && measure != kSam;
}
int hseg_loop_stage_bytes(bool spec, int C, int measure) {
    return use_top2(spec, C, measure) ? kStageBytesTop2 : kStageBytes;
}
size_t hseg_loop_smem(int Rp, int C, int B, bool spec, int measure, int stage_bytes, int nstages) {
    return loop_smem_layout(Rp, C, B, spec, use_top2(spec, C, measure), stage_bytes, nstages)
        .total;
}
int hseg_loop_max_stages() { return kMaxStages; }
int hseg_loop_default_stages() { return RHSEG_STAGES; }
bool hseg_apo_capable(bool spec, int C, int measure) { return apo_capable(spec, C, measure); }
int hseg_loop_max_rows() { return kMaxSlots; }

__device__ __forceinline__ void cache_offer(double& cd, int& cj, double d, int j) {
    if (d < kInf && (d < cd || (d == cd && j < cj))) { cd = d; cj = j; }
}

// ---- TOP2 (SAM): the two smallest (d, j) candidates of a row and stage -------
// A row's list holds its m <= 2 lexicographically smallest candidates; the
// "complete" bit says the list holds every candidate. A merge (a, b) removes a
// and b from every list and offers (d(i, a), a); only a list left empty and
// incomplete needs a rescan from D. Equivalent to the reference's per-row best
// (its head) at every step, with far fewer rescans when many rows share a best
// partner (SAM: a merged region becomes the nearest angle of most rows).
struct Top2 {
    double d0;
    int j0;
    double d1;
    int j1;
    int n;  // candidates seen, capped at 3
};
__device__ __forceinline__ Top2 t2_none() { return Top2{kInf, kNoJ, kInf, kNoJ, 0}; }
__device__ __forceinline__ void t2_put(Top2& t, double d, int j) {
    if (!(d < kInf)) return;
    if (d < t.d0 || (d == t.d0 && j < t.j0)) {
        t.d1 = t.d0; t.j1 = t.j0; t.d0 = d; t.j0 = j;
    } else if (d < t.d1 || (d == t.d1 && j < t.j1)) {
        t.d1 = d; t.j1 = j;
    }
}
__device__ __forceinline__ void t2_offer(Top2& t, double d, int j) {
    if (!(d < kInf)) return;
    t.n = min(t.n + 1, 3);
    t2_put(t, d, j);
}
__device__ __forceinline__ Top2 warp_top2(Top2 t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double d0 = __shfl_xor_sync(0xffffffffu, t.d0, o), d1 = __shfl_xor_sync(0xffffffffu, t.d1, o);
        const int j0 = __shfl_xor_sync(0xffffffffu, t.j0, o), j1 = __shfl_xor_sync(0xffffffffu, t.j1, o);
        const int n = __shfl_xor_sync(0xffffffffu, t.n, o);
        t2_put(t, d0, j0);
        t2_put(t, d1, j1);
        t.n = min(t.n + n, 3);
    }
    return t;
}
__device__ __forceinline__ void l2_remove(double& d0, int& j0, double& d1, int& j1, int x) {
    if (j1 == x) { d1 = kInf; j1 = -1; }
    if (j0 == x) { d0 = d1; j0 = j1; d1 = kInf; j1 = -1; }
}
__device__ __forceinline__ void l2_offer(double& d0, int& j0, double& d1, int& j1, uint8_t& cbits, uint8_t bit,
                                         double d, int j) {
    if (!(d < kInf)) return;
    const bool complete = (cbits & bit) != 0;
    if (j0 < 0) {
        if (complete) { d0 = d; j0 = j; }
        return;
    }
    const bool lt0 = d < d0 || (d == d0 && j < j0);
    if (j1 < 0) {
        if (lt0) { d1 = d0; j1 = j0; d0 = d; j0 = j; }
        else if (complete) { d1 = d; j1 = j; }
        return;
    }
    if (lt0) { d1 = d0; j1 = j0; d0 = d; j0 = j; }
    else if (d < d1 || (d == d1 && j < j1)) { d1 = d; j1 = j; }
    cbits &= (uint8_t)~bit;  // a third candidate exists and is not stored
}
struct Top2Lists {
    double *bAd2, *bNd2;
    int *bAj2, *bNj2;
    uint8_t* cx;
};


// Epilogue for one column j of the row-a pass: D row/column update, offer
// (d, a) to row j's caches, mark rows whose cached partner died.
template <bool SPEC, int M, bool TOP2 = false>
__device__ __forceinline__ void rowa_col(int jq, bool valid, bool isadj, bool need, double s, double nn, int a,
                                         int b, int lo, int Rp, const uint32_t* cnt, double n2a,
                                         const double* __restrict__ n2, double* __restrict__ D,
                                         double* bAd, int* bAj, double* bNd, int* bNj, RowBest& pA, RowBest& pN,
                                         int* inv, int* ninv, Top2Lists t2 = Top2Lists{}) {
    if (!valid) return;
    double d = kInf;
    if (need) {
        d = pair_finish<M>(nn, (double)cnt[jq], s, n2a, M == kSam ? n2[jq] : 0.0);
        D[(size_t)jq * Rp + a] = d;
        D[(size_t)a * Rp + jq] = d;
        if (isadj) rb_offer(pA, d, jq);
        else rb_offer(pN, d, jq);
    }
    // rows whose cached partner was a or b were rescanned (a and b excluded)
    // before this pass, so every row just takes the offer of (d(j, a), a)
    const int r = jq - lo;
    if (TOP2) {
        if (isadj) l2_offer(bAd[r], bAj[r], t2.bAd2[r], t2.bAj2[r], t2.cx[r], 1, d, a);
        else l2_offer(bNd[r], bNj[r], t2.bNd2[r], t2.bNj2[r], t2.cx[r], 2, d, a);
        return;
    }
    if (isadj) cache_offer(bAd[r], bAj[r], d, a);
    else if (SPEC) cache_offer(bNd[r], bNj[r], d, a);
}

// Per-CTA streaming state of the spectral row-a pass (all threads hold the same
// values; only thread 0 issues copies).
struct StreamState {
    uint32_t issued;  // stages issued since the kernel started (ring position)
    int S;            // own compacted columns (ascending ids; holes = -1)
    int holes;
    int cur;          // which mean buffer (mu / mu2) holds the compacted columns
    int S2, KB, nst;  // current step's geometry
    uint32_t base;    // first stage of the current step
};

#ifndef RHSEG_MINBLOCKS
#define RHSEG_MINBLOCKS 2
#endif
#ifndef RHSEG_SPARSE_NUM  // APO rescans walk the live-column list when S / R0 < NUM / DEN
#define RHSEG_SPARSE_NUM 1
#define RHSEG_SPARSE_DEN 2
#endif
#ifndef RHSEG_APO_COMPACT  // APO: compact the live-column list when holes >= S / K
#define RHSEG_APO_COMPACT 8
#endif
#ifndef RHSEG_RESCAN_PIPE
#define RHSEG_RESCAN_PIPE 0  // APO rescans: software-pipelined row walk
#endif
#ifndef RHSEG_RESCAN_SPLIT
#define RHSEG_RESCAN_SPLIT 0  // APO: split the walks of a step with few rescans over idle warps (C4 loop 358 -> 376 ms: off)
#endif
#ifndef RHSEG_EXACT_STG
#define RHSEG_EXACT_STG 1  // APO exact sums: lane 0 adds staged terms (0: shuffle-fed chain in every lane)
#endif
#if RHSEG_EXACT_STG
#define RHSEG_WEXACT(...) warp_exact_stg<M>(__VA_ARGS__)
#else
#define RHSEG_WEXACT(mi, mj, ci, cj, B, lane, stg) warp_exact<M>(mi, mj, ci, cj, B, lane)
#endif
#ifndef RHSEG_AROW_REGS
#define RHSEG_AROW_REGS 0  // APO rescans: the row's adjacency words in registers, shuffled per word (C4 loop 343 -> 418 ms: off)
#endif
#ifndef RHSEG_RPC
#define RHSEG_RPC 1  // APO loop instantiated for compile-time capacities 1024 and 64
#endif
#ifndef RHSEG_KEY32
#define RHSEG_KEY32 1  // APO rescans on 32-bit keys with redux.sync (0: 64-bit keys, shuffle trees)
#endif
#ifndef RHSEG_N_NODEP
#define RHSEG_N_NODEP 1  // APO non-adjacent-only rescans: D loads independent of the adjacency words (C4 loop 311 -> 291.5 ms)
#endif
#ifndef RHSEG_ADJ_GATHER
#define RHSEG_ADJ_GATHER 1  // APO adjacent-only rescans: gather the adjacent columns' D entries only
#endif
#ifndef RHSEG_RESCAN_U
#define RHSEG_RESCAN_U 4  // APO rescans: D loads in flight per lane (C4 loop: 8 -> 427 ms, 4 -> 380, 2 -> 402, 1 -> 387)
#endif
#ifndef RHSEG_APO_MINBLOCKS
#define RHSEG_APO_MINBLOCKS 2
#endif
// RPC: the padded capacity as a compile-time constant (0 = bt.Rp at run time). The APO
// loop is instantiated for the capacities of the BASELINE levels (1024: 32x32 leaves, 64:
// every level above at t=16), so the shared-memory layout and the D / sums / adjacency
// strides fold to constants instead of being recomputed under register pressure.
template <bool CLUSTER, bool SPEC, int M, bool APO = false, int RPC = 0>
__global__ void __launch_bounds__(kThreads, APO ? RHSEG_APO_MINBLOCKS : RHSEG_MINBLOCKS) hseg_loop_kernel(SectionBatch bt) {
    extern __shared__ __align__(128) unsigned char smem[];
    const long long t_entry = clock64();
    const int C = CLUSTER ? bt.C : 1;
    const int rank = CLUSTER ? (int)cluster_rank() : 0;
    const int sec = bt.sec0 + (int)(blockIdx.x / C);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R0 = bt.R0[sec];
    const int B = bt.B, Rp = RPC ? RPC : bt.Rp, W = RPC ? RPC / 32 : bt.W;
    const int target = bt.target[sec];
    const int Rs = own_rows(R0, C);
    const int lo = min(R0, rank * Rs), hi = min(R0, lo + Rs);

    constexpr bool TOP2 = SPEC && !CLUSTER && M == kSam;
    static_assert(!APO || (SPEC && !CLUSTER && M != kSam), "APO: w > 0, one CTA, BSMSE/Euclidean");
    constexpr bool F32 = APO;  // interval-valued D entries and caches (resolved exactly on demand)
    // APO rows keep their two smallest candidates per stage with a "list holds every
    // candidate" bit (the SAM lists, on intervals): a merge removes a and b from every
    // list and only a list left empty and incomplete is rescanned
    constexpr bool T2A = APO && RHSEG_APO_TOP2;
    constexpr bool kLpt = APO && !T2A && RHSEG_RESCAN_LPT;  // (rescan claim order, see the claim loop)
    constexpr bool STREAM = SPEC && !APO;  // row a' from the streamed mean columns
    using SE = double;  // streamed element
    constexpr int ES = (int)sizeof(SE);
    const int SB = bt.stage_bytes;  // ring stage size and depth chosen by the host
    const int NS = bt.nstages;      // (deeper ring when the level has <= 1 CTA per SM)
    const LoopSmem L = loop_smem_layout(Rp, C, B, SPEC, TOP2, APO ? 0 : SB, APO ? 0 : NS);
    Slot* slot = reinterpret_cast<Slot*>(smem + L.slot);
    Slot* rslot = reinterpret_cast<Slot*>(smem + L.rslot);
    Pair* pscr = reinterpret_cast<Pair*>(smem + L.pscr);
    RowBest* rscr = reinterpret_cast<RowBest*>(smem + L.rscr);
    RowBest* spart = reinterpret_cast<RowBest*>(smem + L.spart);
    int* misc = reinterpret_cast<int*>(smem + L.misc);
    int& ninv = misc[0];
    int& sdE = misc[1];
    unsigned long long& sE0 = *reinterpret_cast<unsigned long long*>(misc + 2);
    int& sScan = misc[4];
    RowBest* rpart = reinterpret_cast<RowBest*>(smem + L.rpart);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);  // full: bulk bytes landed
    double* mua = reinterpret_cast<double*>(smem + L.mua);
    double* bAd = reinterpret_cast<double*>(smem + L.bAd);
    double* bNd = reinterpret_cast<double*>(smem + L.bNd);
    int* bAj = reinterpret_cast<int*>(smem + L.bAj);
    int* bNj = reinterpret_cast<int*>(smem + L.bNj);
    int* inv = reinterpret_cast<int*>(smem + L.inv);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L.cnt);
    short* col = reinterpret_cast<short*>(smem + L.col);
    short* slot_of = reinterpret_cast<short*>(smem + L.slot_of);
    // TOP2: second-best partner per row and stage + "list holds every candidate" bits
    double* bAd2 = reinterpret_cast<double*>(smem + L.bAd2);
    double* bNd2 = reinterpret_cast<double*>(smem + L.bNd2);
    int* bAj2 = reinterpret_cast<int*>(smem + L.bAj2);
    int* bNj2 = reinterpret_cast<int*>(smem + L.bNj2);
    uint8_t* cx = reinterpret_cast<uint8_t*>(smem + L.cx);
    unsigned short* nbl = reinterpret_cast<unsigned short*>(smem + L.nbl);
    uint32_t* sra = reinterpret_cast<uint32_t*>(smem + L.sra);
    int& nnb = misc[13];
    double* ring = reinterpret_cast<double*>(smem + L.ring);

    const size_t mus = (size_t)B * Rp;  // (bt.mu_stride() with the folded capacity)
    double* const mu0 = bt.mu + sec * mus;
    double* const mu1 = STREAM ? bt.mu2 + sec * mus : nullptr;
    SE* const sb0 = mu0;  // the streamed mean buffers (ping-pong)
    SE* const sb1 = mu1;
    // APO: region-major copy of the exact cached means [Rp][B] (in the mu2 allocation)
    // APO: versioned region-major means [2 Rp][B] (row i: initial mean of region i; row
    // R0 + t: the mean created by step t) -- the exact re-evaluations read them, and
    // the log's exact values are computed after the loop from (old a, b) versions
    double* const mr = APO ? bt.mu2 + 2 * sec * mus : nullptr;
    unsigned short* ver = reinterpret_cast<unsigned short*>(smem + L.ver);  // APO: region -> mr row
    uint32_t* livew = reinterpret_cast<uint32_t*>(smem + L.livew);          // APO: live regions
    RsSlice* rs_part = reinterpret_cast<RsSlice*>(smem + L.rsp);              // APO: rescan slices
    double* const xstg = reinterpret_cast<double*>(smem + L.xstg) + (size_t)warp * B;  // APO: this warp's staging row
    double* const rbuf = reinterpret_cast<double*>(smem + L.rbuf);  // APO: staged D rows of the first rescans
    uint32_t rbph = 0u;  // (uniform) parity each staged-row barrier completes next
    double* __restrict__ D = bt.D + (size_t)(sec - bt.sec0) * ((size_t)Rp * Rp);
    double* __restrict__ n2g = M == kSam ? bt.nrm2 + (size_t)sec * Rp : nullptr;
    double* __restrict__ sums = bt.sums + ((size_t)sec * C + rank) * ((size_t)Rp * B);
    uint32_t* __restrict__ adj = bt.adj + ((size_t)sec * C + rank) * ((size_t)Rp * W);

    // Rescan of one owned row from D (mask bit0: adjacent stage, bit1: non-adjacent
    // stage) -- the full-row search of _kernels.py restricted to rows whose cached
    // partner was merged away. Adjacent-only rescans walk the adjacency bitset;
    // non-adjacent ones stream the D row with 8 loads in flight per lane.
    StreamState ss{};
    int rs_exb = -1;  // APO: a column every rescan also skips (b while the merge runs beside them)
    auto rescan = [&](int i, int mask, int ex) {  // ex: column skipped (-1 = none)
        RowBest ba = rb_none(), bn = rb_none();
        if (cnt[i] != 0u) {
            const uint32_t* arow = adj + (size_t)i * W;
            const double* drow = D + (size_t)i * Rp;
            if (!(SPEC && (mask & 2))) {
                for (int w0 = 0; w0 < W; w0 += 32) {
                    const int w = w0 + lane;
                    uint32_t bits = w < W ? arow[w] : 0u;
                    while (bits) {
                        const int j = (w << 5) + __ffs(bits) - 1;
                        bits &= bits - 1;
                        if (j < R0 && j != ex && cnt[j] != 0u) rb_offer(ba, __ldcg(drow + j), j);
                    }
                }
            } else if (!CLUSTER) {
                // one CTA owns every column: walk the compacted live-column list
                // (ascending ids, holes = -1), 16 D loads in flight per lane
                constexpr int U = 16;
                for (int s0 = 0; s0 < ss.S; s0 += 32 * U) {
                    double dv[U];
                    int jv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int sl = s0 + 32 * u + lane;
                        const int j = sl < ss.S ? col[sl] : -1;
                        jv[u] = j;
                        dv[u] = j >= 0 ? __ldcs(drow + j) : kInf;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = jv[u];
                        if (j >= 0 && j != i && j != ex && j != rs_exb && cnt[j] != 0u) {
                            if ((arow[j >> 5] >> (j & 31)) & 1u) {
                                if (mask & 1) rb_offer(ba, dv[u], j);
                            } else {
                                rb_offer(bn, dv[u], j);
                            }
                        }
                    }
                }
            } else {
                for (int j0 = 0; j0 < R0; j0 += 256) {
                    double dv[8];
                    uint32_t wv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = j0 + 32 * u + lane;
                        const bool in = j < R0;
                        dv[u] = in ? __ldcs(drow + j) : kInf;
                        wv[u] = (j0 + 32 * u) < R0 ? arow[(j0 >> 5) + u] : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = j0 + 32 * u + lane;
                        if (j < R0 && j != i && j != ex && j != rs_exb && cnt[j] != 0u) {
                            if ((wv[u] >> lane) & 1u) {
                                if (mask & 1) rb_offer(ba, dv[u], j);
                            } else {
                                rb_offer(bn, dv[u], j);
                            }
                        }
                    }
                }
            }
        }
        ba = warp_min_rb(ba);
        if (SPEC) bn = warp_min_rb(bn);
        if (lane == 0) {
            const int r = i - lo;
            if (mask & 1) { bAd[r] = ba.d; bAj[r] = ba.j == kNoJ ? -1 : ba.j; }
            if (SPEC && (mask & 2)) { bNd[r] = bn.d; bNj[r] = bn.j == kNoJ ? -1 : bn.j; }
        }
    };

    // APO rescan: D rows hold exact values and intervals, and so may the cached best.
    // One pass finds, per stage, the smallest upper bound U and the two smallest
    // lower bounds: if the second lies above U, the entry with the smallest lower
    // bound is the row's minimum (cached as it is, interval or not); otherwise
    // a second pass takes the exact lexicographic minimum of every entry whose lower
    // bound reaches U (intervals evaluated by the warp and written back to D).
    struct Lo2 {
        double l1, v1, l2, u;
        int j1;
    };
    auto lo2_put = [](Lo2& x, double l, int j, double v) {
        if (l < x.l1 || (l == x.l1 && j < x.j1)) {
            x.l2 = x.l1;
            x.l1 = l; x.j1 = j; x.v1 = v;
        } else if (l < x.l2) {
            x.l2 = l;
        }
    };
    auto exact_pair = [&](int i, int j) {  // whole warp; lane 0 writes D back
        const long long t0 = clock64();
        const double d = RHSEG_WEXACT(mr + (size_t)ver[i] * B, mr + (size_t)ver[j] * B, (double)cnt[i],
                                           (double)cnt[j], B, lane, xstg);
        if (bt.prof && lane == 0) {
            atomicAdd(bt.prof + 11, 1ull);
            atomicAdd(bt.prof + 12, (unsigned long long)(clock64() - t0));
        }
        if (lane == 0) {
            D[(size_t)i * Rp + j] = d;
            D[(size_t)j * Rp + i] = d;
        }
        return d;
    };
    auto rescanf_full = [&](int i, int mask, int ex) {
        const uint32_t* arow = adj + (size_t)i * W;
        double* drow = D + (size_t)i * Rp;
        const bool live_i = cnt[i] != 0u;
        Lo2 xa{kInf, kInf, kInf, kInf, kNoJ}, xn{kInf, kInf, kInf, kInf, kNoJ};
        constexpr int U = 8;
        if (live_i) {
            // id-ordered walk, one bitset word per warp-iteration: lane l takes id
            // 32 w + l, whose liveness and adjacency bits come from two broadcast words,
            // and the D loads of a warp are one contiguous 256-byte row segment
            for (int w0 = 0; w0 < W; w0 += U) {
                double dv[U];
                uint32_t sel[U];  // bit0: candidate, bit1: adjacent
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int w = w0 + u;
                    const uint32_t lw = w < W ? livew[w] : 0u, aw = w < W ? arow[w] : 0u;
                    const int j = (w << 5) + lane;
                    const bool aj = (aw >> lane) & 1u;
                    const bool c = ((lw >> lane) & 1u) && j != i && j != ex && j != rs_exb && (aj ? (mask & 1) : (mask & 2));
                    sel[u] = (c ? 1u : 0u) | (aj ? 2u : 0u);
                    dv[u] = c ? __ldcs(drow + j) : kInf;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (!(sel[u] & 1u)) continue;
                    const int j = ((w0 + u) << 5) + lane;
                    const bool aj = sel[u] & 2u;
                    double lo2, hi2;
                    d_unpack(dv[u], lo2, hi2);
                    Lo2& x = aj ? xa : xn;
                    x.u = fmin(x.u, hi2);
                    lo2_put(x, lo2, j, dv[u]);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int st = 0; st < 2; ++st) {
                Lo2& x = st ? xn : xa;
                const double l1 = __shfl_xor_sync(0xffffffffu, x.l1, o), v1 = __shfl_xor_sync(0xffffffffu, x.v1, o);
                const double l2 = __shfl_xor_sync(0xffffffffu, x.l2, o), u2 = __shfl_xor_sync(0xffffffffu, x.u, o);
                const int j1 = __shfl_xor_sync(0xffffffffu, x.j1, o);
                x.u = fmin(x.u, u2);
                if (j1 != kNoJ) lo2_put(x, l1, j1, v1);
                if (l2 < x.l2) x.l2 = l2;
            }
        }
        RowBest ba{xa.v1, xa.j1}, bn{xn.v1, xn.j1};  // single candidate (or none)
        const bool multA = xa.j1 != kNoJ && xa.l2 <= xa.u, multN = xn.j1 != kNoJ && xn.l2 <= xn.u;
        if (live_i && (multA || multN)) {
            if (multA) ba = rb_none();
            if (multN) bn = rb_none();
            for (int s0 = 0; s0 < ss.S; s0 += 32) {
                const int sl = s0 + lane;
                const int j = sl < ss.S ? col[sl] : -1;
                bool cand = false, aj = false;
                double v = kInf;
                if (j >= 0 && j != i && j != ex && j != rs_exb && cnt[j] != 0u) {
                    aj = (arow[j >> 5] >> (j & 31)) & 1u;
                    if (aj ? (mask & 1) && multA : (mask & 2) && multN) {
                        v = __ldcs(drow + j);
                        double lo2, hi2;
                        d_unpack(v, lo2, hi2);
                        cand = lo2 <= (aj ? xa.u : xn.u);
                    }
                }
                if (cand && !d_is_interval(v)) {
                    if (aj) rb_offer(ba, v, j);
                    else rb_offer(bn, v, j);
                }
                unsigned m = __ballot_sync(0xffffffffu, cand && d_is_interval(v));
                while (m) {
                    const int src = __ffs(m) - 1;
                    m &= m - 1;
                    const int jj = __shfl_sync(0xffffffffu, j, src);
                    const bool ajj = __shfl_sync(0xffffffffu, aj, src);
                    const double d = exact_pair(i, jj);
                    if (lane == src) {
                        if (ajj) rb_offer(ba, d, jj);
                        else rb_offer(bn, d, jj);
                    }
                }
            }
            if (multA) ba = warp_min_rb(ba);
            if (multN) bn = warp_min_rb(bn);
        }
        if (lane == 0) {
            const int r = i - lo;
            if (mask & 1) { bAd[r] = ba.d; bAj[r] = ba.j == kNoJ ? -1 : ba.j; }
            if (mask & 2) { bNd[r] = bn.d; bNj[r] = bn.j == kNoJ ? -1 : bn.j; }
            if (T2A) {  // (first partner only: complete iff the stage has no candidate)
                uint8_t c = cx[r];
                if (mask & 1) { bAd2[r] = kInf; bAj2[r] = -1; c = ba.j == kNoJ ? (c | 1) : (c & ~1); }
                if (mask & 2) { bNd2[r] = kInf; bNj2[r] = -1; c = bn.j == kNoJ ? (c | 2) : (c & ~2); }
                cx[r] = c;
            }
        }
    };

    // APO rescan, fast path: one branch-free pass over the row keeps, per stage, the
    // two smallest 64-bit keys (D bits with the sign cleared -- the exact value or an
    // interval's centre -- truncated by 14 bits, with the column id in the low 14 bits:
    // non-negative doubles order like their bit patterns) and the widest interval code.
    // If the smallest key's entry has its upper bound below the lower bound of every
    // other entry (bounded through the second key and the widest code), it is the
    // row's minimum; otherwise that stage falls back to rescanf_full.
    constexpr unsigned long long kKeyHi = 0x7fffffffffffc000ULL, kKeyNone = ~0ULL;
    auto key_unique = [&](unsigned long long k1, unsigned long long k2, int kmax, const double* drow,
                          double& v1) {
        v1 = __ldcg(drow + (int)(k1 & 0x3fff));
        if (k2 == kKeyNone) return true;
        double l1, h1;
        d_unpack(v1, l1, h1);
        // other entries: centre >= c2 (truncated: relative 2^-38), interval >= centre (1 - rho)
        const double c2 = __longlong_as_double((long long)(k2 & kKeyHi));
        const double rho = __longlong_as_double((long long)(kmax - 46 + 1023) << 52) + 0x1p-37;
        return h1 < __dmul_rd(c2, __dsub_rd(1.0, rho));
    };
#if RHSEG_KEY32
    // 32-bit keys: the high word of the D bits with the sign cleared (exponent and 20
    // mantissa bits: non-negative doubles order like it), kept per lane with the column
    // and D value of the smallest; warp minima by redux.sync instead of 64-bit shuffle
    // trees. Two entries within 2^-20 of each other share a key and fail the uniqueness
    // test like any interval overlap (exact fallback), so the result is the same.
    // part / nparts: this warp walks one slice of the row (nparts > 1: idle warps share the
    // rescans of a step with few of them; the slice's keys go to rs_part[item] and
    // rescanf_finish combines them after the post-rescan barrier)
    auto rescanf = [&](int i, int mask, int ex, int part, int nparts, int item, const double* sbuf = nullptr) {
        const uint32_t* arow = adj + (size_t)i * W;
        const double* drow = D + (size_t)i * Rp;
        unsigned a1 = ~0u, a2 = ~0u, n1 = ~0u, n2 = ~0u;
        int ja = -1, jn = -1;
        double va = kInf, vn = kInf;
        int km = 0;  // widest interval code over both stages (only widens the test)
        constexpr int U = RHSEG_RESCAN_U;
        // high-word walk: the keys are the high words of the D bits, so a walk can load 32
        // bits per entry (twice the entries in flight for the same registers); the
        // winner's full entry is reloaded afterwards and the interval width bound comes
        // from the section-wide maximum code (misc[15], every interval ever written to D)
        const int kms = misc[15];
        const bool hi_ok = RHSEG_RESCAN_HI && kRsStage == 0 && !sbuf && nparts == 1 && kms <= RHSEG_RESCAN_HI_KMAX;
        bool hi_used = false;
        // the row's adjacency words (W <= 64 on APO sections), one or two per lane, loaded
        // once: every walk iteration then waits on its D loads only, not on a global
        // adjacency load in front of them (the merges rewrite these rows, so L1 rarely
        // holds them)
        uint32_t awl0 = 0u, awl1 = 0u;
        const bool areg = RHSEG_AROW_REGS && W <= 64;  // (uniform)
        if (areg) {
            awl0 = lane < W ? arow[lane] : 0u;
            awl1 = 32 + lane < W ? arow[32 + lane] : 0u;
        }
        auto aword = [&](int w) -> uint32_t {  // word w of the row (w uniform or per lane)
            if (!areg) return arow[w];
            const uint32_t x0 = __shfl_sync(0xffffffffu, awl0, w & 31), x1 = __shfl_sync(0xffffffffu, awl1, w & 31);
            return w < 32 ? x0 : x1;
        };
        // the walk is specialised on the stage mask: a single-stage rescan (the common
        // case) tracks one pair of keys
        auto walk = [&](auto MKC) {
            constexpr int MK = decltype(MKC)::value;
            auto take = [&](double v, int j, bool c, bool aj) {
                const unsigned hw = (unsigned)__double2hiint(v), lw = (unsigned)__double2loint(v);
                km = max(km, (int)(hw >> 31) * (int)(lw & 63u));
                const unsigned key = c ? (hw & 0x7fffffffu) : ~0u;
                if (MK == 1 || MK == 3) {
                    const unsigned ka = (MK == 1 || aj) ? key : ~0u;
                    if (ka < a1) { a2 = a1; a1 = ka; ja = j; va = v; }
                    else a2 = min(a2, ka);
                }
                if (MK == 2 || MK == 3) {
                    const unsigned kn = (MK == 2 || !aj) ? key : ~0u;
                    if (kn < n1) { n2 = n1; n1 = kn; jn = j; vn = v; }
                    else n2 = min(n2, kn);
                }
            };
            if (MK == 1 && RHSEG_ADJ_GATHER && nparts == 1 && W <= 64 && !areg) {
                // adjacent-only rescan: the row's adjacency words in one coalesced load,
                // then the D entries of the (few) adjacent live columns only -- two rounds
                // of loads instead of a dependent (adjacency word, D) pair per batch of words
                uint32_t w0 = lane < W ? arow[lane] & livew[lane] : 0u;
                uint32_t w1 = 32 + lane < W ? arow[32 + lane] & livew[32 + lane] : 0u;
                auto clr = [&](int j) {
                    if (j < 0) return;
                    if ((j >> 5) == lane) w0 &= ~(1u << (j & 31));
                    if ((j >> 5) == 32 + lane) w1 &= ~(1u << (j & 31));
                };
                clr(i);
                clr(ex);
                clr(rs_exb);
                const int cb = __popc(w0) + __popc(w1);
                int incl = cb;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int tot = __shfl_sync(0xffffffffu, incl, 31);
                if (tot <= 2 * B) {  // (uniform) the list fits this warp's staging row
                    int* lst = reinterpret_cast<int*>(xstg);
                    int k = incl - cb;
                    for (uint32_t m = w0; m; m &= m - 1) lst[k++] = (lane << 5) + __ffs(m) - 1;
                    for (uint32_t m = w1; m; m &= m - 1) lst[k++] = ((32 + lane) << 5) + __ffs(m) - 1;
                    __syncwarp();
                    for (int t0 = 0; t0 < tot; t0 += 32 * U) {
                        double dv[U];
                        int jv[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int t = t0 + 32 * u + lane;
                            jv[u] = t < tot ? lst[t] : -1;
                            dv[u] = jv[u] >= 0 ? __ldcs(drow + jv[u]) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) take(dv[u], jv[u], jv[u] >= 0, true);
                    }
                    __syncwarp();  // (the staging row is the exact fallback's next)
                    return;
                }
            }
            if (RHSEG_SPARSE_DEN * ss.S < RHSEG_SPARSE_NUM * R0) {
                // sparse (most regions merged away): walk the compacted live-column list
                const int slo = part * ss.S / nparts, shi = (part + 1) * ss.S / nparts;
                for (int s0 = slo; s0 < shi; s0 += 32 * U) {
                    double dv[U];
                    int jv[U];
                    uint32_t sel[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int sl = s0 + 32 * u + lane;
                        const int j = sl < shi ? col[sl] : -1;
                        const uint32_t awj = aword(j >= 0 ? j >> 5 : 0);  // (every lane: shuffles)
                        bool c = false, aj = false;
                        const bool lv = j >= 0 && j != i && j != ex && j != rs_exb && ((livew[j >> 5] >> (j & 31)) & 1u);
                        if (lv) {
                            aj = (awj >> (j & 31)) & 1u;
                            c = aj ? (MK & 1) : (MK & 2);
                        }
                        jv[u] = j;
                        sel[u] = (c ? 1u : 0u) | (aj ? 2u : 0u);
                        const bool ld = (MK == 2 && RHSEG_N_NODEP) ? lv : c;  // (see the id-ordered walk)
                        dv[u] = ld ? (sbuf ? sbuf[j] : __ldcs(drow + j)) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) take(dv[u], jv[u], sel[u] & 1u, sel[u] & 2u);
                }
            } else {
                // id-ordered walk, one bitset word per warp-iteration: lane l takes id
                // 32 w + l, whose liveness and adjacency bits come from two broadcast
                // words, and the D loads of a warp are one contiguous 256-byte segment
                const int wlo = part * W / nparts, whi = (part + 1) * W / nparts;
                auto issue = [&](int w0, double* dv, uint32_t* sel) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int w = w0 + u;
                        const uint32_t lw = w < whi ? livew[w] : 0u, aw = w < whi ? aword(w) : 0u;
                        const int j = (w << 5) + lane;
                        const bool aj = (aw >> lane) & 1u;
                        const bool lv = ((lw >> lane) & 1u) && j != i && j != ex && j != rs_exb;
                        const bool c = lv && (aj ? (MK & 1) : (MK & 2));
                        sel[u] = (c ? 1u : 0u) | (aj ? 2u : 0u);
                        // non-adjacent-only walks load every live column's entry, so the D
                        // load does not wait on the adjacency word (c masks the adjacent ones)
                        const bool ld = (MK == 2 && RHSEG_N_NODEP) ? lv : c;
                        dv[u] = ld ? (sbuf ? sbuf[j] : __ldcs(drow + j)) : 0.0;
                    }
                };
                if (hi_ok) {
                    hi_used = true;
                    constexpr int UH = 2 * U;
                    auto take_hi = [&](unsigned hw, int j, bool c, bool aj) {
                        const unsigned key = c ? (hw & 0x7fffffffu) : ~0u;
                        if (MK == 1 || MK == 3) {
                            const unsigned ka = (MK == 1 || aj) ? key : ~0u;
                            if (ka < a1) { a2 = a1; a1 = ka; ja = j; }
                            else a2 = min(a2, ka);
                        }
                        if (MK == 2 || MK == 3) {
                            const unsigned kn = (MK == 2 || !aj) ? key : ~0u;
                            if (kn < n1) { n2 = n1; n1 = kn; jn = j; }
                            else n2 = min(n2, kn);
                        }
                    };
                    const unsigned* dhw = reinterpret_cast<const unsigned*>(drow) + 1;  // high words
                    for (int w0 = wlo; w0 < whi; w0 += UH) {
                        unsigned hv[UH];
                        uint32_t sel[UH];
#pragma unroll
                        for (int u = 0; u < UH; ++u) {
                            const int w = w0 + u;
                            const uint32_t lw = w < whi ? livew[w] : 0u, aw = w < whi ? aword(w) : 0u;
                            const int j = (w << 5) + lane;
                            const bool aj = (aw >> lane) & 1u;
                            const bool lv = ((lw >> lane) & 1u) && j != i && j != ex && j != rs_exb;
                            const bool c = lv && (aj ? (MK & 1) : (MK & 2));
                            sel[u] = (c ? 1u : 0u) | (aj ? 2u : 0u);
                            const bool ld = (MK == 2 && RHSEG_N_NODEP) ? lv : c;
                            hv[u] = ld ? __ldcs(dhw + 2 * j) : 0u;
                        }
#pragma unroll
                        for (int u = 0; u < UH; ++u) take_hi(hv[u], ((w0 + u) << 5) + lane, sel[u] & 1u, sel[u] & 2u);
                    }
                } else if (RHSEG_RESCAN_PIPE) {
                    // software-pipelined: the next batch's loads are in flight while this
                    // batch is folded into the keys
                    double dv[U], dn[U];
                    uint32_t sel[U], sn[U];
                    issue(wlo, dv, sel);
                    for (int w0 = wlo; w0 < whi; w0 += U) {
                        if (w0 + U < whi) issue(w0 + U, dn, sn);
#pragma unroll
                        for (int u = 0; u < U; ++u) take(dv[u], ((w0 + u) << 5) + lane, sel[u] & 1u, sel[u] & 2u);
#pragma unroll
                        for (int u = 0; u < U; ++u) { dv[u] = dn[u]; sel[u] = sn[u]; }
                    }
                } else {
                    for (int w0 = wlo; w0 < whi; w0 += U) {
                        double dv[U];
                        uint32_t sel[U];
                        issue(w0, dv, sel);
#pragma unroll
                        for (int u = 0; u < U; ++u) take(dv[u], ((w0 + u) << 5) + lane, sel[u] & 1u, sel[u] & 2u);
                    }
                }
            }
        };
        if (cnt[i] != 0u) {
            if (mask == 1) walk(std::integral_constant<int, 1>{});
            else if (mask == 2) walk(std::integral_constant<int, 2>{});
            else walk(std::integral_constant<int, 3>{});
        }
        if (kRsStage && sbuf) fence_proxy_async_shared();  // the buffer's next fill is an async write
        km = hi_used ? kms : __reduce_max_sync(0xffffffffu, km);
        // warp minimum of one stage: the smallest key, the second smallest (== the
        // smallest on a tie), the winner's column and D value
        auto reduce = [&](unsigned& k1, unsigned& k2, int& j1, double& v1) {
            const unsigned m1 = __reduce_min_sync(0xffffffffu, k1);
            const unsigned win = __ballot_sync(0xffffffffu, k1 == m1);
            const int wl = __ffs(win) - 1;
            const unsigned m2 = __popc(win) > 1 ? m1 : __reduce_min_sync(0xffffffffu, lane == wl ? k2 : k1);
            j1 = __shfl_sync(0xffffffffu, j1, wl);
            v1 = __shfl_sync(0xffffffffu, v1, wl);
            k1 = m1;
            k2 = m2;
        };
        // unique iff the smallest key's upper bound lies below the lower bound of every
        // other entry: their centres are >= the second key (truncated), each interval
        // within 2^(km-46) of its centre
        auto unique32 = [&](unsigned k2, double v1) {
            if (k2 == ~0u) return true;
            double l1, h1;
            d_unpack(v1, l1, h1);
            const double c2 = __hiloint2double((int)k2, 0);
            const double rho = __longlong_as_double((long long)(km - 46 + 1023) << 52) + 0x1p-37;
            return h1 < __dmul_rd(c2, __dsub_rd(1.0, rho));
        };
        if (nparts > 1) {  // this slice's warp minima -> rs_part[item]
            if (mask & 1) reduce(a1, a2, ja, va);
            if (mask & 2) reduce(n1, n2, jn, vn);
            if (lane == 0) rs_part[item] = RsSlice{a1, a2, n1, n2, ja, jn, km, 0, va, vn};
            return;
        }
        int slow = 0;
        if (mask & 1) reduce(a1, a2, ja, va);
        if (mask & 2) reduce(n1, n2, jn, vn);
        if (hi_used) {  // the winners' full entries (both in flight at once)
            if ((mask & 1) && a1 != ~0u) va = __ldcs(drow + ja);
            if ((mask & 2) && n1 != ~0u) vn = __ldcs(drow + jn);
        }
        if ((mask & 1) && a1 != ~0u && !unique32(a2, va)) slow |= 1;
        if ((mask & 2) && n1 != ~0u && !unique32(n2, vn)) slow |= 2;
        if (lane == 0) {
            const int r = i - lo;
            if ((mask & 1) && !(slow & 1)) { bAd[r] = a1 == ~0u ? kInf : va; bAj[r] = a1 == ~0u ? -1 : ja; }
            if ((mask & 2) && !(slow & 2)) { bNd[r] = n1 == ~0u ? kInf : vn; bNj[r] = n1 == ~0u ? -1 : jn; }
        }
        if (slow) rescanf_full(i, slow, ex);
    };
    // combine the nparts slices of row i (one warp; after the barrier closing the walks)
    auto rescanf_finish = [&](int i, int mask, int ex, int nparts, int item0) {
        RsSlice p = lane < nparts ? rs_part[item0 + lane]
                                  : RsSlice{~0u, ~0u, ~0u, ~0u, -1, -1, 0, 0, kInf, kInf};
        const int km = __reduce_max_sync(0xffffffffu, p.km);
        auto reduce = [&](unsigned& k1, unsigned& k2, int& j1, double& v1) {
            const unsigned m1 = __reduce_min_sync(0xffffffffu, k1);
            const unsigned win = __ballot_sync(0xffffffffu, k1 == m1);
            const int wl = __ffs(win) - 1;
            const unsigned m2 = __popc(win) > 1 ? m1 : __reduce_min_sync(0xffffffffu, lane == wl ? k2 : k1);
            j1 = __shfl_sync(0xffffffffu, j1, wl);
            v1 = __shfl_sync(0xffffffffu, v1, wl);
            k1 = m1;
            k2 = m2;
        };
        auto unique32 = [&](unsigned k2, double v1) {
            if (k2 == ~0u) return true;
            double l1, h1;
            d_unpack(v1, l1, h1);
            const double c2 = __hiloint2double((int)k2, 0);
            const double rho = __longlong_as_double((long long)(km - 46 + 1023) << 52) + 0x1p-37;
            return h1 < __dmul_rd(c2, __dsub_rd(1.0, rho));
        };
        int slow = 0;
        if (mask & 1) {
            reduce(p.a1, p.a2, p.ja, p.va);
            if (p.a1 != ~0u && !unique32(p.a2, p.va)) slow |= 1;
        }
        if (mask & 2) {
            reduce(p.n1, p.n2, p.jn, p.vn);
            if (p.n1 != ~0u && !unique32(p.n2, p.vn)) slow |= 2;
        }
        if (lane == 0) {
            const int r = i - lo;
            if ((mask & 1) && !(slow & 1)) { bAd[r] = p.a1 == ~0u ? kInf : p.va; bAj[r] = p.a1 == ~0u ? -1 : p.ja; }
            if ((mask & 2) && !(slow & 2)) { bNd[r] = p.n1 == ~0u ? kInf : p.vn; bNj[r] = p.n1 == ~0u ? -1 : p.jn; }
        }
        if (slow) rescanf_full(i, slow, ex);
    };

#else
    auto rescanf = [&](int i, int mask, int ex, int, int, int) {
        const uint32_t* arow = adj + (size_t)i * W;
        const double* drow = D + (size_t)i * Rp;
        unsigned long long a1 = kKeyNone, a2 = kKeyNone, n1 = kKeyNone, n2 = kKeyNone;
        int km = 0;  // widest interval code over both stages (only widens the test)
        constexpr int U = RHSEG_RESCAN_U;
        // the walk is specialised on the stage mask: a single-stage rescan (the common
        // case) tracks one pair of keys
        auto walk = [&](auto MKC) {
            constexpr int MK = decltype(MKC)::value;
            auto take = [&](double v, int j, bool c, bool aj) {
                const unsigned long long r = (unsigned long long)__double_as_longlong(v);
                km = max(km, (int)(r >> 63) * (int)(r & 63));
                const unsigned long long key = c ? ((r & kKeyHi) | (unsigned long long)j) : kKeyNone;
                if (MK == 1 || MK == 3) {
                    const unsigned long long ka = (MK == 1 || aj) ? key : kKeyNone;
                    a2 = min(a2, max(a1, ka));
                    a1 = min(a1, ka);
                }
                if (MK == 2 || MK == 3) {
                    const unsigned long long kn = (MK == 2 || !aj) ? key : kKeyNone;
                    n2 = min(n2, max(n1, kn));
                    n1 = min(n1, kn);
                }
            };
            if (RHSEG_SPARSE_DEN * ss.S < RHSEG_SPARSE_NUM * R0) {
                // sparse (most regions merged away): walk the compacted live-column list
                for (int s0 = 0; s0 < ss.S; s0 += 32 * U) {
                    double dv[U];
                    int jv[U];
                    uint32_t sel[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int sl = s0 + 32 * u + lane;
                        const int j = sl < ss.S ? col[sl] : -1;
                        bool c = false, aj = false;
                        if (j >= 0 && j != i && j != ex && j != rs_exb && ((livew[j >> 5] >> (j & 31)) & 1u)) {
                            aj = (arow[j >> 5] >> (j & 31)) & 1u;
                            c = aj ? (MK & 1) : (MK & 2);
                        }
                        jv[u] = j;
                        sel[u] = (c ? 1u : 0u) | (aj ? 2u : 0u);
                        dv[u] = c ? __ldcs(drow + j) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) take(dv[u], jv[u], sel[u] & 1u, sel[u] & 2u);
                }
            } else {
                // id-ordered walk, one bitset word per warp-iteration: lane l takes id
                // 32 w + l, whose liveness and adjacency bits come from two broadcast
                // words, and the D loads of a warp are one contiguous 256-byte segment
                auto issue = [&](int w0, double* dv, uint32_t* sel) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int w = w0 + u;
                        const uint32_t lw = w < W ? livew[w] : 0u, aw = w < W ? arow[w] : 0u;
                        const int j = (w << 5) + lane;
                        const bool aj = (aw >> lane) & 1u;
                        const bool c = ((lw >> lane) & 1u) && j != i && j != ex && j != rs_exb && (aj ? (MK & 1) : (MK & 2));
                        sel[u] = (c ? 1u : 0u) | (aj ? 2u : 0u);
                        dv[u] = c ? __ldcs(drow + j) : 0.0;
                    }
                };
                if (RHSEG_RESCAN_PIPE) {
                    // software-pipelined: the next batch's loads are in flight while this
                    // batch is folded into the keys
                    double dv[U], dn[U];
                    uint32_t sel[U], sn[U];
                    issue(0, dv, sel);
                    for (int w0 = 0; w0 < W; w0 += U) {
                        if (w0 + U < W) issue(w0 + U, dn, sn);
#pragma unroll
                        for (int u = 0; u < U; ++u) take(dv[u], ((w0 + u) << 5) + lane, sel[u] & 1u, sel[u] & 2u);
#pragma unroll
                        for (int u = 0; u < U; ++u) { dv[u] = dn[u]; sel[u] = sn[u]; }
                    }
                } else {
                    for (int w0 = 0; w0 < W; w0 += U) {
                        double dv[U];
                        uint32_t sel[U];
                        issue(w0, dv, sel);
#pragma unroll
                        for (int u = 0; u < U; ++u) take(dv[u], ((w0 + u) << 5) + lane, sel[u] & 1u, sel[u] & 2u);
                    }
                }
            }
        };
        if (cnt[i] != 0u) {
            if (mask == 1) walk(std::integral_constant<int, 1>{});
            else if (mask == 2) walk(std::integral_constant<int, 2>{});
            else walk(std::integral_constant<int, 3>{});
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long oa1 = __shfl_xor_sync(0xffffffffu, a1, o), oa2 = __shfl_xor_sync(0xffffffffu, a2, o);
            const unsigned long long on1 = __shfl_xor_sync(0xffffffffu, n1, o), on2 = __shfl_xor_sync(0xffffffffu, n2, o);
            km = max(km, __shfl_xor_sync(0xffffffffu, km, o));
            a2 = min(min(a2, oa2), max(a1, oa1));
            a1 = min(a1, oa1);
            n2 = min(min(n2, on2), max(n1, on1));
            n1 = min(n1, on1);
        }
        int slow = 0;
        double va = kInf, vn = kInf;
        if ((mask & 1) && a1 != kKeyNone && !key_unique(a1, a2, km, drow, va)) slow |= 1;
        if ((mask & 2) && n1 != kKeyNone && !key_unique(n1, n2, km, drow, vn)) slow |= 2;
        if (lane == 0) {
            const int r = i - lo;
            if ((mask & 1) && !(slow & 1)) { bAd[r] = va; bAj[r] = a1 == kKeyNone ? -1 : (int)(a1 & 0x3fff); }
            if ((mask & 2) && !(slow & 2)) { bNd[r] = vn; bNj[r] = n1 == kKeyNone ? -1 : (int)(n1 & 0x3fff); }
        }
        if (slow) rescanf_full(i, slow, ex);
    };

#endif
    // TOP2-APO rescan: per masked stage the entries of the two smallest 32-bit keys and
    // the third key; the first is certified as in rescanf (upper bound below the second
    // key's lower bound), the second when its upper bound lies below the third key's; a
    // list is complete when it holds every candidate of the stage.
    struct K3 {
        unsigned k1, k2, k3;
        int j1, j2, n;
        double v1, v2;
    };
    auto rescant = [&](int i, int mask, int ex) {
        const uint32_t* arow = adj + (size_t)i * W;
        const double* drow = D + (size_t)i * Rp;
        K3 xa{~0u, ~0u, ~0u, -1, -1, 0, kInf, kInf}, xn = xa;
        int km = 0;
        auto put = [](K3& x, unsigned key, int j, double v) {
            x.n += 1;
            if (key < x.k1) {
                x.k3 = x.k2; x.k2 = x.k1; x.j2 = x.j1; x.v2 = x.v1;
                x.k1 = key; x.j1 = j; x.v1 = v;
            } else if (key < x.k2) {
                x.k3 = x.k2; x.k2 = key; x.j2 = j; x.v2 = v;
            } else {
                x.k3 = min(x.k3, key);
            }
        };
        auto take = [&](double v, int j, bool c, bool aj) {
            if (!c) return;
            const unsigned hw = (unsigned)__double2hiint(v), lw = (unsigned)__double2loint(v);
            km = max(km, (int)(hw >> 31) * (int)(lw & 63u));
            if (aj) put(xa, hw & 0x7fffffffu, j, v);
            else put(xn, hw & 0x7fffffffu, j, v);
        };
        constexpr int U = RHSEG_RESCAN_U;
        if (cnt[i] != 0u) {
            if (RHSEG_SPARSE_DEN * ss.S < RHSEG_SPARSE_NUM * R0) {
                for (int s0 = 0; s0 < ss.S; s0 += 32 * U) {
                    double dv[U];
                    int jv[U];
                    uint32_t sel[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int sl = s0 + 32 * u + lane;
                        const int j = sl < ss.S ? col[sl] : -1;
                        bool c = false, aj = false;
                        if (j >= 0 && j != i && j != ex && j != rs_exb && ((livew[j >> 5] >> (j & 31)) & 1u)) {
                            aj = (arow[j >> 5] >> (j & 31)) & 1u;
                            c = aj ? (mask & 1) : (mask & 2);
                        }
                        jv[u] = j;
                        sel[u] = (c ? 1u : 0u) | (aj ? 2u : 0u);
                        dv[u] = c ? __ldcs(drow + j) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) take(dv[u], jv[u], sel[u] & 1u, sel[u] & 2u);
                }
            } else {
                for (int w0 = 0; w0 < W; w0 += U) {
                    double dv[U];
                    uint32_t sel[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int w = w0 + u;
                        const uint32_t lw = w < W ? livew[w] : 0u, aw = w < W ? arow[w] : 0u;
                        const int j = (w << 5) + lane;
                        const bool aj = (aw >> lane) & 1u;
                        const bool c = ((lw >> lane) & 1u) && j != i && j != ex && j != rs_exb && (aj ? (mask & 1) : (mask & 2));
                        sel[u] = (c ? 1u : 0u) | (aj ? 2u : 0u);
                        dv[u] = c ? __ldcs(drow + j) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) take(dv[u], ((w0 + u) << 5) + lane, sel[u] & 1u, sel[u] & 2u);
                }
            }
        }
        km = __reduce_max_sync(0xffffffffu, km);
        const double rho = __longlong_as_double((long long)(km - 46 + 1023) << 52) + 0x1p-37;
        auto below = [&](double v, unsigned knext) {  // v's upper bound < every entry keyed >= knext
            if (knext == ~0u) return true;
            double l, h;
            d_unpack(v, l, h);
            return h < __dmul_rd(__hiloint2double((int)knext, 0), __dsub_rd(1.0, rho));
        };
        // warp top-2 of one stage (+ the third key); res: 0 empty, 1 first only, 2 both, -1 slow
        auto reduce3 = [&](K3& x, int& res, bool& complete) {
            const int n = __reduce_add_sync(0xffffffffu, x.n);
            const unsigned m1 = __reduce_min_sync(0xffffffffu, x.k1);
            const unsigned b1 = __ballot_sync(0xffffffffu, x.k1 == m1);
            const int w1 = __ffs(b1) - 1;
            const bool tie1 = __popc(b1) > 1;
            const unsigned o2 = lane == w1 ? x.k2 : x.k1;
            const unsigned m2 = tie1 ? m1 : __reduce_min_sync(0xffffffffu, o2);
            const unsigned b2 = __ballot_sync(0xffffffffu, o2 == m2);
            const int w2 = __ffs(b2) - 1;
            const bool tie2 = tie1 || __popc(b2) > 1;
            const unsigned o3 = lane == w1 ? (w2 == w1 ? x.k3 : x.k2) : (lane == w2 ? x.k2 : x.k1);
            const unsigned m3 = tie2 ? m2 : __reduce_min_sync(0xffffffffu, o3);
            const double v1 = __shfl_sync(0xffffffffu, x.v1, w1);
            const int j1 = __shfl_sync(0xffffffffu, x.j1, w1);
            const double v2 = __shfl_sync(0xffffffffu, w2 == w1 ? x.v2 : x.v1, w2);
            const int j2 = __shfl_sync(0xffffffffu, w2 == w1 ? x.j2 : x.j1, w2);
            x.v1 = v1; x.j1 = j1; x.v2 = v2; x.j2 = j2;
            if (m1 == ~0u) { res = 0; complete = true; return; }
            if (!below(v1, m2)) { res = -1; complete = false; return; }
            res = (m2 != ~0u && !tie2 && below(v2, m3)) ? 2 : 1;
            complete = n <= res;
        };
        int slow = 0, ra = 0, rn = 0;
        bool ca = false, cn = false;
        if (mask & 1) { reduce3(xa, ra, ca); if (ra < 0) slow |= 1; }
        if (mask & 2) { reduce3(xn, rn, cn); if (rn < 0) slow |= 2; }
        if (lane == 0) {
            const int r = i - lo;
            uint8_t c = cx[r];
            if ((mask & 1) && ra >= 0) {
                bAd[r] = ra ? xa.v1 : kInf; bAj[r] = ra ? xa.j1 : -1;
                bAd2[r] = ra == 2 ? xa.v2 : kInf; bAj2[r] = ra == 2 ? xa.j2 : -1;
                c = ca ? (c | 1) : (c & ~1);
            }
            if ((mask & 2) && rn >= 0) {
                bNd[r] = rn ? xn.v1 : kInf; bNj[r] = rn ? xn.j1 : -1;
                bNd2[r] = rn == 2 ? xn.v2 : kInf; bNj2[r] = rn == 2 ? xn.j2 : -1;
                c = cn ? (c | 2) : (c & ~2);
            }
            cx[r] = c;
        }
        if (slow) rescanf_full(i, slow, ex);
    };

    // TOP2 rescan: the two best candidates per masked stage + the complete bit,
    // over the compacted live-column list (one CTA owns every column).
    auto rescan2 = [&](int i, int mask, int ex) {
        Top2 ta = t2_none(), tn = t2_none();
        if (cnt[i] != 0u) {
            const uint32_t* arow = adj + (size_t)i * W;
            const double* drow = D + (size_t)i * Rp;
            constexpr int U = 16;
            for (int s0 = 0; s0 < ss.S; s0 += 32 * U) {
                double dv[U];
                int jv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int sl = s0 + 32 * u + lane;
                    const int j = sl < ss.S ? col[sl] : -1;
                    jv[u] = j;
                    dv[u] = j >= 0 ? __ldcs(drow + j) : kInf;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = jv[u];
                    if (j >= 0 && j != i && j != ex && j != rs_exb && cnt[j] != 0u) {
                        if ((arow[j >> 5] >> (j & 31)) & 1u) {
                            if (mask & 1) t2_offer(ta, dv[u], j);
                        } else if (mask & 2) {
                            t2_offer(tn, dv[u], j);
                        }
                    }
                }
            }
        }
        ta = warp_top2(ta);
        tn = warp_top2(tn);
        if (lane == 0) {
            const int r = i - lo;
            uint8_t c = cx[r];
            if (mask & 1) {
                bAd[r] = ta.d0; bAj[r] = ta.j0 == kNoJ ? -1 : ta.j0;
                bAd2[r] = ta.d1; bAj2[r] = ta.j1 == kNoJ ? -1 : ta.j1;
                c = ta.n <= 2 ? (c | 1) : (c & ~1);
            }
            if (mask & 2) {
                bNd[r] = tn.d0; bNj[r] = tn.j0 == kNoJ ? -1 : tn.j0;
                bNd2[r] = tn.d1; bNj2[r] = tn.j1 == kNoJ ? -1 : tn.j1;
                c = tn.n <= 2 ? (c | 2) : (c & ~2);
            }
            cx[r] = c;
        }
    };

    // ---- streaming ring (SPEC) ----
    // Stage `i` of the current step into ring slot abs_stage % NS. Called by
    // all lanes of warp 0: lane 0 arms the full barrier, the lanes issue one bulk
    // copy per band row in parallel.
    auto issue_stage = [&](uint32_t abs_stage, int i) {
        const int sl = (int)(abs_stage % NS);
        const int k0 = i * ss.KB;
        const int kb = min(ss.KB, B - k0);
        const uint32_t rowb = (uint32_t)ss.S2 * (uint32_t)ES;
        if (lane == 0) {
            fence_proxy_async_shared();
            mbar_arrive_expect_tx(&bars[sl], rowb * (uint32_t)kb);
        }
        __syncwarp();
        char* dst = reinterpret_cast<char*>(ring) + (size_t)sl * SB;
        const SE* src = (ss.cur ? sb1 : sb0) + lo;
        for (int kk = lane; kk < kb; kk += 32)
            bulk_g2s(dst + (size_t)kk * rowb, src + (size_t)(k0 + kk) * Rp, rowb, &bars[sl]);
    };
    // Block-wide exclusive scan of 0/1 flags (two __syncthreads).
    auto block_scan = [&](int v, int& total) {
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        int* scr = reinterpret_cast<int*>(pscr);
        if (lane == 31) scr[warp] = x;
        __syncthreads();
        int wbase = 0, tot = 0;
        for (int w = 0; w < kWarps; ++w) {
            if (w < warp) wbase += scr[w];
            tot += scr[w];
        }
        __syncthreads();
        total = tot;
        return wbase + x - v;
    };
    // Stable in-place compaction of this CTA's live columns into the other mean
    // buffer (ids stay ascending, so slot order == id order for every tie-break).
    auto compact = [&]() {
        int base = 0;
        for (int c0 = 0; c0 < ss.S; c0 += kThreads) {
            const int s = c0 + tid;
            const int id = s < ss.S ? col[s] : -1;
            int tot;
            const int np = base + block_scan(id >= 0 ? 1 : 0, tot);
            const SE* src = (ss.cur ? sb1 : sb0) + lo + s;
            SE* dst = (ss.cur ? sb0 : sb1) + lo + np;
            if (id >= 0) {
                if (STREAM) {
#pragma unroll 8
                    for (int k = 0; k < B; ++k) dst[(size_t)k * Rp] = src[(size_t)k * Rp];
                }
                slot_of[id - lo] = np;
            }
            __syncthreads();  // every read of col[] in this chunk precedes the writes below
            if (id >= 0) col[np] = id;
            base += tot;
        }
        if (STREAM) fence_proxy_async_global();
        __syncthreads();
        ss.S = base;
        ss.holes = 0;
        ss.cur ^= 1;
    };

    // Geometry of the next step's stream + its first NS band chunks in flight
    // (compacting first when >= 25% of the own columns are holes).
    auto begin_stream = [&]() {
        // compact when holes >= 2 sqrt(S): balances the streamed holes (~1/sqrt(S) of
        // the bytes) against the copy cost (2 S B words every 2 sqrt(S) merges)
        if (!STREAM) {  // APO: only the column list (no mean columns) is compacted
            if (ss.S >= 64 && ss.holes * RHSEG_APO_COMPACT >= ss.S) compact();
            return;
        }
        if (ss.S >= 64 && ss.holes * ss.holes >= RHSEG_COMPACT_K * ss.S) compact();
        constexpr int kAlign = 16 / ES;  // bulk copies move multiples of 16 bytes
        ss.S2 = (ss.S + kAlign - 1) / kAlign * kAlign;
        ss.KB = ss.S2 > 0 ? max(1, min(B, SB / (ss.S2 * ES))) : B;
        ss.nst = ss.S2 > 0 ? (B + ss.KB - 1) / ss.KB : 0;
        ss.base = ss.issued;
        const int pre = min(NS, ss.nst);
        if (warp == 0)
            for (int i = 0; i < pre; ++i) issue_stage(ss.base + i, i);
        ss.issued += pre;
    };

    // ---- prologue: counts, per-row caches, initial adjacent-pair count ----
    for (int i = tid; i < Rp; i += kThreads) cnt[i] = i < R0 ? bt.count[(size_t)sec * Rp + i] : 0u;
    if (SPEC) {
        for (int r = tid; r < hi - lo; r += kThreads) {
            col[r] = lo + r;
            slot_of[r] = r;
        }
        ss.S = max(0, hi - lo);
        if (STREAM && tid == 0)
            for (int s = 0; s < NS; ++s) {
                mbar_init(&bars[s], 1);
            }
        if (APO && kRsStage && tid == 0)
            for (int s = 0; s < kRsStage; ++s) mbar_init(&bars[s], 1);
        mbar_init_fence();
    }
    if (tid == 0) {
        ninv = 0;
        misc[14] = 0;
        misc[10] = 0;
        // widest interval code in D so far: the all-pairs init's intervals c (1 -/+ 2^(k-46))
        // around d (1 -/+ rho), rho = 2 (B + 4) u, need 2^(k-46) >= rho + 2^-45 (truncated
        // centre); +1 spare. apo_rows raises it with every interval it writes.
        misc[15] = APO ? 47 + (int)ceil(log2(2.0 * (B + 4) * kU64 + 0x1p-45)) : 0;
        misc[12] = 0;
        sdE = 0;
        sE0 = 0ull;
        sScan = 0;
        rpart[0] = rb_none();
        rpart[1] = rb_none();
    }
    __syncthreads();
    double apoE = 0.0, apoEe = 0.0;
    if (APO) {
        // ||m|| bound for the whole loop: every later mean is a weighted average of the
        // initial ones (times (1 + u)^depth), so per band max_i |m_i[k]| bounds |m[k]|
        double* sx = reinterpret_cast<double*>(misc + 8);
        if (tid == 0) *sx = 0.0;
        __syncthreads();
        double acc = 0.0;
        for (int k = warp; k < B; k += kWarps) {
            double mx = 0.0;
            for (int i = lane; i < R0; i += 32)
                if (cnt[i] != 0u) mx = fmax(mx, fabs(mu0[(size_t)k * Rp + i]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            acc = __dadd_ru(acc, __dmul_ru(mx, mx));
        }
        if (lane == 0) atomicAdd(sx, acc);  // (any order: rounded up afterwards)
        __syncthreads();
        apoE = (double)(B + 8) * kU64 * 1.01;
        for (size_t e = tid; e < (size_t)R0 * B; e += kThreads) {
            const int i = (int)(e / B);
            if (cnt[i] != 0u) mr[e] = __ddiv_rn(sums[e], (double)cnt[i]);  // == the cached mean, bit for bit
        }
        for (int i = tid; i < Rp; i += kThreads) ver[i] = (unsigned short)i;
        for (int w = tid; w < W; w += kThreads) {
            uint32_t m = 0u;
            for (int t = 0; t < 32; ++t) m |= (cnt[(w << 5) + t] != 0u ? 1u : 0u) << t;
            livew[w] = m;
        }
        __syncthreads();
        apoEe = sqrt(*sx * (1.0 + 1e-9)) * (10.0 * kU64 * 1.01);  // see apo_interval
        __syncthreads();
    }
    if (TOP2) {
        for (int r = tid; r < hi - lo; r += kThreads) cx[r] = 0;
        __syncthreads();
        for (int i = lo + warp; i < hi; i += kWarps) rescan2(i, 3, -1);
    } else if (T2A) {
        for (int r = tid; r < hi - lo; r += kThreads) {
            cx[r] = 0;
            bAd2[r] = kInf; bAj2[r] = -1;
            bNd2[r] = kInf; bNj2[r] = -1;
        }
        __syncthreads();
        for (int i = lo + warp; i < hi; i += kWarps) rescant(i, 3, -1);
    } else if (F32) {
        for (int i = lo + warp; i < hi; i += kWarps) rescanf(i, 3, -1, 0, 1, 0);
    } else {
        for (int i = lo + warp; i < hi; i += kWarps) rescan(i, SPEC ? 3 : 1, -1);
    }
    long long E = 0;
    if (SPEC && rank == 0) {
        unsigned long long e = 0;
        for (size_t w = tid; w < (size_t)R0 * W; w += kThreads) e += __popc(adj[w]);
        atomicAdd(&sE0, e);
    }
    __syncthreads();
    if (SPEC) E = (long long)(sE0 / 2);
    // every CTA of the cluster has started (and initialised its shared memory)
    // before any peer pushes a slot into it with DSMEM stores
    if (CLUSTER) cluster_barrier();
    if (SPEC && R0 > target) begin_stream();

    if (APO) {
        unsigned* ak0 = reinterpret_cast<unsigned*>(smem + L.apk);
        if (tid == 0) {
            ninv = 0;
            nnb = 0;
            sScan = 0;
            ak0[0] = ak0[1] = ak0[4] = ak0[5] = 0xffffffffu;
            ak0[2] = ak0[3] = 0u;
        }
        __syncthreads();
    }
    int a_prev = -1, step = 0, conv = 0;
    long long pairs = 0, nresc = 0;  // (nresc: row rescans, the loop's D-row reads; thread 0)
    // optional per-phase cycle accounting (RHSEG_PROFILE=1): thread 0 of every CTA
    unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // (+ APO counters at prof[8..15])
    long long tmark = clock64();
    pc[6] = (unsigned long long)(tmark - t_entry);  // prologue (caches, initial rescans, E)
    auto mark = [&](int ph) {
        if (bt.prof && tid == 0) {
            const long long t = clock64();
            pc[ph] += (unsigned long long)(t - tmark);
            tmark = t;
        }
    };
    while (R0 - step > target) {
        const int par = step & 1;
        // (0) the spectral stream of this step was put in flight at the end of the
        // previous step (or in the prologue); columns a and b of this step are never
        // read from it.
        // (A) best pair over this CTA's rows (engine.py:281-296 restricted to own rows)
        Pair A = pair_none(), N = pair_none();
        RowBest PA = rb_none(), PN = rb_none();
        unsigned* ak = reinterpret_cast<unsigned*>(smem + L.apk);  // APO: [0..1] min key, [2..3] max key, [4..5] min row
        if (APO) {
            // row caches may hold intervals. Per stage, the minimum lies among the rows
            // whose lower bound reaches the smallest upper bound; when those rows all
            // hold the same pair (typically rows i and j of the winning pair) it is the
            // winner, interval or not. Otherwise their intervals are made exact.
            // (a_prev's caches and this scratch were set at the end of the last step,
            // or before the loop)
            double uA = kInf, uN = kInf;
            for (int i = lo + tid; i < hi; i += kThreads) {
                if (cnt[i] == 0u) continue;
                const int r = i - lo;
                double l2, h2;
                if (bAj[r] >= 0) { d_unpack(bAd[r], l2, h2); uA = fmin(uA, h2); }
                if (bNj[r] >= 0) { d_unpack(bNd[r], l2, h2); uN = fmin(uN, h2); }
            }
            {
                RowBest x{uA, 0}, y{uN, 0};
                block_min_rb2(x, y, rscr);
                uA = x.d;
                uN = y.d;
            }
            unsigned short* clist = reinterpret_cast<unsigned short*>(inv);
            for (int i = lo + tid; i < hi; i += kThreads) {
                if (cnt[i] == 0u) continue;
                const int r = i - lo;
#pragma unroll
                for (int st = 0; st < 2; ++st) {
                    const int j = st ? bNj[r] : bAj[r];
                    if (j < 0) continue;
                    double l2, h2;
                    d_unpack(st ? bNd[r] : bAd[r], l2, h2);
                    if (!(l2 <= (st ? uN : uA))) continue;
                    const unsigned key = ((unsigned)min(i, j) << 16) | (unsigned)max(i, j);
                    atomicMin(&ak[st], key);
                    atomicMax(&ak[2 + st], key);
                    atomicMin(&ak[4 + st], (unsigned)i);
                    clist[atomicAdd(&sScan, 1)] = (unsigned short)(i | (st << 14));
                }
            }
            __syncthreads();
            const bool hasCA = ak[4] != 0xffffffffu, hasCN = ak[5] != 0xffffffffu;
            const bool multA = hasCA && ak[0] != ak[2], multN = hasCN && ak[1] != ak[3];
            if (multA || multN) {  // distinct pairs within each other's intervals (ties)
                const int nc = sScan;
                for (int t = warp; t < nc; t += kWarps) {
                    const int e = clist[t], i = e & 0x3fff, st = e >> 14, r = i - lo;
                    if (!(st ? multN : multA)) continue;
                    const int j = st ? bNj[r] : bAj[r];
                    if (!d_is_interval(st ? bNd[r] : bAd[r])) continue;
                    const double d = exact_pair(i, j);
                    __syncwarp();
                    if (lane == 0) {
                        if (st) bNd[r] = d;
                        else bAd[r] = d;
                    }
                }
                __syncthreads();
                Pair ca = pair_none(), cn = pair_none();
                for (int t = tid; t < nc; t += kThreads) {
                    const int e = clist[t], i = e & 0x3fff, r = i - lo;
                    if (e >> 14) {
                        if (multN) pair_offer(cn, make_pair(bNd[r], i, bNj[r]));
                    } else if (multA) {
                        pair_offer(ca, make_pair(bAd[r], i, bAj[r]));
                    }
                }
                block_min_pair2(ca, cn, pscr);
                if (multA) A = ca;
                if (multN) N = cn;
            }
            if (hasCA && !multA) {
                const int i = (int)ak[4], r = i - lo;
                A = make_pair(bAd[r], i, bAj[r]);
            }
            if (hasCN && !multN) {
                const int i = (int)ak[5], r = i - lo;
                N = make_pair(bNd[r], i, bNj[r]);
            }
            mark(0);
        } else {
            // (A) best pair over this CTA's rows (engine.py:281-296 restricted to own rows)
            Pair ca = pair_none(), cn = pair_none();
            for (int i = lo + tid; i < hi; i += kThreads) {
                if (cnt[i] == 0u || i == a_prev) continue;
                const int r = i - lo;
                if (bAj[r] >= 0) pair_offer(ca, make_pair(bAd[r], i, bAj[r]));
                if (SPEC && bNj[r] >= 0) pair_offer(cn, make_pair(bNd[r], i, bNj[r]));
            }
            if (tid == 0) { ninv = 0; nnb = 0; }
            if (SPEC) block_min_pair2(ca, cn, pscr);
            else ca = block_min_pair(ca, pscr);
            if (tid == 0) {
                slot[par].selA = ca;
                slot[par].selN = cn;
                slot[par].rpA = rpart[0];
                slot[par].rpN = rpart[1];
            }
            if (CLUSTER) {
                // push this CTA's slot into rslot[par][rank] of every CTA of the cluster
                // (fire-and-forget DSMEM stores); after the release/acquire cluster
                // barrier every CTA combines the C slots from its own shared memory
                __syncthreads();
                if (tid < C * 16) {
                    const int r = tid >> 4, w = tid & 15;
                    const uint32_t v = reinterpret_cast<const uint32_t*>(&slot[par])[w];
                    dsmem_st_u32(dsmem_addr(&rslot[par * kMaxCluster + rank], (unsigned)r) + 4u * w, v);
                }
                cluster_barrier();
            } else {
                __syncthreads();
            }

            mark(0);
            // (B) combine the C slots: identical decision in every CTA
            for (int r = 0; r < C; ++r) {
                const Slot& s = CLUSTER ? rslot[par * kMaxCluster + r] : slot[par];
                pair_offer(A, s.selA);
                rb_offer(PA, s.rpA.d, s.rpA.j);
                if (SPEC) {
                    pair_offer(N, s.selN);
                    rb_offer(PN, s.rpN.d, s.rpN.j);
                }
            }
            if (a_prev >= 0) {
                if (PA.j != kNoJ) pair_offer(A, make_pair(PA.d, a_prev, PA.j));
                if (SPEC && PN.j != kNoJ) pair_offer(N, make_pair(PN.d, a_prev, PN.j));
                if (tid == 0 && a_prev >= lo && a_prev < hi) {
                    const int r = a_prev - lo;
                    bAd[r] = PA.d;
                    bAj[r] = PA.j == kNoJ ? -1 : PA.j;
                    if (SPEC) { bNd[r] = PN.d; bNj[r] = PN.j == kNoJ ? -1 : PN.j; }
                    if (TOP2) {  // a's fresh row: its best only (complete iff it has none)
                        bAd2[r] = kInf; bAj2[r] = -1;
                        bNd2[r] = kInf; bNj2[r] = -1;
                        cx[r] = (uint8_t)((PA.j == kNoJ ? 1 : 0) | (PN.j == kNoJ ? 2 : 0));
                    }
                }
            }
        }
        // merge rule (engine.py:322-339): spectral wins iff d_s < w * d_a, strictly
        int a = -1, b = -1, kind = 0;
        double dch = 0.0;
        const bool hasA = A.hi != kNoJ;
        if (SPEC && N.hi != kNoJ) {
            if (APO) {
                // decide on the intervals (rounding w * d_a is monotone); when they
                // cannot, both dissimilarities are made exact (warps 0 and 1)
                double nl, nh, al = kInf, ah = kInf;
                d_unpack(N.d, nl, nh);
                if (hasA) d_unpack(A.d, al, ah);
                int dec = nh < __dmul_rn(bt.weight, al) ? 1 : (nl >= __dmul_rn(bt.weight, ah) ? 0 : -1);
                if (dec < 0) {
                    double* xs = reinterpret_cast<double*>(smem + L.apk + 32);
                    if (warp == 0) {
                        const double d = exact_pair(N.lo, N.hi);
                        if (lane == 0) xs[0] = d;
                    } else if (warp == 1 && hasA) {
                        const double d = exact_pair(A.lo, A.hi);
                        if (lane == 0) xs[1] = d;
                    }
                    __syncthreads();
                    N.d = xs[0];
                    if (hasA) A.d = xs[1];
                    dec = N.d < __dmul_rn(bt.weight, hasA ? A.d : kInf) ? 1 : 0;
                }
                if (dec) { a = N.lo; b = N.hi; dch = N.d; kind = 1; }
            } else {
                const double da = hasA ? A.d : kInf;
                if (N.d < __dmul_rn(bt.weight, da)) { a = N.lo; b = N.hi; dch = N.d; kind = 1; }
            }
        }
        if (a < 0 && hasA) { a = A.lo; b = A.hi; dch = A.d; kind = 0; }
        if (a < 0) {
            conv = 1;
            if (STREAM) {  // drain the copies put in flight for this step
                for (int i = 0; i < min(NS, ss.nst); ++i) {
                    const uint32_t g = ss.base + i;
                    mbar_wait(&bars[g % NS], (g / NS) & 1u);
                }
            }
            break;
        }

        mark(1);
        // (C1) rows whose cached partner was a or b (rescanned in C2, after the
        // merge); their D rows are prefetched into L2 while the merge runs.
        // The barrier publishes thread 0's update of a_prev's caches (above). (APO: those
        // were published at the end of the last step, and the argmin's shared reads are
        // fenced by its own barriers.)
        if (!APO) __syncthreads();
        for (int i = lo + tid; i < hi; i += kThreads) {
            if (cnt[i] == 0u || i == a || i == b) continue;
            const int r = i - lo;
            int mask = 0;
            if (TOP2 || T2A) {
                l2_remove(bAd[r], bAj[r], bAd2[r], bAj2[r], a);
                l2_remove(bAd[r], bAj[r], bAd2[r], bAj2[r], b);
                l2_remove(bNd[r], bNj[r], bNd2[r], bNj2[r], a);
                l2_remove(bNd[r], bNj[r], bNd2[r], bNj2[r], b);
                if (bAj[r] < 0 && !(cx[r] & 1)) mask |= 1;
                if (bNj[r] < 0 && !(cx[r] & 2)) mask |= 2;
            } else {
                if (bAj[r] == a || bAj[r] == b) mask |= 1;
                if (SPEC && (bNj[r] == a || bNj[r] == b)) mask |= 2;
            }
            if (mask) {
                if (kLpt && mask == 1) inv[Rs - 1 - atomicAdd(&misc[14], 1)] = (i << 2) | mask;  // cheap: last
                else inv[atomicAdd(&ninv, 1)] = (i << 2) | mask;
                // its D row is read by the rescan after the merge: start the fetch now
                if (RHSEG_RESCAN_PREFETCH) bulk_prefetch_l2(D + (size_t)i * Rp, (uint32_t)(((R0 + 1) & ~1) * 8));
            }
        }
        if (APO && tid == 0) {  // rows a and b feed the row-a' pass after the merge
            bulk_prefetch_l2(D + (size_t)a * Rp, (uint32_t)(((R0 + 1) & ~1) * 8));
            bulk_prefetch_l2(D + (size_t)b * Rp, (uint32_t)(((R0 + 1) & ~1) * 8));
        }
        // (C) merge (graph.py:229-264) on this CTA's private copies
        const double nn = __dadd_rn((double)cnt[a], (double)cnt[b]);
        const bool own_a = a >= lo && a < hi;
        const double na0 = (double)cnt[a], nb0 = (double)cnt[b];  // (APO: the log's exact value, in C2)
        ApoStep ap{};
        if (APO) ap = apo_step<M>(na0, nb0, dch, apoE, apoEe);
        // APO: the merge runs on warps 0-1 (named barrier) while the other warps start
        // the rescans (which skip a and b and read nothing the merge writes but bits a
        // and b of neighbour rows' adjacency words); the others merge with every thread
        constexpr int MT = APO ? 2 * 32 : kThreads;  // merging threads
        uint32_t rbph_now = 0u;
        if (APO) {
            __syncthreads();  // the invalidated-row list is complete
            rs_exb = b;
            if (kRsStage) {
                // the first kRsStage listed rows: one bulk copy of the D row into shared
                // memory each (issued by warp 2, which then starts the rescans too)
                const int nst = min(ninv, kRsStage);
                rbph_now = rbph;
                rbph ^= (1u << nst) - 1u;
                if (warp == 2 && lane < nst) {
                    const int i = inv[lane] >> 2;
                    const uint32_t bytes = (uint32_t)(((R0 + 1) & ~1) * 8);
                    mbar_arrive_expect_tx(&bars[lane], bytes);
                    bulk_g2s(rbuf + (size_t)lane * Rp, D + (size_t)i * Rp, bytes, &bars[lane]);
                }
            }
        }
        uint32_t* ra = adj + (size_t)a * W;
        if (!APO || warp < 2) {
        {
            double* sa = sums + (size_t)a * B;
            const double* sb = sums + (size_t)b * B;
            SE* mu_a = STREAM ? (own_a ? (ss.cur ? sb1 : sb0) + lo + slot_of[a - lo] : nullptr)
                              : (SPEC ? nullptr : mu0 + a);
            for (int k = tid; k < B; k += MT) {
                const double s = __dadd_rn(sa[k], sb[k]);
                sa[k] = s;
                const double m = __ddiv_rn(s, nn);
                mua[k] = m;  // (APO: written to mr row R0 + step at the end of the step)
                if ((STREAM || !SPEC) && own_a) mu_a[(size_t)k * Rp] = m;
            }
            if (STREAM && own_a) fence_proxy_async_global();
        }
        {
            // adjacency union (A|B)\{a,b}; b's neighbours are collected first and then
            // re-pointed b -> a one per thread (not serially per bitset word)
            uint32_t* rbw = adj + (size_t)b * W;
            const int wa = a >> 5, wb = b >> 5;
            const uint32_t ma = 1u << (a & 31), mb = 1u << (b & 31);
            auto repoint = [&](int n) {
                uint32_t* rn = adj + (size_t)n * W;
                if (wa == wb) rn[wa] = (rn[wa] | ma) & ~mb;
                else { rn[wa] |= ma; rn[wb] &= ~mb; }
            };
            int dE = 0;
            for (int w = tid; w < W; w += MT) {
                const uint32_t oa = ra[w], ob = rbw[w];
                uint32_t nw = oa | ob;
                if (w == wa) nw &= ~ma;
                if (w == wb) nw &= ~mb;
                if (SPEC) {
                    dE += __popc(nw) - __popc(oa) - __popc(ob);
                    if (w == wb && (oa & mb)) dE += 1;
                }
                ra[w] = nw;
                sra[w] = nw;
                rbw[w] = 0u;
                uint32_t bits = w == wa ? ob & ~ma : ob;
                while (bits) {
                    const int n = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int k = atomicAdd(&nnb, 1);
                    if (k < kNbList) nbl[k] = (unsigned short)n;
                    else repoint(n);  // overflow (very high degree): in place
                }
            }
            if (SPEC && dE) atomicAdd(&sdE, dE);
            if (APO) asm volatile("bar.sync 1, %0;" ::"n"(MT) : "memory");
            else __syncthreads();
            const int nb = min(nnb, kNbList);
            for (int k = tid; k < nb; k += MT) repoint(nbl[k]);
        }
        }  // (merging threads)
        if (APO) {
            // the rescans: rows claimed from a shared counter (the merge warps join when done)
            const long long tr0 = clock64();
            int nr = 0;
            // full walks first, adjacent-only gathers (a few loads) last: the slowest warp
            // sets the step, so the long items go out first (LPT)
            const int nf = ninv, ni = nf + (kLpt ? misc[14] : 0);
            for (;;) {
                int k = 0;
                if (lane == 0) k = atomicAdd(&misc[12], 1);
                k = __shfl_sync(0xffffffffu, k, 0);
                if (k >= ni) break;
                const int e = k < nf ? inv[k] : inv[Rs - 1 - (k - nf)];
                if (kRsStage && k < kRsStage) {
                    mbar_wait(&bars[k], (rbph_now >> k) & 1u);
                    rescanf(e >> 2, e & 3, a, 0, 1, 0, rbuf + (size_t)k * Rp);
                } else {
                    rescanf(e >> 2, e & 3, a, 0, 1, 0);
                }
                ++nr;
            }
            if (bt.prof && lane == 0 && nr) {
                const unsigned long long dt = (unsigned long long)(clock64() - tr0);
                atomicAdd(bt.prof + 13, dt);
                atomicAdd(bt.prof + 14, (unsigned long long)nr);
                atomicMax(bt.prof + 15, dt);
            }
            if (tid == 0) nresc += ni;
            if (bt.prof && tid == 0) pc[5] += (unsigned long long)ni;
            rs_exb = -1;
        }
        __syncthreads();  // every thread has read cnt[a], cnt[b] (nn) before they change
        if (tid == 0) {
            cnt[a] = (uint32_t)nn;
            cnt[b] = 0u;
            if (APO) livew[b >> 5] &= ~(1u << (b & 31));
            if (own_a) {
                bAd[a - lo] = kInf; bAj[a - lo] = -1;
                bNd[a - lo] = kInf; bNj[a - lo] = -1;
            }
            if (rank == 0) {
                const size_t o = (size_t)sec * Rp + step;
                bt.log_a[o] = a;
                bt.log_b[o] = b;
                bt.log_d[o] = dch;
                if (APO && d_is_interval(dch))  // exact value after the loop (versions of a and b)
                    bt.apo_rec[o] = make_uint4(ver[a], ver[b], (unsigned)na0, (unsigned)nb0);
                bt.log_k[o] = (uint8_t)kind;
                bt.parent[(size_t)sec * Rp + b] = a;
                if (SPEC) {
                    const long long R = R0 - step;
                    pairs += R * (R - 1) / 2 - E;
                }
            }
        }
        if (!APO) __syncthreads();  // (APO: nothing below reads cnt[a], cnt[b] or the live set before the next barrier)
        if (SPEC) E += sdE;
        mark(2);

        // (C2) rows whose cached partner was a or b: rescan them from D now,
        // skipping a (its entries are refreshed by the row-a pass, which then
        // offers (d(i, a), a) to every row) and b (dead). Their D loads overlap the
        // row-a stream already in flight. (APO: the merge's closing barrier suffices.)
        if (!APO) __syncthreads();
        double apo_uA = kInf, apo_uN = kInf;  // this thread's smallest upper bounds of row a'
        // APO: interval around every d(a', j) from the old D rows a and b (parallelogram
        // identity, apo_interval), written to D; bounds kept per slot for the offers
        auto apo_rows = [&]() {
            double* sdl = reinterpret_cast<double*>(smem + L.sdv);
            double* sdh = sdl + Rs;
            int kw = 0;  // widest interval code this thread writes to D
            const double* Da = D + (size_t)a * Rp;
            const double* Db = D + (size_t)b * Rp;
            constexpr int NQ = kMaxSlots / kThreads;
            double ra[NQ], rb[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {  // all loads in flight first
                const int sl = tid + q * kThreads;
                const int j = sl < ss.S ? col[sl] : -1;
                const bool ok = j >= 0 && j != a && j != b && cnt[j] != 0u;
                ra[q] = ok ? __ldcg(Da + j) : 0.0;
                rb[q] = ok ? __ldcg(Db + j) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int sl = tid + q * kThreads;
                if (sl < ss.S) { sdl[sl] = ra[q]; sdh[sl] = rb[q]; }
            }
#pragma unroll 1
            for (int sl = tid; sl < ss.S; sl += kThreads) {
                const int j = col[sl];
                if (j < 0 || j == a || j == b || cnt[j] == 0u) continue;
                double dlo, dhi, v;
                apo_interval<M>(ap, sdl[sl], sdh[sl], (double)cnt[j], dlo, dhi);
                sdl[sl] = dlo;
                sdh[sl] = dhi;
                const bool aj = (sra[j >> 5] >> (j & 31)) & 1u;
                if (aj) apo_uA = fmin(apo_uA, dhi);
                else apo_uN = fmin(apo_uN, dhi);
                const bool packed = d_pack_interval(dlo, dhi, v);
                if (packed) {  // (too wide: made exact after C2)
                    D[(size_t)j * Rp + a] = v;
                    D[(size_t)a * Rp + j] = v;
                    if (RHSEG_RESCAN_HI && d_is_interval(v)) kw = max(kw, (int)(__double2loint(v) & 63));
                }
                if (kFuseOffers) {
                    // the offer (d(a', j), a) to row j, decided on the intervals unless they
                    // overlap row j's cached best (then exact, after the barrier below)
                    const unsigned short e = (unsigned short)(j | (aj ? 0 : 0x4000));
                    unsigned short* l1 = reinterpret_cast<unsigned short*>(inv);
                    if (!packed) {
                        l1[atomicAdd(&misc[10], 1)] = (unsigned short)(e | 0x8000);
                        continue;
                    }
                    const int r = j - lo;
                    double& bv = aj ? bAd[r] : bNd[r];
                    int& bj = aj ? bAj[r] : bNj[r];
                    if (bj < 0) {
                        bv = v;
                        bj = a;
                    } else {
                        double bl, bh;
                        d_unpack(bv, bl, bh);
                        if (dhi < bl) { bv = v; bj = a; }
                        else if (!(dlo > bh)) l1[atomicAdd(&misc[10], 1)] = e;
                    }
                }
            }
            if (RHSEG_RESCAN_HI && kw > 0) atomicMax(&misc[15], kw);  // (read by the next step's rescans)
        };
        if (APO && tid == 0) { sScan = 0; if (!kFuseOffers) misc[10] = 0; ak[6] = 0u; ak[7] = 0u; }
        // split APO rescans: with ni <= kWarps / 2 rows each row's walk is cut into the
        // largest power-of-two number of slices that keeps every warp busy
        const int nsplit = 1;  // (split rescans: measured slower, and APO now rescans beside the merge)
        if (!APO) {
            const int ni = ninv;
            if (tid == 0) nresc += ni;
            if (bt.prof && tid == 0) pc[5] += (unsigned long long)ni;
            if (TOP2) {
                for (int k = warp; k < ni; k += kWarps) rescan2(inv[k] >> 2, inv[k] & 3, a);
            } else if (CLUSTER) {
                // big sections: every warp takes a slice of the row, so one rescan
                // costs one round of loads instead of R0/256 sequential ones
                const int per = (((R0 + kWarps - 1) / kWarps) + 31) & ~31;
                const int c0 = min(R0, warp * per), c1 = min(R0, c0 + per);
                for (int k = 0; k < ni; ++k) {
                    const int i = inv[k] >> 2, mask = inv[k] & 3;
                    RowBest ba = rb_none(), bn = rb_none();
                    const uint32_t* arow = adj + (size_t)i * W;
                    const double* drow = D + (size_t)i * Rp;
                    for (int j0 = c0; j0 < c1; j0 += 32 * 16) {
                        double dv[16];
                        uint32_t wv[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const int j = j0 + 32 * u + lane;
                            dv[u] = j < c1 ? __ldcs(drow + j) : kInf;
                            wv[u] = (j0 + 32 * u) < c1 ? arow[(j0 >> 5) + u] : 0u;
                        }
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const int j = j0 + 32 * u + lane;
                            if (j < c1 && j != i && j != a && cnt[j] != 0u) {
                                if ((wv[u] >> lane) & 1u) {
                                    if (mask & 1) rb_offer(ba, dv[u], j);
                                } else if (SPEC && (mask & 2)) {
                                    rb_offer(bn, dv[u], j);
                                }
                            }
                        }
                    }
                    ba = warp_min_rb(ba);
                    if (SPEC) bn = warp_min_rb(bn);
                    RowBest* part = rscr;  // kWarps entries per stage (rscr + rpart area)
                    if (lane == 0) {
                        part[warp] = ba;
                        if (SPEC) spart[warp] = bn;
                    }
                    __syncthreads();
                    if (tid == 0) {
                        RowBest fa = rb_none(), fn = rb_none();
                        for (int w = 0; w < kWarps; ++w) {
                            rb_offer(fa, part[w].d, part[w].j);
                            if (SPEC) rb_offer(fn, spart[w].d, spart[w].j);
                        }
                        const int r = i - lo;
                        if (mask & 1) { bAd[r] = fa.d; bAj[r] = fa.j == kNoJ ? -1 : fa.j; }
                        if (SPEC && (mask & 2)) { bNd[r] = fn.d; bNj[r] = fn.j == kNoJ ? -1 : fn.j; }
                    }
                    __syncthreads();
                }
            } else if (APO) {
                const long long tr0 = clock64();
                int nr = 0;
                if (T2A) {
                    for (int k = warp; k < ni; k += kWarps, ++nr) rescant(inv[k] >> 2, inv[k] & 3, a);
                } else if (nsplit > 1) {  // few rescans: every row's walk split over idle warps
                    for (int t = warp; t < ni * nsplit; t += kWarps, ++nr)
                        rescanf(inv[t / nsplit] >> 2, inv[t / nsplit] & 3, a, t % nsplit, nsplit, t);
                } else {
                    for (int k = warp; k < ni; k += kWarps, ++nr) rescanf(inv[k] >> 2, inv[k] & 3, a, 0, 1, 0);
                }
                // then, without waiting for the other warps' rescans: the intervals of
                // row a' (D rows a and b are not touched by the rescans, which skip a)
                if (RHSEG_APO_OVERLAP) apo_rows();
                if (bt.prof && lane == 0 && nr) {
                    const unsigned long long dt = (unsigned long long)(clock64() - tr0);
                    atomicAdd(bt.prof + 13, dt);             // warp-rescan cycles
                    atomicAdd(bt.prof + 14, (unsigned long long)nr);  // rescans
                    atomicMax(bt.prof + 15, dt);
                }
            } else {
                for (int k = warp; k < ni; k += kWarps) rescan(inv[k] >> 2, inv[k] & 3, a);
            }
        }
        if (!APO) __syncthreads();  // (APO: the rescans ran beside the merge)
        if (nsplit > 1) {  // combine the slices (the offers' reduction barrier follows)
            const int ni = ninv;
            for (int k = warp; k < ni; k += kWarps) rescanf_finish(inv[k] >> 2, inv[k] & 3, a, nsplit, k * nsplit);
        }
        if (APO && !RHSEG_APO_OVERLAP) {
            const long long ta = bt.prof ? clock64() : 0;
            apo_rows();
            if (bt.prof && tid == 0) atomicAdd(bt.prof + 10, (unsigned long long)(clock64() - ta));  // (part of phase 4)
        }  // (own slots only: the offers' reduction barrier follows)
        mark(4);
        // (D) row-a pass over own columns: fresh d(a, j), D update, cache offers
        RowBest pA = rb_none(), pN = rb_none();
        double n2a = 0.0;
        if (M == kSam) {  // squared norm of a's new mean, sequential (oracle order)
            double* sn2a = reinterpret_cast<double*>(misc + 6);
            if (tid == 0) {
                *sn2a = norm2_seq(mua, 1, B);
                if (own_a) n2g[a] = *sn2a;
            }
            __syncthreads();
            n2a = *sn2a;
        }
        if (SPEC) {
            // columns of this thread: compacted slots tid + 256 q (q < 8)
            constexpr int NQ = kMaxSlots / kThreads;
            int jq[NQ];
            bool valid[NQ], isadj[NQ];
            double s[NQ];
            const int nq = (ss.S + kThreads - 1) / kThreads;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int sl = tid + q * kThreads;
                const int j = (q < nq && sl < ss.S) ? col[sl] : -1;
                jq[q] = j;
                valid[q] = j >= 0 && j != a && j != b && cnt[j] != 0u;
                isadj[q] = valid[q] && ((sra[j >> 5] >> (j & 31)) & 1u);
                s[q] = 0.0;
            }
            if (STREAM) {
                for (int i = 0; i < ss.nst; ++i) {
                    const uint32_t g = ss.base + i;
                    mbar_wait(&bars[g % NS], (g / NS) & 1u);
                    const SE* tile = reinterpret_cast<const SE*>(ring) + (size_t)(g % NS) * (SB / ES);
                    const int k0 = i * ss.KB, kb = min(ss.KB, B - k0);
                    // exactly nq columns per thread, unpredicated (slots >= S, holes, a and b
                    // accumulate garbage that the epilogue discards via valid[])
                    switch (nq) {
#define RHSEG_CONSUME(NQC)                                                        \
    case NQC:                                                                     \
        for (int kk = 0; kk < kb; ++kk) {                                         \
            const double m = mua[k0 + kk];                                        \
            const SE* row = tile + (size_t)kk * ss.S2 + tid;                      \
            _Pragma("unroll") for (int q = 0; q < NQC; ++q) s[q] = acc_step<M>(s[q], m, (double)row[q * kThreads]); \
        }                                                                         \
        break;
                        RHSEG_CONSUME(1) RHSEG_CONSUME(2) RHSEG_CONSUME(3) RHSEG_CONSUME(4)
                        RHSEG_CONSUME(5) RHSEG_CONSUME(6) RHSEG_CONSUME(7) RHSEG_CONSUME(8)
#undef RHSEG_CONSUME
                        default: break;
                    }
                    __syncthreads();  // slot g % NS is free again
                    if (i + NS < ss.nst) {
                        if (warp == 0) issue_stage(g + NS, i + NS);
                    }
                }
                ss.issued += max(0, ss.nst - NS);
            }
            if (APO) {
                // (row a' intervals: apo_rows, run by each warp right after its rescans)
                // offers: decided on the intervals unless they overlap row j's cached
                // best (then both sides are made exact below); a's own best: the columns
                // whose lower bound reaches the stage's smallest upper bound
                double* sdl = reinterpret_cast<double*>(smem + L.sdv);
                double* sdh = sdl + Rs;
                int* cntF = misc + 10;  // offers that need the exact d(a', j)
                unsigned short* l1 = reinterpret_cast<unsigned short*>(inv);  // exact offers
                unsigned short* l2 = l1 + Rs;                                 // a's candidates
                // (l1 and l2 each hold at most one entry per own column; entry = j |
                // 0x4000 non-adjacent stage | 0x8000 interval too wide to store)
                double uA = apo_uA, uN = apo_uN;
                {
                    RowBest x{uA, 0}, y{uN, 0};
                    block_min_rb2(x, y, rscr);
                    uA = x.d;
                    uN = y.d;
                }
#pragma unroll 1
                for (int sl = tid; sl < ss.S; sl += kThreads) {
                    const int j = col[sl];
                    if (j < 0 || j == a || j == b || cnt[j] == 0u) continue;
                    const bool aj = (sra[j >> 5] >> (j & 31)) & 1u;
                    const int r = j - lo;
                    const double dlo = sdl[sl], dhi = sdh[sl];
                    const unsigned short e = (unsigned short)(j | (aj ? 0 : 0x4000));
                    if (dlo <= (aj ? uA : uN)) {
                        l2[atomicAdd(&sScan, 1)] = e;
                        atomicAdd(&ak[aj ? 6 : 7], 1u);
                    }
                    if (kFuseOffers) continue;  // (offered in the interval pass)
                    double v;
                    if (!d_pack_interval(dlo, dhi, v)) {  // exact d(a', j) below, then the offer
                        l1[atomicAdd(&cntF[0], 1)] = (unsigned short)(e | 0x8000);
                        continue;
                    }
                    double& bv = aj ? bAd[r] : bNd[r];
                    int& bj = aj ? bAj[r] : bNj[r];
                    if (T2A) {
                        // insert (d(a', j), a) into row j's two-entry list on the intervals
                        // (an empty list is complete here: incomplete ones were rescanned)
                        double& bv2 = aj ? bAd2[r] : bNd2[r];
                        int& bj2 = aj ? bAj2[r] : bNj2[r];
                        const uint8_t bit = aj ? 1 : 2;
                        if (bj < 0) {
                            bv = v;
                            bj = a;
                        } else {
                            double bl, bh;
                            d_unpack(bv, bl, bh);
                            if (dhi < bl) {  // a' first; a listed second drops out
                                if (bj2 >= 0) cx[r] &= (uint8_t)~bit;
                                bv2 = bv; bj2 = bj;
                                bv = v; bj = a;
                            } else if (dlo > bh) {
                                if (bj2 < 0) {
                                    // complete single entry: a' is the second; otherwise a'
                                    // may sit behind unlisted candidates (not listed)
                                    if (cx[r] & bit) { bv2 = v; bj2 = a; }
                                } else {
                                    double cl, ch;
                                    d_unpack(bv2, cl, ch);
                                    if (dhi < cl) { bv2 = v; bj2 = a; cx[r] &= (uint8_t)~bit; }
                                    else if (dlo > ch) cx[r] &= (uint8_t)~bit;
                                    else l1[atomicAdd(&cntF[0], 1)] = e;
                                }
                            } else {
                                l1[atomicAdd(&cntF[0], 1)] = e;
                            }
                        }
                    } else if (bj < 0) {
                        bv = v;
                        bj = a;
                    } else {
                        double bl, bh;
                        d_unpack(bv, bl, bh);
                        if (dhi < bl) { bv = v; bj = a; }
                        else if (!(dlo > bh)) l1[atomicAdd(&cntF[0], 1)] = e;
                    }
                }
                __syncthreads();
                const int n1 = cntF[0], n2 = sScan;
                if (bt.prof && tid == 0) {
                    atomicAdd(bt.prof + 8, (unsigned long long)n1);
                    atomicAdd(bt.prof + 9, (unsigned long long)n2);
                }
                // overlaps with row j's cached best: exact d(a', j) and exact best
                for (int t = warp; t < n1; t += kWarps) {
                    const int e = l1[t], j = e & 0x3fff, r = j - lo;
                    const bool aj = !(e & 0x4000);
                    const double daj = RHSEG_WEXACT(mua, mr + (size_t)ver[j] * B, nn, (double)cnt[j], B, lane, xstg);
                    const int bj = aj ? bAj[r] : bNj[r];
                    double db = aj ? bAd[r] : bNd[r];
                    const bool binterval = bj >= 0 && d_is_interval(db);
                    if (binterval) db = exact_pair(j, bj);
                    const bool take_a = bj < 0 || daj < db || (daj == db && a < bj);
                    if (T2A) {
                        // exact insertion into the two-entry list (uniform decisions: every
                        // lane read the same cache entries)
                        const uint8_t bit = aj ? 1 : 2;
                        const int bj2 = aj ? bAj2[r] : bNj2[r];
                        double db2 = aj ? bAd2[r] : bNd2[r];
                        const bool complete = cx[r] & bit;
                        bool take2 = false;
                        if (!take_a && bj2 >= 0) {
                            if (d_is_interval(db2)) db2 = exact_pair(j, bj2);
                            take2 = daj < db2 || (daj == db2 && a < bj2);
                        }
                        __syncwarp();
                        if (lane == 0) {
                            D[(size_t)j * Rp + a] = daj;
                            D[(size_t)a * Rp + j] = daj;
                            double n1d = db, n2d = db2;
                            int n1j = bj, n2j = bj2;
                            uint8_t c = cx[r];
                            if (bj < 0) { n1d = daj; n1j = a; }
                            else if (take_a) {
                                if (bj2 >= 0) c &= (uint8_t)~bit;
                                n2d = db; n2j = bj; n1d = daj; n1j = a;
                            } else if (bj2 < 0) {
                                if (complete) { n2d = daj; n2j = a; }
                            } else {
                                if (take2) { n2d = daj; n2j = a; }
                                c &= (uint8_t)~bit;
                            }
                            if (aj) { bAd[r] = n1d; bAj[r] = n1j; bAd2[r] = n2d; bAj2[r] = n2j; }
                            else { bNd[r] = n1d; bNj[r] = n1j; bNd2[r] = n2d; bNj2[r] = n2j; }
                            cx[r] = c;
                        }
                        continue;
                    }
                    __syncwarp();  // every lane has read row j's cache before lane 0 rewrites it
                    if (lane == 0) {
                        D[(size_t)j * Rp + a] = daj;
                        D[(size_t)a * Rp + j] = daj;
                        if (aj) { bAd[r] = take_a ? daj : db; bAj[r] = take_a ? a : bj; }
                        else { bNd[r] = take_a ? daj : db; bNj[r] = take_a ? a : bj; }
                    }
                }
                if (n1) __syncthreads();  // (uniform: n1 was read after a barrier)
                // a's best per stage: a single candidate is the minimum as it is
                // (interval or not); several are compared exactly
                const int nA = ak[6], nN = ak[7];
                for (int t = warp; t < n2; t += kWarps) {
                    const int e = l2[t], j = e & 0x3fff;
                    const bool aj = !(e & 0x4000);
                    const double v = __ldcg(D + (size_t)a * Rp + j);
                    if ((aj ? nA : nN) == 1 || !d_is_interval(v)) {
                        if (lane == 0) {
                            if (aj) rb_offer_iv(pA, v, j);
                            else rb_offer_iv(pN, v, j);
                        }
                    } else {
                        const double d = RHSEG_WEXACT(mua, mr + (size_t)ver[j] * B, nn, (double)cnt[j], B, lane, xstg);
                        if (lane == 0) {
                            D[(size_t)j * Rp + a] = d;
                            D[(size_t)a * Rp + j] = d;
                            if (aj) rb_offer(pA, d, j);
                            else rb_offer(pN, d, j);
                        }
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    rowa_col<true, M, TOP2>(jq[q], valid[q], isadj[q], valid[q], s[q], nn, a, b, lo, Rp, cnt, n2a, n2g,
                                            D, bAd, bAj, bNd, bNj, pA, pN, inv, &ninv,
                                            Top2Lists{bAd2, bNd2, bAj2, bNj2, cx});
            }
        } else {
            // w = 0: only a's (own) neighbours need d(a, j). One warp per neighbour:
            // the lanes load j's region-major band sums coalesced, divide by the count
            // (the exact cached mean) and the ascending-band accumulation runs through
            // warp shuffles -- no strided, latency-bound walks over the band-major cache.
            if (tid == 0) sScan = 0;
            __syncthreads();
            for (int w = tid; w < W; w += kThreads) {
                uint32_t bits = ra[w];
                while (bits) {
                    const int j = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    if (j >= lo && j < hi && j != b && cnt[j] != 0u) inv[atomicAdd(&sScan, 1)] = j;
                }
            }
            __syncthreads();
            const int nnb = sScan;
            for (int t = warp; t < nnb; t += kWarps) {
                const int j = inv[t];
                const double* sj = sums + (size_t)j * B;
                const double cj = (double)cnt[j];
                double sacc = 0.0;
                for (int k0 = 0; k0 < B; k0 += 32) {
                    const double v = k0 + lane < B ? __ddiv_rn(sj[k0 + lane], cj) : 0.0;
                    const int kn = min(32, B - k0);
                    for (int kk = 0; kk < kn; ++kk)
                        sacc = acc_step<M>(sacc, mua[k0 + kk], __shfl_sync(0xffffffffu, v, kk));
                }
                if (lane == 0)
                    rowa_col<false, M>(j, true, true, true, sacc, nn, a, b, lo, Rp, cnt, n2a, n2g, D, bAd, bAj, nullptr,
                                       nullptr, pA, pN, inv, &ninv);
            }
        }
        // staged rescans bulk-copy D rows (async proxy) that this step's column a' writes
        // (generic proxy) feed: order them before the next step's copies
        if (APO && kRsStage) fence_proxy_async_global();
        if (SPEC) block_min_rb2(pA, pN, rscr);
        else pA = block_min_rb(pA, rscr);
        if (APO) {  // a's new mean becomes version R0 + step (the old one stays for the log)
            for (int k = tid; k < B; k += kThreads) mr[(size_t)(R0 + step) * B + k] = mua[k];
            if (tid == 0) {
                ver[a] = (unsigned short)(R0 + step);
                // a's fresh caches and the next argmin's scratch, published by the
                // barrier closing this step (no barrier needed at the next step's start)
                const int r = a - lo;
                bAd[r] = pA.d;
                bAj[r] = pA.j == kNoJ ? -1 : pA.j;
                bNd[r] = pN.d;
                bNj[r] = pN.j == kNoJ ? -1 : pN.j;
                if (T2A) {  // a's fresh row: its best only (complete iff the stage has none)
                    bAd2[r] = kInf; bAj2[r] = -1;
                    bNd2[r] = kInf; bNj2[r] = -1;
                    cx[r] = (uint8_t)((pA.j == kNoJ ? 1 : 0) | (pN.j == kNoJ ? 2 : 0));
                }
                ninv = 0;
                misc[14] = 0;
                nnb = 0;
                sScan = 0;
                misc[10] = 0;  // exact offers (the fused offers count them before any barrier)
                misc[12] = 0;  // rescan claim counter
                ak[0] = ak[1] = ak[4] = ak[5] = 0xffffffffu;
                ak[2] = ak[3] = 0u;
            }
        }
        if (tid == 0) {
            rpart[0] = pA;
            rpart[1] = pN;
            if (SPEC) sdE = 0;
            if (SPEC && b >= lo && b < hi) {  // b's column becomes a hole of the stream
                col[slot_of[b - lo]] = -1;
                slot_of[b - lo] = -1;
            }
        }
        if (SPEC && b >= lo && b < hi) ss.holes += 1;
        __syncthreads();
        // next step's stream overlaps the rescans below and the next argmin
        if (SPEC && R0 - (step + 1) > target) begin_stream();

        mark(3);
        a_prev = a;
        ++step;
    }
    if (APO) {
        // the log's dissimilarities still held as intervals: exact values now, one
        // thread per step (the reference's ascending-band sum from the two versions)
        __syncthreads();
        for (int t = tid; t < step; t += kThreads) {
            const size_t o = (size_t)sec * Rp + t;
            if (!d_is_interval(bt.log_d[o])) continue;
            const uint4 rc = bt.apo_rec[o];
            const double* mi = mr + (size_t)rc.x * B;
            const double* mj = mr + (size_t)rc.y * B;
            double sacc = 0.0;
            for (int k = 0; k < B; ++k) sacc = acc_step<M>(sacc, mi[k], mj[k]);
            bt.log_d[o] = pair_finish<M>((double)rc.z, (double)rc.w, sacc, 0.0, 0.0);
        }
    }
    if (CLUSTER) cluster_barrier();  // keep our slots alive until every peer is done reading
    if (bt.prof && tid == 0) {
        pc[7] = (unsigned long long)(clock64() - t_entry);  // whole kernel
        for (int q = 0; q < 8; ++q) atomicAdd(bt.prof + q, pc[q]);
    }
    if (rank == 0) {
        for (int i = tid; i < Rp; i += kThreads) bt.count[(size_t)sec * Rp + i] = cnt[i];
        if (tid == 0) {
            bt.nlog[sec] = step;
            bt.conv[sec] = conv;
            if (bt.pairs) bt.pairs[sec] = pairs;
            if (bt.nresc) bt.nresc[sec] = nresc;
        }
    }
}

int launch_hseg_loop(const SectionBatch& b, int nrun, cudaStream_t st) {
    if (nrun == 0) return 0;
    // APO sections: the APO variant below; RHSEG_APO_V2=1 selects the re-cut loop of
    // apo_loop.cu (bit-identical, currently slower: see profiles/r02_apo_v2.md)
    static const bool v1 = [] {
        const char* e = getenv("RHSEG_APO_V2");  // the re-cut loop is opt-in while it is slower
        return !(e && e[0] == '1');
    }();
    if (b.apo && !v1) return launch_apo_loop(b, nrun, st);
    // w = 0, one CTA per section: adj_loop.cu (RHSEG_ADJ_V1=1: the generic loop below)
    static const bool adj_v1 = [] {
        const char* e = getenv("RHSEG_ADJ_V1");
        return e && e[0] == '1';
    }();
    if (!b.spec && b.C == 1 && !adj_v1) {
        static const int nsm = [] {
            int dev = 0, n = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
            return n;
        }();
        return launch_adj_loop(b, nrun, nsm, st);
    }
    const size_t smem = hseg_loop_smem(b.Rp, b.C, b.B, b.spec != 0, b.measure, b.stage_bytes, b.nstages);
    void (*kern)(SectionBatch);
#define RHSEG_PICK(M)                                                                              \
    if (b.C > 1) kern = b.spec ? hseg_loop_kernel<true, true, M> : hseg_loop_kernel<true, false, M>; \
    else kern = b.spec ? hseg_loop_kernel<false, true, M> : hseg_loop_kernel<false, false, M>;
    if (b.measure == kSam) {
        RHSEG_PICK(kSam)
    } else if (b.measure == kEuclid) {
        RHSEG_PICK(kEuclid)
        if (b.apo)
            kern = (RHSEG_RPC && b.Rp == 1024) ? hseg_loop_kernel<false, true, kEuclid, true, 1024>
                   : (RHSEG_RPC && b.Rp == 64) ? hseg_loop_kernel<false, true, kEuclid, true, 64>
                                               : hseg_loop_kernel<false, true, kEuclid, true>;
    } else {
        RHSEG_PICK(kBsmse)
        if (b.apo)
            kern = (RHSEG_RPC && b.Rp == 1024) ? hseg_loop_kernel<false, true, kBsmse, true, 1024>
                   : (RHSEG_RPC && b.Rp == 64) ? hseg_loop_kernel<false, true, kBsmse, true, 64>
                                               : hseg_loop_kernel<false, true, kBsmse, true>;
    }
    if (b.apo && !apo_capable(b.spec != 0, b.C, b.measure)) return cudaErrorInvalidValue;
#undef RHSEG_PICK
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (b.C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nrun * b.C), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (b.C > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)b.C;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (b.l2_window_bytes > 0) {  // keep a small level's streamed means resident in L2
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = b.l2_window_base;
        attr[na].val.accessPolicyWindow.num_bytes = b.l2_window_bytes;
        attr[na].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, b);
}

}  // namespace rhseg
