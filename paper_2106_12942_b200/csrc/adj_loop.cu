// adj_loop.cu -- the HSEG merge loop for spectral_weight = 0 (adjacent merges only),
// one CTA per section, every section of a quadtree level in one persistent launch.
//
// Reference semantics (rhseg, read-only at /root/reference/pkg/src):
//   engine.py:309-342 hseg_step with w = 0 (engine.py:326 skips the spectral stage),
//   _kernels.py:31-59 scan_adjacent (per-row best neighbour, fp64, strict <, ascending
//   columns), engine.py:281-296 reduce_best (lexicographic (d, min id, max id)),
//   graph.py:229-264 merge_regions (smaller id survives), dissim.py:33-42 op order.
//
// Every D entry this loop reads is an exact fp64 dissimilarity of an adjacent pair
// (dinit_sparse_kernel, then the row-a' pass below). A step:
//  (A) argmin over the row caches: one block reduction of (d, min, max).
//  (C) rows whose cached neighbour is a or b are listed.
//  (X) merge || rescans: two warps merge (band sums, mean, adjacency union, neighbour
//      re-point, a' neighbour list); the other warps -- and the merge warps once done --
//      claim listed rows and re-minimise them over their adjacency from D, excluding a
//      and b (a rescan reads nothing the merge writes but bits a, b it skips).
//  (R) row a': d(a', j) for every neighbour j from the region-major means (no division:
//      the mean cache of Appendix A.3, sums / count, kept per region): a warp loads up to
//      8 neighbours' rows at once and stages the per-band terms, one lane per neighbour
//      runs the reference's ascending-band sum; D written, (d, a') offered to row j,
//      a's best by one block reduction.
//  (E) one thread publishes the merge (counts, log, a's cache); a's mean row updated.
// Five block barriers per step (round 1's generic loop: ~12 and a division per band
// per neighbour, 24k cycles per step on a C5 leaf).
#include <cuda_runtime.h>

#include <cstdlib>

#include "rhseg_batch.h"
#include "rhseg_device.cuh"

namespace rhseg {

// CTA shapes: 256 threads (8 warps, two of them merging) for levels with few
// sections, 128 threads (4 warps, one merging) with up to 7 CTAs per SM when the level
// has many: the step is a latency chain, so resident sections, not threads per
// section, set the throughput (C5 leaves: 1024 sections in one wave instead of three).
template <int NT>
struct AdjShape {
    static constexpr int kW = NT / 32;
    static constexpr int kMergeWarps = NT >= 256 ? 2 : 1;
    static constexpr int kMergeThreads = kMergeWarps * 32;
    static constexpr int kMinBlocks = NT >= 256 ? 3 : 7;
};
constexpr int kAdjNbList = 512;
constexpr int kAdjStage = 256;   // doubles of per-warp term staging (row a' pass; the
                                 // 128-thread shape keeps 7 CTAs per SM within 32 KB)
constexpr int kAdjStageNb = 8;   // neighbours per warp round

struct AdjSmem {
    size_t misc, red, cnt, bAd, bAj, inv, nbr, nbl, mua, terms, total;
};
__host__ __device__ inline size_t adj_align(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline AdjSmem adj_smem_layout(int Rp, int B, int nwarps) {
    AdjSmem L;
    const size_t R = (size_t)Rp;
    size_t o = 0;
    L.misc = o; o += 128;
    L.red = o;  o += 2 * 8 * sizeof(Pair);  // [parity][warp] (<= 8 warps)
    L.cnt = o;  o = adj_align(o + R * 4);
    L.bAd = o;  o = adj_align(o + R * 8);
    L.bAj = o;  o = adj_align(o + R * 4);
    L.inv = o;  o = adj_align(o + R * 2);            // listed rows
    L.nbr = o;  o = adj_align(o + R * 2);            // neighbours of a'
    L.nbl = o;  o = adj_align(o + kAdjNbList * 2);   // b's neighbours (re-point)
    L.mua = o;  o = adj_align(o + (size_t)B * 8);
    L.terms = o; o = adj_align(o + (size_t)nwarps * kAdjStage * 8);  // [warp][kAdjStage]
    L.total = o;
    return L;
}
size_t adj_loop_smem(int Rp, int B, int nwarps) { return adj_smem_layout(Rp, B, nwarps).total; }

enum { kAmNinv = 0, kAmIctr, kAmNnb, kAmNnbr };

template <int MT>
__device__ __forceinline__ void adj_bar_merge() {
    if (MT == 32) __syncwarp();
    else asm volatile("bar.sync 1, %0;" ::"n"(MT) : "memory");
}
__device__ __forceinline__ unsigned pair_key(int i, int j) {
    return ((unsigned)min(i, j) << 16) | (unsigned)max(i, j);
}
// lexicographic (d, key) minimum; key = min id << 16 | max id
__device__ __forceinline__ void dk_offer(double& d, unsigned& k, double d2, unsigned k2) {
    if (d2 < d || (d2 == d && k2 < k)) { d = d2; k = k2; }
}

template <int M, int NT>
__global__ void __launch_bounds__(NT, AdjShape<NT>::kMinBlocks) hseg_adj_kernel(SectionBatch bt) {
    constexpr int kThreads = NT, kWarps = AdjShape<NT>::kW, kAdjMergeThreads = AdjShape<NT>::kMergeThreads;
    extern __shared__ __align__(128) unsigned char smem[];
    const long long t_entry = clock64();
    const int sec = bt.sec0 + (int)blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R0 = bt.R0[sec];
    const int B = bt.B, Rp = bt.Rp, W = bt.W;
    const int target = bt.target[sec];
    const AdjSmem L = adj_smem_layout(Rp, B, kWarps);
    int* misc = reinterpret_cast<int*>(smem + L.misc);
    Pair* red = reinterpret_cast<Pair*>(smem + L.red);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L.cnt);
    double* bAd = reinterpret_cast<double*>(smem + L.bAd);
    int* bAj = reinterpret_cast<int*>(smem + L.bAj);
    unsigned short* inv = reinterpret_cast<unsigned short*>(smem + L.inv);
    unsigned short* nbr = reinterpret_cast<unsigned short*>(smem + L.nbr);
    unsigned short* nbl = reinterpret_cast<unsigned short*>(smem + L.nbl);
    double* mua = reinterpret_cast<double*>(smem + L.mua);
    double* terms = reinterpret_cast<double*>(smem + L.terms);
    double* n2s = reinterpret_cast<double*>(misc + 8);  // SAM: squared norm of a's new mean

    double* const mr = bt.mu2 + sec * bt.mu_stride();  // region-major exact means [Rp][B]
    double* __restrict__ D = bt.D + (sec - bt.sec0) * bt.d_stride();
    double* __restrict__ sums = bt.sums + (size_t)sec * bt.sums_copy();
    uint32_t* __restrict__ adj = bt.adj + (size_t)sec * bt.adj_copy();
    const double* __restrict__ n2g = M == kSam ? bt.nrm2 + (size_t)sec * Rp : nullptr;
    const bool prof = bt.prof != nullptr;

    // row i's best neighbour from D (the whole warp): lane l takes bitset word l, l+32, ...
    auto rescan = [&](int i, int exA, int exB) {
        const uint32_t* arow = adj + (size_t)i * W;
        const double* drow = D + (size_t)i * Rp;
        double bd = kInf;
        unsigned bj = 0xffffffffu;
        for (int w0 = 0; w0 < W; w0 += 32) {
            const int w = w0 + lane;
            uint32_t bits = w < W ? arow[w] : 0u;
            // at most a few neighbours per word: issue their loads first
            while (bits) {
                const int j = (w << 5) + __ffs(bits) - 1;
                bits &= bits - 1;
                if (j == i || j == exA || j == exB || j >= R0 || cnt[j] == 0u) continue;
                const double d = __ldcg(drow + j);
                if (d < bd || (d == bd && (unsigned)j < bj)) { bd = d; bj = (unsigned)j; }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, o);
            const unsigned oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (od < bd || (od == bd && oj < bj)) { bd = od; bj = oj; }
        }
        if (lane == 0) {
            bAd[i] = bd;
            bAj[i] = bj == 0xffffffffu ? -1 : (int)bj;
        }
    };
    // listed rows inv[0..ni) by all warps (warps < nmerge first run `merge`)
    auto rescan_rows = [&](int ni, int exA, int exB, auto&& merge, int nmerge) {
        if (warp < nmerge) merge();
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&misc[kAmIctr], 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= ni) break;
            rescan(inv[t], exA, exB);
        }
        __syncthreads();
    };

    // ---- prologue: counts, region-major means, initial per-row bests ----
    for (int i = tid; i < Rp; i += kThreads) {
        cnt[i] = i < R0 ? bt.count[(size_t)sec * Rp + i] : 0u;
        bAd[i] = kInf;
        bAj[i] = -1;
    }
    if (tid < 32) misc[tid] = 0;
    __syncthreads();
    for (size_t e = tid; e < (size_t)R0 * B; e += kThreads) {
        const int i = (int)(e / B);
        if (cnt[i] != 0u) mr[e] = __ddiv_rn(sums[e], (double)cnt[i]);  // == the cached mean, bit for bit
    }
    for (int i = tid; i < R0; i += kThreads)
        if (cnt[i] != 0u) inv[atomicAdd(&misc[kAmNinv], 1)] = (unsigned short)i;
    __syncthreads();
    rescan_rows(misc[kAmNinv], -1, -1, [] {}, 0);
    if (tid == 0) { misc[kAmNinv] = 0; misc[kAmIctr] = 0; }
    __syncthreads();

    int step = 0, conv = 0;
    long long nresc = 0;
    unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tmark = clock64();
    pc[6] = (unsigned long long)(tmark - t_entry);
    auto mark = [&](int ph) {
        if (prof && tid == 0) {
            const long long t = clock64();
            pc[ph] += (unsigned long long)(t - tmark);
            tmark = t;
        }
    };
    while (R0 - step > target) {
        const int par = step & 1;
        // ---- (A) argmin (engine.py:281-296 over the scan_adjacent table) ----
        double gd = kInf;
        unsigned gk = 0xffffffffu;
        for (int i = tid; i < R0; i += kThreads)
            if (cnt[i] != 0u && bAj[i] >= 0) dk_offer(gd, gk, bAd[i], pair_key(i, bAj[i]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, gd, o);
            const unsigned ok = __shfl_xor_sync(0xffffffffu, gk, o);
            dk_offer(gd, gk, od, ok);
        }
        Pair* scr = red + par * kWarps;
        if (lane == 0) scr[warp] = Pair{gd, (int)(gk >> 16), (int)(gk & 0xffffu)};
        __syncthreads();
        {   // every warp combines the kWarps partials in its lanes (3 shuffle rounds)
            const Pair p = lane < kWarps ? scr[lane] : Pair{kInf, 0, 0};
            gd = p.d;
            gk = p.d < kInf ? ((unsigned)p.lo << 16) | (unsigned)p.hi : 0xffffffffu;
#pragma unroll
            for (int o = kWarps / 2; o > 0; o >>= 1) {  // (lanes < kWarps hold the partials)
                const double od = __shfl_xor_sync(0xffffffffu, gd, o);
                const unsigned ok = __shfl_xor_sync(0xffffffffu, gk, o);
                dk_offer(gd, gk, od, ok);
            }
            gd = __shfl_sync(0xffffffffu, gd, 0);
            gk = __shfl_sync(0xffffffffu, gk, 0);
        }
        if (!(gd < kInf)) { conv = 1; break; }
        const int a = (int)(gk >> 16), b = (int)(gk & 0xffffu);
        const double dch = gd;
        const double nn = __dadd_rn((double)cnt[a], (double)cnt[b]);
        mark(0);

        // ---- (C) rows whose cached neighbour is a or b ----
        for (int i = tid; i < R0; i += kThreads) {
            if (cnt[i] == 0u || i == a || i == b) continue;
            if (bAj[i] == a || bAj[i] == b) inv[atomicAdd(&misc[kAmNinv], 1)] = (unsigned short)i;
        }
        __syncthreads();
        const int ni = misc[kAmNinv];
        nresc += ni;
        if (prof && tid == 0) pc[5] += (unsigned long long)ni;

        // ---- (X) merge (graph.py:229-264) || rescans ----
        auto merge = [&]() {
            const double* sb = sums + (size_t)b * B;
            double* sa = sums + (size_t)a * B;
            for (int k = tid; k < B; k += kAdjMergeThreads) {
                const double s = __dadd_rn(sa[k], sb[k]);
                sa[k] = s;
                mua[k] = __ddiv_rn(s, nn);
            }
            uint32_t* ra = adj + (size_t)a * W;
            uint32_t* rbw = adj + (size_t)b * W;
            const int wa = a >> 5, wb = b >> 5;
            const uint32_t ma = 1u << (a & 31), mb = 1u << (b & 31);
            auto repoint = [&](int n) {
                uint32_t* rn = adj + (size_t)n * W;
                if (wa == wb) rn[wa] = (rn[wa] | ma) & ~mb;
                else { rn[wa] |= ma; rn[wb] &= ~mb; }
            };
            for (int w = tid; w < W; w += kAdjMergeThreads) {
                const uint32_t oa = ra[w], ob = rbw[w];
                uint32_t nw = oa | ob;
                if (w == wa) nw &= ~ma;
                if (w == wb) nw &= ~mb;
                ra[w] = nw;
                rbw[w] = 0u;
                // a' neighbour list for the row-a' pass
                uint32_t nbits = nw;
                while (nbits) {
                    const int n = (w << 5) + __ffs(nbits) - 1;
                    nbits &= nbits - 1;
                    nbr[atomicAdd(&misc[kAmNnbr], 1)] = (unsigned short)n;
                }
                uint32_t bits = w == wa ? ob & ~ma : ob;
                while (bits) {
                    const int n = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int k = atomicAdd(&misc[kAmNnb], 1);
                    if (k < kAdjNbList) nbl[k] = (unsigned short)n;
                    else repoint(n);
                }
            }
            adj_bar_merge<kAdjMergeThreads>();
            if (M == kSam && tid == 0) *n2s = norm2_seq(mua, 1, B);  // sequential (oracle order)
            const int nb = min(misc[kAmNnb], kAdjNbList);
            for (int k = tid; k < nb; k += kAdjMergeThreads) repoint(nbl[k]);
        };
        rescan_rows(ni, a, b, merge, AdjShape<NT>::kMergeWarps);
        mark(2);

        // ---- (R) row a': d(a', j) for every neighbour j, offers, a's best ----
        const int nnbr = misc[kAmNnbr];
        const double n2a = M == kSam ? *n2s : 0.0;
        double pd = kInf;
        unsigned pj = 0xffffffffu;
        // per warp, rounds of up to NQ neighbours: the lanes load the neighbours' mean rows
        // (all loads of a round in flight together) and stage the per-band terms in
        // shared memory; then one lane per neighbour runs the ascending-band sum -- a
        // serial chain anyway (a warp-wide shuffle chain would execute it 32 times over)
        const int NQ = max(1, min(kAdjStageNb, kAdjStage / max(B, 1)));
        const int KC = kAdjStage / NQ;  // bands staged per pass (all of them unless B > kAdjStage)
        double* stg = terms + (size_t)warp * kAdjStage;
        for (int t0 = warp * NQ; t0 < nnbr; t0 += kWarps * NQ) {
            const int nq = min(NQ, nnbr - t0);
            double s = 0.0;  // lane q < nq: running ascending-band sum of neighbour t0 + q
            for (int kc0 = 0; kc0 < B; kc0 += KC) {
                const int kc1 = min(B, kc0 + KC);
                for (int k0 = kc0; k0 < kc1; k0 += 32) {
                    const int k = k0 + lane;
                    const bool in = k < kc1;
                    const double m = in ? mua[k] : 0.0;
                    double v[kAdjStageNb];
#pragma unroll
                    for (int q = 0; q < kAdjStageNb; ++q)
                        v[q] = (q < nq && in) ? __ldcg(mr + (size_t)nbr[t0 + q] * B + k) : 0.0;
#pragma unroll
                    for (int q = 0; q < kAdjStageNb; ++q) {
                        if (q < nq && in) {
                            double term;
                            if (M == kSam) term = __dmul_rn(m, v[q]);
                            else {
                                const double df = __dsub_rn(m, v[q]);
                                term = __dmul_rn(df, df);
                            }
                            stg[q * KC + (k - kc0)] = term;
                        }
                    }
                }
                __syncwarp();
                if (lane < nq) {
                    const double* tj = stg + lane * KC;
                    for (int k = 0; k < kc1 - kc0; ++k) s = __dadd_rn(s, tj[k]);
                }
                __syncwarp();  // the staging buffer is rewritten by the next pass
            }
            if (lane < nq) {
                const int j = nbr[t0 + lane];
                const double d = pair_finish<M>(nn, (double)cnt[j], s, n2a, M == kSam ? n2g[j] : 0.0);
                D[(size_t)a * Rp + j] = d;
                D[(size_t)j * Rp + a] = d;
                // rows whose cached neighbour was a or b were rescanned (a, b excluded)
                // above, so every neighbour just takes the offer (d(j, a'), a)
                if (bAj[j] < 0 || d < bAd[j] || (d == bAd[j] && a < bAj[j])) {
                    bAd[j] = d;
                    bAj[j] = a;
                }
                if (d < pd || (d == pd && (unsigned)j < pj)) { pd = d; pj = (unsigned)j; }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, pd, o);
            const unsigned oj = __shfl_xor_sync(0xffffffffu, pj, o);
            if (od < pd || (od == pd && oj < pj)) { pd = od; pj = oj; }
        }
        Pair* scr2 = red + (par ^ 1) * kWarps;
        if (lane == 0) scr2[warp] = Pair{pd, (int)pj, 0};
        __syncthreads();
        mark(3);

        // ---- (E) publish ----
        for (int k = tid; k < B; k += kThreads) mr[(size_t)a * B + k] = mua[k];
        if (M == kSam && tid == 0) bt.nrm2[(size_t)sec * Rp + a] = n2a;
        if (tid == 0) {
            double fd = kInf;
            unsigned fj = 0xffffffffu;
            for (int w = 0; w < kWarps; ++w) {
                const Pair p = scr2[w];
                if (p.d < fd || (p.d == fd && (unsigned)p.lo < fj)) { fd = p.d; fj = (unsigned)p.lo; }
            }
            cnt[a] = (uint32_t)nn;
            cnt[b] = 0u;
            bAd[a] = fd;
            bAj[a] = fj == 0xffffffffu ? -1 : (int)fj;
            bAd[b] = kInf;
            bAj[b] = -1;
            const size_t o = (size_t)sec * Rp + step;
            bt.log_a[o] = a;
            bt.log_b[o] = b;
            bt.log_d[o] = dch;
            bt.log_k[o] = 0;
            bt.parent[(size_t)sec * Rp + b] = a;
            misc[kAmNinv] = 0;
            misc[kAmIctr] = 0;
            misc[kAmNnb] = 0;
            misc[kAmNnbr] = 0;
        }
        __syncthreads();
        mark(4);
        ++step;
    }
    if (prof && tid == 0) {
        pc[7] = (unsigned long long)(clock64() - t_entry);
        for (int q = 0; q < 8; ++q) atomicAdd(bt.prof + q, pc[q]);
    }
    for (int i = tid; i < Rp; i += kThreads) bt.count[(size_t)sec * Rp + i] = cnt[i];
    if (tid == 0) {
        bt.nlog[sec] = step;
        bt.conv[sec] = conv;
        if (bt.pairs) bt.pairs[sec] = 0;
        if (bt.nresc) bt.nresc[sec] = nresc;
    }
}

int launch_adj_loop(const SectionBatch& b, int nrun, int nsm, cudaStream_t st) {
    if (nrun == 0) return 0;
    // many sections: narrow CTAs, more of them resident (RHSEG_ADJ_NT=128|256 forces)
    static const int forced = [] {
        const char* e = getenv("RHSEG_ADJ_NT");
        return e ? atoi(e) : 0;
    }();
    const bool narrow = forced ? forced == 128 : nrun > 2 * nsm;
    void (*kern)(SectionBatch);
#define RHSEG_ADJ_PICK(NT)                                                             \
    kern = b.measure == kSam      ? hseg_adj_kernel<kSam, NT>                          \
           : b.measure == kEuclid ? hseg_adj_kernel<kEuclid, NT>                       \
                                  : hseg_adj_kernel<kBsmse, NT>;
    if (narrow) {
        RHSEG_ADJ_PICK(128)
    } else {
        RHSEG_ADJ_PICK(256)
    }
#undef RHSEG_ADJ_PICK
    const size_t smem = adj_loop_smem(b.Rp, b.B, narrow ? 4 : 8);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<nrun, narrow ? 128 : 256, smem, st>>>(b);
    return cudaGetLastError();
}

}  // namespace rhseg
