// grid_loop.cu -- the HSEG merge loop for sections one thread-block cluster cannot hold.
//
// Reference semantics (rhseg, read-only at /root/reference/pkg/src): engine.py:345-371
// hseg_run / 309-342 hseg_step, _kernels.py:31-115 (per-row best partners, strict < over
// ascending columns), engine.py:281-296 reduce_best, graph.py:229-264 merge_regions; the
// reference runs any section size (sections.py:57-79), so this loop has no region limit
// beyond what D (R^2 fp64) leaves of HBM.
//
// The cluster loop (hseg_kernels.cu) keeps a section's row state in the shared memory of at
// most 16 CTAs (16384 regions). Here a GROUP of G co-resident CTAs (a cooperative launch:
// up to one CTA per SM for one section) owns a section, with the state in HBM:
//   * D [Rp][Rp] exact fp64 dissimilarities (dinit_dense/sparse_kernel), adjacency bitset
//     rows [Rp][W], band-major means mu [B][Rp], region-major sums [Rp][B], a live bitset;
//   * ownership by 32-region chunks dealt round-robin (chunk c -> CTA c % G): CTA g keeps
//     the per-row cached bests (d, partner) of its rows in shared memory, computes d(a', i)
//     for its columns i and rescans its own invalidated rows -- no other CTA writes them.
// No barrier per merge step: each CTA publishes its slot (its rows' best adjacent /
// non-adjacent pair, and its share of row a_prev's new best) as 14 flag-carrying 64-bit
// words (32-bit payload | 32-bit step sequence, single-copy atomic; release-ordered after
// all of the CTA's writes of the step) into 16 replicas, and every CTA polls all G slots of
// its replica (acquire) -- the data arrives with its own flag, and the G^2 reads spread over
// the replicas instead of one hot line. Every CTA combines the G slots redundantly, so the
// decision is identical everywhere without a second exchange:
//   1. combine slots -> row a_prev's caches, the stage minima, the merge rule
//      (engine.py:322-339: spectral if d_s < w * d_a, else adjacent);
//   2. m' = (sums_a + sums_b) / (n_a + n_b) (IEEE, every CTA), then over own columns i:
//      d(a', i) with the reference's op order (dissim.py:33-42), D[i][a] = D[a][i] = d,
//      adjacency re-pointed (b -> a), offers to row i's caches, rows whose partner was a
//      or b queued for a rescan;
//   3. rescans of the queued rows from D (the whole CTA per row, one 32-bit adjacency /
//      live word per 32 columns), then this CTA's minima -> its slot -> group barrier.
// Writes a concurrent reader could see are routed around: the survivor's sums and count
// are published as a pending record and committed one step later (readers of a_prev use
// the record), b's count is zeroed with that commit, liveness comes from the bitset with b
// excluded explicitly in the step that kills it. Cross-CTA data is read with ld.global.cg.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "rhseg_batch.h"
#include "rhseg_device.cuh"

namespace rhseg {

#ifndef RHSEG_GRID_THREADS
#define RHSEG_GRID_THREADS 256  // C1 on the grid loop: 73.4 ms at 512, 69.8 ms at 256 threads
#endif
constexpr int kGT = RHSEG_GRID_THREADS;  // threads per CTA: one CTA per SM
constexpr int kMaxGridCTAs = 160;         // CTAs per section (>= the SM count)
#ifndef RHSEG_GRID_BACKOFF_NS
#define RHSEG_GRID_BACKOFF_NS 64  // slot polling back-off
#endif
constexpr int kGW = kGT / 32;

struct GSlot {
    Pair selA, selN;   // this CTA's best adjacent / non-adjacent pair over its rows
    RowBest rpA, rpN;  // this CTA's part of row a_prev's best over its columns
};
static_assert(sizeof(GSlot) == 64, "slot layout");

struct GPend {  // survivor of the previous step, committed one step later
    int a, b;
    unsigned n;
    int pad;
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// GSlot <-> 14 payload words
constexpr int kSlotWords = 14;
__device__ __forceinline__ uint32_t slot_word(const GSlot& s, int w) {
    auto lo = [](double d) { return (uint32_t)__double2loint(d); };
    auto hi = [](double d) { return (uint32_t)__double2hiint(d); };
    switch (w) {
        case 0: return lo(s.selA.d);
        case 1: return hi(s.selA.d);
        case 2: return (uint32_t)s.selA.lo;
        case 3: return (uint32_t)s.selA.hi;
        case 4: return lo(s.selN.d);
        case 5: return hi(s.selN.d);
        case 6: return (uint32_t)s.selN.lo;
        case 7: return (uint32_t)s.selN.hi;
        case 8: return lo(s.rpA.d);
        case 9: return hi(s.rpA.d);
        case 10: return (uint32_t)s.rpA.j;
        case 11: return lo(s.rpN.d);
        case 12: return hi(s.rpN.d);
        default: return (uint32_t)s.rpN.j;
    }
}
__device__ __forceinline__ GSlot slot_from_words(const uint32_t* w) {
    auto dd = [](uint32_t l, uint32_t h) { return __hiloint2double((int)h, (int)l); };
    GSlot s;
    s.selA = Pair{dd(w[0], w[1]), (int)w[2], (int)w[3]};
    s.selN = Pair{dd(w[4], w[5]), (int)w[6], (int)w[7]};
    s.rpA = RowBest{dd(w[8], w[9]), (int)w[10]};
    s.rpN = RowBest{dd(w[11], w[12]), (int)w[13]};
    return s;
}

__device__ __forceinline__ unsigned ld_acq_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Group barrier over the G CTAs of one section: a monotone arrival counter (zeroed by the
// host before the launch); the k-th barrier completes at G * k arrivals.
__device__ __forceinline__ void group_barrier(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_acq_u32(ctr) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
    return __ldcg(p);
}

__device__ __forceinline__ RowBest rb_min(RowBest x, const RowBest& y) {
    if (y.d < x.d || (y.d == x.d && y.j < x.j)) x = y;
    return x;
}
__device__ __forceinline__ void cache_offer_g(double& cd, int& cj, double d, int j) {
    if (d < kInf && (d < cd || (d == cd && j < cj))) {
        cd = d;
        cj = j;
    }
}

// Block-wide minima of two pairs and two row bests in one shared exchange: warp minima,
// then every warp reduces the kGW per-warp entries with a 5-level butterfly (no serial
// per-thread pass over the entries: that tail dominated the kernel's instruction count).
__device__ __forceinline__ void gslot_min(GSlot& v, const GSlot& c) {
    if (pair_less(c.selA, v.selA)) v.selA = c.selA;
    if (pair_less(c.selN, v.selN)) v.selN = c.selN;
    v.rpA = rb_min(v.rpA, c.rpA);
    v.rpN = rb_min(v.rpN, c.rpN);
}
__device__ __forceinline__ GSlot gslot_shfl(const GSlot& v, int o) {
    GSlot c;
    c.selA.d = __shfl_xor_sync(0xffffffffu, v.selA.d, o);
    c.selA.lo = __shfl_xor_sync(0xffffffffu, v.selA.lo, o);
    c.selA.hi = __shfl_xor_sync(0xffffffffu, v.selA.hi, o);
    c.selN.d = __shfl_xor_sync(0xffffffffu, v.selN.d, o);
    c.selN.lo = __shfl_xor_sync(0xffffffffu, v.selN.lo, o);
    c.selN.hi = __shfl_xor_sync(0xffffffffu, v.selN.hi, o);
    c.rpA.d = __shfl_xor_sync(0xffffffffu, v.rpA.d, o);
    c.rpA.j = __shfl_xor_sync(0xffffffffu, v.rpA.j, o);
    c.rpN.d = __shfl_xor_sync(0xffffffffu, v.rpN.d, o);
    c.rpN.j = __shfl_xor_sync(0xffffffffu, v.rpN.j, o);
    return c;
}
__device__ __forceinline__ GSlot gslot_none() { return GSlot{pair_none(), pair_none(), rb_none(), rb_none()}; }
__device__ __forceinline__ void block_min4(Pair& pa, Pair& pn, RowBest& ra, RowBest& rn, GSlot* scr) {
    GSlot v{pa, pn, ra, rn};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gslot_min(v, gslot_shfl(v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) scr[warp] = v;
    __syncthreads();
    v = lane < kGW ? scr[lane] : gslot_none();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gslot_min(v, gslot_shfl(v, o));
    __syncthreads();
    pa = v.selA;
    pn = v.selN;
    ra = v.rpA;
    rn = v.rpN;
}
// The same for two row bests only (the rescans).
__device__ __forceinline__ void block_min2rb(RowBest& ra, RowBest& rn, GSlot* scr) {
    auto sh = [](RowBest& x, int o) {
        RowBest c;
        c.d = __shfl_xor_sync(0xffffffffu, x.d, o);
        c.j = __shfl_xor_sync(0xffffffffu, x.j, o);
        x = rb_min(x, c);
    };
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sh(ra, o);
        sh(rn, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        scr[warp].rpA = ra;
        scr[warp].rpN = rn;
    }
    __syncthreads();
    ra = lane < kGW ? scr[lane].rpA : rb_none();
    rn = lane < kGW ? scr[lane].rpN : rb_none();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sh(ra, o);
        sh(rn, o);
    }
    __syncthreads();
}

// dynamic shared memory: caches and counts of up to `rows` own rows, m' [B], the rescan
// queue, this CTA's copy of the section's live bitset [W] (kept current locally: every CTA
// knows which region dies each step)
struct GSmem {
    double* cAd;
    double* cNd;
    int* cAj;
    int* cNj;
    uint32_t* cown;
    double* mnew;
    int* queue;
    uint32_t* lsm;
    uint32_t* sw;  // [G][16] polled slot words
    GSlot* scr;
    int* misc;  // [0] queue length
};
__host__ __device__ inline size_t grid_smem_bytes(int rows, int B, int W, int G) {
    return sizeof(GSlot) * kGW + (size_t)rows * (8 + 8 + 4 + 4 + 4) + (size_t)B * 8 + (size_t)rows * 2 * 4 +
           (size_t)W * 4 + (size_t)G * 16 * 4 + 64;
}
__device__ inline GSmem grid_smem(unsigned char* base, int rows, int B, int W, int G) {
    GSmem s;
    s.scr = reinterpret_cast<GSlot*>(base);
    base += sizeof(GSlot) * kGW;
    s.cAd = reinterpret_cast<double*>(base);
    s.cNd = s.cAd + rows;
    s.mnew = s.cNd + rows;
    s.cAj = reinterpret_cast<int*>(s.mnew + B);
    s.cNj = s.cAj + rows;
    s.cown = reinterpret_cast<uint32_t*>(s.cNj + rows);
    s.queue = reinterpret_cast<int*>(s.cown + rows);
    s.lsm = reinterpret_cast<uint32_t*>(s.queue + 2 * rows);
    s.sw = s.lsm + W;
    s.misc = reinterpret_cast<int*>(s.sw + (size_t)G * 16);
    return s;
}

// Rescan row i (section id) over D for stage mask `which` (bit 0 adjacent, bit 1
// non-adjacent) with the whole CTA; column `skip` (the region dying this step) excluded.
// Warp w walks a contiguous range of bitset words: one coalesced load of up to 32 of the
// row's adjacency words, then the D loads of 8 words (256 bytes each) in flight at once,
// liveness from the CTA's shared-memory bitset. Returns the block minima in every thread
// (two __syncthreads inside).
template <bool SPEC>
__device__ __forceinline__ void rescan_row(int i, int which, int skip, const double* __restrict__ D,
                                           const uint32_t* __restrict__ adj, const uint32_t* __restrict__ lsm,
                                           int Rp, int W, RowBest& oA, RowBest& oN, GSlot* scr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t* ar = adj + (size_t)i * W;
    const double* drow = D + (size_t)i * Rp;
    RowBest bA = rb_none(), bN = rb_none();
    const int iw = i >> 5, sw = skip >> 5;
    const uint32_t ib = 1u << (i & 31), sb = skip >= 0 ? 1u << (skip & 31) : 0u;
    const int per = (W + kGW - 1) / kGW, w0 = min(W, warp * per), w1 = min(W, w0 + per);
    for (int base = w0; base < w1; base += 32) {
        const int nwd = min(32, w1 - base);
        const uint32_t aw = lane < nwd ? ldcg(ar + base + lane) : 0u;
        for (int u0 = 0; u0 < nwd; u0 += 8) {
            double dv[8];
            uint32_t sel = 0u;  // bit u: candidate, bit 8 + u: adjacent
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int w = base + u0 + u;
                const uint32_t A = __shfl_sync(0xffffffffu, aw, (u0 + u) & 31);
                uint32_t L = u0 + u < nwd ? lsm[w] : 0u;
                if (w == iw) L &= ~ib;
                if (w == sw) L &= ~sb;
                const uint32_t m = (((which & 1) ? A : 0u) | ((SPEC && (which & 2)) ? ~A : 0u)) & L;
                const bool c = (m >> lane) & 1u;
                dv[u] = c ? ldcg(drow + ((w << 5) | lane)) : kInf;
                sel |= (c ? 1u : 0u) << u;
                sel |= ((A >> lane) & 1u) << (8 + u);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (!((sel >> u) & 1u)) continue;
                const int j = ((base + u0 + u) << 5) | lane;
                if ((sel >> (8 + u)) & 1u) rb_offer(bA, dv[u], j);
                else rb_offer(bN, dv[u], j);
            }
        }
    }
    block_min2rb(bA, bN, scr);
    oA = bA;
    oN = bN;
}

template <bool SPEC, int M>
__global__ void __launch_bounds__(kGT, 1) hseg_grid_kernel(SectionBatch bt) {
    extern __shared__ __align__(16) unsigned char gsm_raw[];
    const int G = bt.G;
    const int g = blockIdx.x % G;
    const int sec = bt.sec0 + blockIdx.x / G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int B = bt.B, Rp = bt.Rp, W = bt.W;
    const int R0 = bt.R0[sec], target = bt.target[sec];
    const int own_ch = g < W ? (W - g + G - 1) / G : 0;  // chunks g, g + G, ...
    const int rows_max = ((W + G - 1) / G) * 32;
    GSmem sm = grid_smem(gsm_raw, rows_max, B, W, G);
    // per-phase cycles (thread 0; RHSEG_PROFILE): combine + rule, column pass, rescans,
    // selection + slot, group barrier
    unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tmark = clock64();
    const long long t_entry = tmark;
    auto mark = [&](int ph) {
        if (bt.prof && tid == 0) {
            const long long t = clock64();
            pc[ph] += (unsigned long long)(t - tmark);
            tmark = t;
        }
    };

    uint32_t* cnt = bt.count + (size_t)sec * Rp;
    double* sums = bt.sums + (size_t)sec * bt.C * bt.sums_copy();  // copy 0
    uint32_t* adj = bt.adj + (size_t)sec * bt.C * bt.adj_copy();
    double* mu = bt.mu + sec * bt.mu_stride();
    double* D = bt.D + (size_t)(sec - bt.sec0) * bt.d_stride();
    double* n2 = M == kSam ? bt.nrm2 + (size_t)sec * Rp : nullptr;
    const GridScrLayout Ly = grid_scr_layout(G, B, W);
    unsigned char* scr = static_cast<unsigned char*>(bt.gscr) + (size_t)sec * Ly.bytes;
    unsigned* ctr = reinterpret_cast<unsigned*>(scr + Ly.bar);
    // slot words [parity][replica][G][16] (flag-carrying; zeroed by the host)
    unsigned long long* slots = reinterpret_cast<unsigned long long*>(scr + Ly.slots);
    const int rep_me = g % kGridSlotRep;
    // publish this CTA's slot for the step that reads sequence `seq` (every thread holds
    // the same values; caller has made all of the CTA's writes precede a __syncthreads)
    auto publish = [&](const GSlot& v, unsigned seq) {
        if (tid < kSlotWords) {
            const unsigned long long word = ((unsigned long long)seq << 32) | slot_word(v, tid);
            fence_acq_rel_gpu();  // release: the CTA's writes of this step (ordered by the barrier)
            const int par = (int)((seq - 1) & 1);
#pragma unroll 4
            for (int r = 0; r < kGridSlotRep; ++r)
                st_relaxed_u64(slots + ((size_t)(par * kGridSlotRep + r) * G + g) * 16 + tid, word);
        }
    };
    // poll every slot of sequence `seq` (acquire) and combine them
    auto collect = [&](unsigned seq, Pair& sA, Pair& sN, RowBest& rA, RowBest& rN) {
        const int par = (int)((seq - 1) & 1);
        const unsigned long long* base = slots + (size_t)(par * kGridSlotRep + rep_me) * G * 16;
        // this thread's words (G * 16 <= K * kGT), all polls in flight at once, a short
        // back-off between rounds so the spinning does not crowd out the step's own L2
        // traffic
        constexpr int K = (kMaxGridCTAs * 16 + kGT - 1) / kGT;
        uint32_t pend = 0u;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int e = tid + k * kGT;
            if (e < G * 16 && (e & 15) < kSlotWords) pend |= 1u << k;
        }
        while (pend) {
            unsigned long long v[K];
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = ((pend >> k) & 1u) ? ld_relaxed_u64(base + tid + k * kGT) : 0ull;
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (((pend >> k) & 1u) && (unsigned)(v[k] >> 32) == seq) {
                    sm.sw[tid + k * kGT] = (uint32_t)v[k];
                    pend &= ~(1u << k);
                }
            if (pend) __nanosleep(RHSEG_GRID_BACKOFF_NS);
        }
        fence_acq_rel_gpu();  // acquire: the producers' writes before their slot words
        __syncthreads();
        for (int q = tid; q < G; q += kGT) {
            const GSlot x = slot_from_words(sm.sw + (size_t)q * 16);
            pair_offer(sA, x.selA);
            pair_offer(sN, x.selN);
            rA = rb_min(rA, x.rpA);
            rN = rb_min(rN, x.rpN);
        }
        block_min4(sA, sN, rA, rN, sm.scr);
    };
    unsigned char* pendb = scr + Ly.pend;                     // [2] x (GPend, sums[B])
    uint32_t* live = reinterpret_cast<uint32_t*>(scr + Ly.live);  // (prologue exchange only)
    long long* acc = reinterpret_cast<long long*>(scr + Ly.acc);
    auto pend_hdr = [&](int p) { return reinterpret_cast<GPend*>(pendb + (size_t)p * Ly.pend_each); };
    auto pend_sums = [&](int p) { return reinterpret_cast<double*>(pendb + (size_t)p * Ly.pend_each + 16); };
    auto row_id = [&](int r) { return ((g + (r >> 5) * G) << 5) | (r & 31); };
    auto owner = [&](int id) { return (id >> 5) % G; };
    auto row_loc = [&](int id) { return (((id >> 5) / G) << 5) | (id & 31); };

    if (R0 <= target) {  // nothing to merge (hseg_run's loop never starts)
        if (g == 0 && tid == 0) {
            bt.nlog[sec] = 0;
            bt.conv[sec] = 0;
        }
        return;
    }
    unsigned nbar = 0;
    // ---- prologue: live bits of own chunks, then every own row's bests from D ----
    for (int k = warp; k < own_ch; k += kGW) {
        const int c = g + k * G, i = (c << 5) | lane;
        const uint32_t n = i < R0 ? cnt[i] : 0u;
        sm.cown[(k << 5) | lane] = n;
        const unsigned m = __ballot_sync(0xffffffffu, n != 0u);
        if (lane == 0) live[c] = m;
    }
    group_barrier(ctr, G * ++nbar);
    for (int w = tid; w < W; w += kGT) sm.lsm[w] = ldcg(live + w);
    __syncthreads();
    long long e2 = 0, e2acc = 0, nresc = 0, pairs_top = 0;  // spectral-pair accounting (see epilogue)
    for (int r = 0; r < own_ch * 32; ++r) {
        const int i = row_id(r);
        const bool isl = (sm.lsm[i >> 5] >> (i & 31)) & 1u;  // (uniform over the CTA)
        RowBest bA = rb_none(), bN = rb_none();
        if (isl) rescan_row<SPEC>(i, SPEC ? 3 : 1, -1, D, adj, sm.lsm, Rp, W, bA, bN, sm.scr);
        if (tid == 0) {
            sm.cAd[r] = bA.d;
            sm.cAj[r] = bA.j;
            sm.cNd[r] = bN.d;
            sm.cNj[r] = bN.j;
        }
        if (SPEC && isl) {  // 2E: the degrees of the live rows
            const uint32_t* ar = adj + (size_t)i * W;
            for (int w = tid; w < W; w += kGT) e2 += __popc(ldcg(ar + w));
        }
    }
    __syncthreads();
    {
        Pair pA = pair_none(), pN = pair_none();
        RowBest xA = rb_none(), xN = rb_none();
        for (int r = tid; r < own_ch * 32; r += kGT) {
            const int i = row_id(r);
            if (!((sm.lsm[i >> 5] >> (i & 31)) & 1u)) continue;
            pair_offer(pA, make_pair(sm.cAd[r], i, sm.cAj[r]));
            if (SPEC) pair_offer(pN, make_pair(sm.cNd[r], i, sm.cNj[r]));
        }
        block_min4(pA, pN, xA, xN, sm.scr);
        publish(GSlot{pA, pN, xA, xN}, 1u);
    }
    if (bt.prof && tid == 0) {
        pc[6] = (unsigned long long)(clock64() - t_entry);
        tmark = clock64();
    }

    // ---- merge loop ----
    int step = 0, a_prev = -1, conv = 0;
    unsigned n_prev = 0;
    for (;; ++step) {
        if (R0 - step <= target) break;
        // 1. combine the slots (every CTA identically)
        Pair sA = pair_none(), sN = pair_none();
        RowBest rA = rb_none(), rN = rb_none();
        collect((unsigned)step + 1u, sA, sN, rA, rN);
        if (a_prev >= 0) {
            if (owner(a_prev) == g && tid == 0) {
                const int r = row_loc(a_prev);
                sm.cAd[r] = rA.d;
                sm.cAj[r] = rA.j;
                sm.cNd[r] = rN.d;
                sm.cNj[r] = rN.j;
            }
            pair_offer(sA, make_pair(rA.d, a_prev, rA.j));
            if (SPEC) pair_offer(sN, make_pair(rN.d, a_prev, rN.j));
        }
        int kind = -1;
        Pair ch = pair_none();
        if (SPEC && sN.d < kInf) {
            const double dA = sA.d < kInf ? sA.d : kInf;
            if (sN.d < __dmul_rn(bt.weight, dA)) {
                ch = sN;
                kind = 1;
            }
        }
        if (kind < 0 && sA.d < kInf) {
            ch = sA;
            kind = 0;
        }
        if (kind < 0) {
            conv = 1;
            break;
        }
        const int a = ch.lo, b = ch.hi;
        mark(0);
        // 2. the survivor's sums / mean (pending record of a_prev for reads of a_prev)
        const GPend* pp = step > 0 ? pend_hdr((step - 1) & 1) : nullptr;
        const double* ps = step > 0 ? pend_sums((step - 1) & 1) : nullptr;
        const unsigned na = (a == a_prev) ? n_prev : ldcg(cnt + a);
        const unsigned nb = (b == a_prev) ? n_prev : ldcg(cnt + b);
        const unsigned nn = na + nb;
        const double dn = (double)nn;
        const int cur = step & 1;
        double* psn = pend_sums(cur);
        for (int k = tid; k < B; k += kGT) {
            const double sa = (a == a_prev) ? ldcg(ps + k) : ldcg(sums + (size_t)a * B + k);
            const double sb = (b == a_prev) ? ldcg(ps + k) : ldcg(sums + (size_t)b * B + k);
            const double s = __dadd_rn(sa, sb);
            const double m = __ddiv_rn(s, dn);
            sm.mnew[k] = m;
            if (g == 0) psn[k] = s;
            if (owner(a) == g) mu[(size_t)k * Rp + a] = m;
        }
        if (g == 0) {
            // commit the previous step's survivor (nobody reads these words this step:
            // a_prev's readers use the pending record, b_prev is dead)
            if (step > 0) {
                const int ap = pp->a, bp = pp->b;
                for (int k = tid; k < B; k += kGT) sums[(size_t)ap * B + k] = ldcg(ps + k);
                if (tid == 0) {
                    cnt[ap] = pp->n;
                    cnt[bp] = 0u;
                }
            }
            if (tid == 0) {
                GPend* h = pend_hdr(cur);
                h->a = a;
                h->b = b;
                h->n = nn;
                const size_t o = (size_t)sec * Rp + step;
                bt.log_a[o] = a;
                bt.log_b[o] = b;
                bt.log_d[o] = ch.d;
                bt.log_k[o] = (uint8_t)kind;
                bt.parent[(size_t)sec * Rp + b] = a;
                if (SPEC) {
                    const long long R = R0 - step;
                    pairs_top += R * (R - 1) / 2;
                }
            }
        }
        if (tid == 0) {
            sm.misc[0] = 0;
            sm.lsm[b >> 5] &= ~(1u << (b & 31));
            if (owner(a) == g) sm.cown[row_loc(a)] = nn;
            if (owner(b) == g) sm.cown[row_loc(b)] = 0u;
        }
        __syncthreads();  // m', live bits, own counts visible; queue empty
        double n2new = 0.0;
        if (M == kSam) {
            n2new = norm2_seq(sm.mnew, 1, B);  // every thread, same bits (oracle inc_mean order)
            if (owner(a) == g && tid == 0) n2[a] = n2new;
        }
        // 3. own columns: d(a', i), adjacency re-point, offers, rescan queue
        if (SPEC) e2acc += e2;
        RowBest pA = rb_none(), pN = rb_none();
        for (int k = warp; k < own_ch; k += kGW) {
            const int c = g + k * G, i = (c << 5) | lane;
            const uint32_t Aw = ldcg(adj + (size_t)a * W + c), Bw = ldcg(adj + (size_t)b * W + c);
            const uint32_t Lw = sm.lsm[c];
            uint32_t Nw = Aw | Bw;
            if (c == (a >> 5)) Nw &= ~(1u << (a & 31));
            if (c == (b >> 5)) Nw &= ~(1u << (b & 31));
            __syncwarp();
            if (lane == 0) {
                adj[(size_t)a * W + c] = Nw;
                adj[(size_t)b * W + c] = 0u;
                if (SPEC) {
                    e2 += 2LL * (__popc(Nw) - __popc(Aw) - __popc(Bw));
                    if (c == (b >> 5) && ((Aw >> (b & 31)) & 1u)) e2 += 2;  // the edge (a, b) itself
                }
            }
            const bool isl = ((Lw >> lane) & 1u) && i != a && i != b;
            if (!isl) continue;
            const bool adjn = (Nw >> lane) & 1u;
            double d = kInf;
            if (SPEC || adjn) {
                const unsigned ni = sm.cown[(k << 5) | lane];
                double s = 0.0;
                const double* mc = mu + i;
#pragma unroll 8
                for (int q = 0; q < B; ++q) s = acc_step<M>(s, sm.mnew[q], mc[(size_t)q * Rp]);
                d = pair_finish<M>(dn, (double)ni, s, n2new, M == kSam ? n2[i] : 0.0);
                D[(size_t)i * Rp + a] = d;
                D[(size_t)a * Rp + i] = d;
                if (adjn) rb_offer(pA, d, i);
                else rb_offer(pN, d, i);
            }
            if ((Bw >> lane) & 1u) {  // row i: b -> a (graph.py:240-247)
                uint32_t* ar = adj + (size_t)i * W;
                if ((a >> 5) == (b >> 5)) {
                    ar[a >> 5] = (ar[a >> 5] & ~(1u << (b & 31))) | (1u << (a & 31));
                } else {
                    ar[b >> 5] &= ~(1u << (b & 31));
                    ar[a >> 5] |= 1u << (a & 31);
                }
            }
            const int r = (k << 5) | lane;
            int q = 0;
            if (sm.cAj[r] == a || sm.cAj[r] == b) q |= 1;
            else if (adjn) cache_offer_g(sm.cAd[r], sm.cAj[r], d, a);
            if (SPEC) {
                if (sm.cNj[r] == a || sm.cNj[r] == b) q |= 2;
                else if (!adjn) cache_offer_g(sm.cNd[r], sm.cNj[r], d, a);
            }
            if (q) sm.queue[atomicAdd(&sm.misc[0], 1)] = (r << 2) | q;
        }
        __syncthreads();
        mark(1);
        // 4. rescans of the queued rows (each over the whole CTA)
        const int nq = sm.misc[0];
        for (int e = 0; e < nq; ++e) {
            const int qe = sm.queue[e], r = qe >> 2, which = qe & 3;
            RowBest bA, bN;
            rescan_row<SPEC>(row_id(r), which, b, D, adj, sm.lsm, Rp, W, bA, bN, sm.scr);
            if (tid == 0) {
                if (which & 1) {
                    sm.cAd[r] = bA.d;
                    sm.cAj[r] = bA.j;
                }
                if (which & 2) {
                    sm.cNd[r] = bN.d;
                    sm.cNj[r] = bN.j;
                }
            }
        }
        if (tid == 0) nresc += nq;
        __syncthreads();
        mark(2);
        // 5. this CTA's minima (rows other than a and b) and its part of row a's best
        {
            Pair xA = pair_none(), xN = pair_none();
            for (int r = tid; r < own_ch * 32; r += kGT) {
                const int i = row_id(r);
                if (i == a || i == b || !((sm.lsm[i >> 5] >> (i & 31)) & 1u)) continue;
                pair_offer(xA, make_pair(sm.cAd[r], i, sm.cAj[r]));
                if (SPEC) pair_offer(xN, make_pair(sm.cNd[r], i, sm.cNj[r]));
            }
            block_min4(xA, xN, pA, pN, sm.scr);
            publish(GSlot{xA, xN, pA, pN}, (unsigned)step + 2u);
        }
        mark(3);
        a_prev = a;
        n_prev = nn;
    }
    // ---- epilogue: commit the last survivor, counters ----
    if (g == 0 && step > 0) {
        const GPend* pp = pend_hdr((step - 1) & 1);
        const double* ps = pend_sums((step - 1) & 1);
        for (int k = tid; k < B; k += kGT) sums[(size_t)pp->a * B + k] = ldcg(ps + k);
        if (tid == 0) {
            cnt[pp->a] = pp->n;
            cnt[pp->b] = 0u;
        }
    }
    // spectral pairs the reference evaluates: sum_t R_t (R_t - 1) / 2 - E_t, E_t = (sum of
    // every CTA's share of 2E) / 2
    if (SPEC) {
        // e2acc per thread: lanes 0 hold their warps' shares; fold over the block
        long long v = e2acc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(acc), (unsigned long long)v);
    }
    if (tid == 0 && nresc) atomicAdd(reinterpret_cast<unsigned long long*>(acc + 1), (unsigned long long)nresc);
    if (bt.prof && tid == 0) {
        pc[5] = (unsigned long long)nresc;
        pc[7] = (unsigned long long)(clock64() - t_entry);
        for (int q = 0; q < 8; ++q) atomicAdd(bt.prof + q, pc[q]);
    }
    group_barrier(ctr, G * ++nbar);
    if (g == 0 && tid == 0) {
        bt.nlog[sec] = step;
        bt.conv[sec] = conv;
        if (bt.pairs) bt.pairs[sec] = SPEC ? pairs_top - ldcg(acc) / 2 : 0;
        if (bt.nresc) bt.nresc[sec] = ldcg(acc + 1);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
template <bool SPEC, int M>
static void* grid_kernel_ptr() {
    return reinterpret_cast<void*>(hseg_grid_kernel<SPEC, M>);
}
static void* pick_grid_kernel(bool spec, int measure) {
    if (measure == kSam) return spec ? grid_kernel_ptr<true, kSam>() : grid_kernel_ptr<false, kSam>();
    if (measure == kEuclid) return spec ? grid_kernel_ptr<true, kEuclid>() : grid_kernel_ptr<false, kEuclid>();
    return spec ? grid_kernel_ptr<true, kBsmse>() : grid_kernel_ptr<false, kBsmse>();
}

int grid_loop_resident(int nsm) {
    // one CTA per SM by construction (__launch_bounds__(kGT, 1), <= ~60 KB of shared memory)
    return std::min(nsm, kMaxGridCTAs);
}

int launch_grid_loop(const SectionBatch& b0, int nrun, int nsm, cudaStream_t st, int* G_used) {
    if (nrun == 0) return 0;
    const int total = grid_loop_resident(nsm);
    const int per = std::min(nrun, total);  // sections per launch
    void* kern = pick_grid_kernel(b0.spec != 0, b0.measure);
    for (int s0 = 0; s0 < nrun; s0 += per) {
        const int n = std::min(per, nrun - s0);
        SectionBatch b = b0;
        b.sec0 = b0.sec0 + s0;
        b.D = b0.D + (size_t)s0 * b0.d_stride();
        b.G = std::max(1, std::min(b.W, total / n));
        if (b0.G > 0) b.G = std::min(b.G, b0.G);  // host cap (RHSEG_GRID_CTAS)
        if (G_used) *G_used = b.G;
        const int rows = ((b.W + b.G - 1) / b.G) * 32;
        const size_t smem = grid_smem_bytes(rows, b.B, b.W, b.G);
        const GridScrLayout Ly = grid_scr_layout(b.G, b.B, b.W);
        cudaError_t e = cudaMemsetAsync(static_cast<unsigned char*>(b.gscr) + (size_t)b.sec0 * Ly.bytes, 0,
                                        (size_t)n * Ly.bytes, st);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(n * b.G), 1, 1);
        cfg.blockDim = dim3(kGT, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;  // co-residency of the group is required
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        void* args[] = {&b};
        e = cudaLaunchKernelExC(&cfg, kern, args);
        if (e != cudaSuccess) return e;
    }
    return 0;
}

size_t grid_loop_scratch_bytes(int nsm, int B, int W) {
    // per section, for the largest group a launch can form
    return grid_scr_layout(grid_loop_resident(nsm), B, W).bytes;
}

}  // namespace rhseg
