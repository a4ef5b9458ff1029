// apo_loop.cu -- the APO merge loop: HSEG region growing for w > 0 (BSMSE / Euclidean),
// one CTA per section, every section of a quadtree level in one persistent launch.
//
// Reference semantics (rhseg, read-only at /root/reference/pkg/src):
//   engine.py:309-342 hseg_step, engine.py:345-371 hseg_run, _kernels.py:31-115 (per-row
//   best partner, fp64, strict <, ascending columns), engine.py:281-296 reduce_best
//   (lexicographic (d, min id, max id)), engine.py:322-339 merge rule (spectral iff
//   d_s < w * d_a), graph.py:229-264 merge_regions (smaller id survives).
//
// Same invariants as the first APO variant in hseg_kernels.cu (D holds exact values or
// rigorous intervals around them, apo_device.cuh; per-row cached bests equal the
// reference's per-row table entries; exact values wherever a comparison needs them),
// with the step re-cut around its latency chain (round 1 measured ~47k cycles per step
// on a C4 leaf, half of it in rescans serialised per warp, the rest in ~12 barrier-
// separated phases with a dependent global round trip in most of them):
//
//  (A) argmin: ONE pass over the row caches keeps, per stage, the smallest lower bound
//      and its pair, the smallest lower bound of any other pair and the smallest upper
//      bound; the winner is unique iff no other pair can reach below that upper bound
//      (one block reduction; the exact tie-break pass only when it is not unique).
//  (C) rows whose cached partner is a or b are listed; D rows a and b start streaming
//      into shared memory (cp.async) for the row-a' pass.
//  (X) merge || rescans: two warps merge (band sums, mean, adjacency union, neighbour
//      re-point); every other warp -- and the merge warps once done -- claims rescan
//      CHUNKS (128 columns of one invalidated row) from a shared counter and folds them
//      into per-chunk key partials. A rescan excludes a and b, and reads nothing the
//      merge writes (row caches of other rows, D rows, the live set before the merge),
//      so the two are independent; a row costs one round trip per chunk instead of
//      R0/128 sequential ones, spread over all warps.
//  (F) finalize: one warp per invalidated row combines its chunk partials (exact
//      fallback when the two best keys are within their intervals).
//  (R) row a': intervals from the shared copies of D rows a and b, written to D, offered
//      to every row's cache in the same pass, and a's own best by the same unique-or-
//      exact reduction as (A).
//  (E) one thread publishes the merge (counts, live set, log, a's caches).
#include <cuda_runtime.h>

#include "apo_device.cuh"
#include "rhseg_batch.h"
#include "rhseg_device.cuh"

namespace rhseg {

#ifndef RHSEG_APO_MERGE_WARPS
#define RHSEG_APO_MERGE_WARPS 2  // warps that merge while the others start the rescans
#endif
#ifndef RHSEG_APO_PARTS
#define RHSEG_APO_PARTS 256  // rescan chunk partials per batch (shared memory)
#endif
#ifndef RHSEG_APO_COMPACT
#define RHSEG_APO_COMPACT 8  // compact the live-column list when holes >= S / K
#endif
constexpr int kApoMergeThreads = RHSEG_APO_MERGE_WARPS * 32;
constexpr int kApoNbList = 256;
constexpr unsigned long long kKeyHi = 0x7fffffffffffc000ULL, kKeyNone = ~0ULL;
constexpr unsigned kPairNone = 0xffffffffu;
#define RHSEG_UNPACKED __longlong_as_double(0x7ff8000000000001LL)  // row a' entry too wide to store

// Two smallest 64-bit keys of one stage (D bits, sign cleared, truncated by 14 bits,
// column id in the low 14 bits: non-negative doubles order like their bit patterns)
// and the D value of the smallest.
struct RsPart {
    unsigned long long a1, a2, n1, n2;
    double va, vn;
    int km, pad[3];
};
static_assert(sizeof(RsPart) == 64, "rescan partial");

// Per-stage state of the unique-or-exact reductions (argmin over row caches, a's best
// over row a'): smallest lower bound l1 with its key k1 and value v1, the smallest
// lower bound of any other key l2, the smallest upper bound u.
struct ArgSt {
    double l1, v1, l2, u;
    unsigned k1;
    int pad;
};
__device__ __forceinline__ ArgSt as_none() { return ArgSt{kInf, kInf, kInf, kInf, kPairNone, 0}; }
__device__ __forceinline__ void as_put(ArgSt& x, double l, double h, unsigned key, double v) {
    x.u = fmin(x.u, h);
    if (key == x.k1) {
        if (l < x.l1) { x.l1 = l; x.v1 = v; }
    } else if (l < x.l1 || (l == x.l1 && key < x.k1)) {
        x.l2 = fmin(x.l2, x.l1);
        x.l1 = l; x.k1 = key; x.v1 = v;
    } else {
        x.l2 = fmin(x.l2, l);
    }
}
__device__ __forceinline__ void as_merge(ArgSt& x, const ArgSt& y) {
    x.u = fmin(x.u, y.u);
    if (y.k1 == kPairNone) return;
    if (y.k1 == x.k1) {
        if (y.l1 < x.l1) { x.l1 = y.l1; x.v1 = y.v1; }
        x.l2 = fmin(x.l2, y.l2);
    } else if (y.l1 < x.l1 || (y.l1 == x.l1 && y.k1 < x.k1)) {
        x.l2 = fmin(y.l2, x.l1);
        x.l1 = y.l1; x.k1 = y.k1; x.v1 = y.v1;
    } else {
        x.l2 = fmin(x.l2, y.l1);
    }
}
__device__ __forceinline__ ArgSt as_shfl(const ArgSt& x, int o) {
    ArgSt y;
    y.l1 = __shfl_xor_sync(0xffffffffu, x.l1, o);
    y.v1 = __shfl_xor_sync(0xffffffffu, x.v1, o);
    y.l2 = __shfl_xor_sync(0xffffffffu, x.l2, o);
    y.u = __shfl_xor_sync(0xffffffffu, x.u, o);
    y.k1 = __shfl_xor_sync(0xffffffffu, x.k1, o);
    y.pad = 0;
    return y;
}
// block-wide reduction of two stages; scratch holds [kWarps][2] entries (callers
// alternate two scratch buffers by step parity, so one barrier suffices)
__device__ __forceinline__ void as_block2(ArgSt& x, ArgSt& y, ArgSt* scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const ArgSt ox = as_shfl(x, o), oy = as_shfl(y, o);
        as_merge(x, ox);
        as_merge(y, oy);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        scratch[2 * warp] = x;
        scratch[2 * warp + 1] = y;
    }
    __syncthreads();
    x = scratch[0];
    y = scratch[1];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) {
        as_merge(x, scratch[2 * w]);
        as_merge(y, scratch[2 * w + 1]);
    }
}
__device__ __forceinline__ bool as_unique(const ArgSt& x) { return x.k1 != kPairNone && x.l2 > x.u; }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void bar_merge() {  // named barrier of the merge warps
    asm volatile("bar.sync 1, %0;" ::"n"(kApoMergeThreads) : "memory");
}

struct ApoSmem {
    size_t misc, red, pscr, rscr, part, cnt, bAd, bNd, bAj, bNj, inv, col, slot_of, ver, livew, sra, nbl, mua, rowA,
        rowB, total;
};
__host__ __device__ inline size_t apo_align(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline ApoSmem apo_smem_layout(int Rp, int B) {
    ApoSmem L;
    const size_t R = (size_t)Rp, W = (size_t)(Rp / 32);
    size_t o = 0;
    L.misc = o;    o += 128;
    L.red = o;     o += 2 * kWarps * 2 * sizeof(ArgSt);  // [parity][warp][stage]
    L.pscr = o;    o += 2 * kWarps * sizeof(Pair);
    L.rscr = o;    o += 2 * kWarps * sizeof(RowBest);
    o = (o + 63) & ~size_t(63);
    L.part = o;    o += (size_t)RHSEG_APO_PARTS * sizeof(RsPart);
    L.cnt = o;     o = apo_align(o + R * 4);
    L.bAd = o;     o = apo_align(o + R * 8);
    L.bNd = o;     o = apo_align(o + R * 8);
    L.bAj = o;     o = apo_align(o + R * 4);
    L.bNj = o;     o = apo_align(o + R * 4);
    L.inv = o;     o = apo_align(o + R * 4);  // invalidated rows; later two ushort lists
    L.col = o;     o = apo_align(o + R * 2);  // compacted live columns (ascending, holes -1)
    L.slot_of = o; o = apo_align(o + R * 2);
    L.ver = o;     o = apo_align(o + R * 2);  // region -> row of the versioned means
    L.livew = o;   o = apo_align(o + W * 4);
    L.sra = o;     o = apo_align(o + W * 4);  // a's new adjacency row
    L.nbl = o;     o = apo_align(o + kApoNbList * 2);
    L.mua = o;     o = apo_align(o + (size_t)B * 8);
    L.rowA = o;    o = apo_align(o + R * 8);  // D rows a and b of the current step
    L.rowB = o;    o = apo_align(o + R * 8);
    L.total = o;
    return L;
}
size_t apo_loop_smem(int Rp, int B) { return apo_smem_layout(Rp, B).total; }

// misc[] slots
enum { kMiscNinv = 0, kMiscIctr, kMiscNnb, kMiscDE, kMiscN1, kMiscN2, kMiscNc, kMiscNx = 8 };

template <int M>
__global__ void __launch_bounds__(kThreads, 2) hseg_apo_kernel(SectionBatch bt) {
    extern __shared__ __align__(128) unsigned char smem[];
    const long long t_entry = clock64();
    const int sec = bt.sec0 + (int)blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R0 = bt.R0[sec];
    const int B = bt.B, Rp = bt.Rp, W = bt.W;
    const int Wr = (R0 + 31) >> 5;  // bitset words holding ids < R0
    const int target = bt.target[sec];
    const ApoSmem L = apo_smem_layout(Rp, B);
    int* misc = reinterpret_cast<int*>(smem + L.misc);
    ArgSt* red = reinterpret_cast<ArgSt*>(smem + L.red);
    Pair* pscr = reinterpret_cast<Pair*>(smem + L.pscr);
    RowBest* rscr = reinterpret_cast<RowBest*>(smem + L.rscr);
    RsPart* part = reinterpret_cast<RsPart*>(smem + L.part);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L.cnt);
    double* bAd = reinterpret_cast<double*>(smem + L.bAd);
    double* bNd = reinterpret_cast<double*>(smem + L.bNd);
    int* bAj = reinterpret_cast<int*>(smem + L.bAj);
    int* bNj = reinterpret_cast<int*>(smem + L.bNj);
    int* inv = reinterpret_cast<int*>(smem + L.inv);
    short* col = reinterpret_cast<short*>(smem + L.col);
    short* slot_of = reinterpret_cast<short*>(smem + L.slot_of);
    unsigned short* ver = reinterpret_cast<unsigned short*>(smem + L.ver);
    uint32_t* livew = reinterpret_cast<uint32_t*>(smem + L.livew);
    uint32_t* sra = reinterpret_cast<uint32_t*>(smem + L.sra);
    unsigned short* nbl = reinterpret_cast<unsigned short*>(smem + L.nbl);
    double* mua = reinterpret_cast<double*>(smem + L.mua);
    double* rowA = reinterpret_cast<double*>(smem + L.rowA);
    double* rowB = reinterpret_cast<double*>(smem + L.rowB);
    unsigned long long* sE0 = reinterpret_cast<unsigned long long*>(misc + kMiscNx);
    double* sx = reinterpret_cast<double*>(misc + kMiscNx + 2);
    double* xs = reinterpret_cast<double*>(misc + kMiscNx + 4);  // [2] exact d of the rule

    const double* const mu0 = bt.mu + sec * bt.mu_stride();     // band-major initial means
    double* const mr = bt.mu2 + 2 * sec * bt.mu_stride();      // versioned region-major means
    double* __restrict__ D = bt.D + (sec - bt.sec0) * bt.d_stride();
    double* __restrict__ sums = bt.sums + (size_t)sec * bt.sums_copy();
    uint32_t* __restrict__ adj = bt.adj + (size_t)sec * bt.adj_copy();
    const bool prof = bt.prof != nullptr;

    int S = R0, holes = 0;  // live-column list length (holes = -1 entries)

    // ---- exact d(i, j) by one warp from the versioned means; lane 0 writes D back ----
    auto exact_pair = [&](int i, int j) {
        const long long t0 = clock64();
        const double d = warp_exact<M>(mr + (size_t)ver[i] * B, mr + (size_t)ver[j] * B, (double)cnt[i],
                                       (double)cnt[j], B, lane);
        if (prof && lane == 0) {
            atomicAdd(bt.prof + 11, 1ull);
            atomicAdd(bt.prof + 12, (unsigned long long)(clock64() - t0));
        }
        if (lane == 0) {
            D[(size_t)i * Rp + j] = d;
            D[(size_t)j * Rp + i] = d;
        }
        return d;
    };

    // ---- exact fallback rescan of row i (the whole warp): the minimum of every entry
    // whose lower bound reaches the stage's smallest upper bound (intervals evaluated
    // exactly). Columns exA / exB excluded (a and b of the step). ----
    auto rescan_exact = [&](int i, int mask, int exA, int exB) {
        const uint32_t* arow = adj + (size_t)i * W;
        const double* drow = D + (size_t)i * Rp;
        double uA = kInf, uN = kInf;
        for (int s0 = 0; s0 < S; s0 += 32) {
            const int sl = s0 + lane;
            const int j = sl < S ? col[sl] : -1;
            if (j >= 0 && j != i && j != exA && j != exB && ((livew[j >> 5] >> (j & 31)) & 1u)) {
                const bool aj = (arow[j >> 5] >> (j & 31)) & 1u;
                if (aj ? (mask & 1) : (mask & 2)) {
                    double l2, h2;
                    d_unpack(__ldcg(drow + j), l2, h2);
                    if (aj) uA = fmin(uA, h2);
                    else uN = fmin(uN, h2);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uA = fmin(uA, __shfl_xor_sync(0xffffffffu, uA, o));
            uN = fmin(uN, __shfl_xor_sync(0xffffffffu, uN, o));
        }
        RowBest ba = rb_none(), bn = rb_none();
        for (int s0 = 0; s0 < S; s0 += 32) {
            const int sl = s0 + lane;
            const int j = sl < S ? col[sl] : -1;
            bool cand = false, aj = false;
            double v = kInf;
            if (j >= 0 && j != i && j != exA && j != exB && ((livew[j >> 5] >> (j & 31)) & 1u)) {
                aj = (arow[j >> 5] >> (j & 31)) & 1u;
                if (aj ? (mask & 1) : (mask & 2)) {
                    v = __ldcg(drow + j);
                    double l2, h2;
                    d_unpack(v, l2, h2);
                    cand = l2 <= (aj ? uA : uN);
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
        ba = warp_min_rb(ba);
        bn = warp_min_rb(bn);
        if (lane == 0) {
            if (mask & 1) { bAd[i] = ba.d; bAj[i] = ba.j == kNoJ ? -1 : ba.j; }
            if (mask & 2) { bNd[i] = bn.d; bNj[i] = bn.j == kNoJ ? -1 : bn.j; }
        }
    };

    // ---- rescan chunks: 128 columns of one listed row -> one key partial ----
    // dense: bitset words [4c, 4c+4) (lane l takes id 32w + l, coalesced D loads);
    // sparse (most regions merged away): live-column list slots [128c, 128c+128)
    struct Chunk {
        double dv[4];
        uint32_t sel;  // per u: bit 2u candidate, bit 2u+1 adjacent
        int c;         // chunk index (the column ids are recomputed in the fold)
    };
    auto chunk_load = [&](Chunk& ck, int i, int mask, int c, bool dense, int exA, int exB) {
        const uint32_t* arow = adj + (size_t)i * W;
        const double* drow = D + (size_t)i * Rp;
        ck.sel = 0u;
        ck.c = c;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int j;
            bool live, aj;
            if (dense) {
                const int w = 4 * c + u;
                const uint32_t lw = w < Wr ? livew[w] : 0u, aw = w < Wr ? arow[w] : 0u;
                j = (w << 5) + lane;
                live = (lw >> lane) & 1u;
                aj = (aw >> lane) & 1u;
            } else {
                const int sl = 128 * c + 32 * u + lane;
                j = sl < S ? col[sl] : -1;
                live = j >= 0 && ((livew[j >> 5] >> (j & 31)) & 1u);
                aj = live && ((arow[j >> 5] >> (j & 31)) & 1u);
            }
            const bool cnd = live && j != i && j != exA && j != exB && (aj ? (mask & 1) : (mask & 2));
            ck.sel |= (cnd ? 1u : 0u) << (2 * u) | (aj ? 2u : 0u) << (2 * u);
            ck.dv[u] = cnd ? __ldcs(drow + j) : 0.0;
        }
    };
    auto chunk_fold = [&](const Chunk& ck, bool dense, RsPart* out) {
        unsigned long long a1 = kKeyNone, a2 = kKeyNone, n1 = kKeyNone, n2 = kKeyNone;
        double va = 0.0, vn = 0.0;
        int km = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (!((ck.sel >> (2 * u)) & 1u)) continue;
            const unsigned long long r = (unsigned long long)__double_as_longlong(ck.dv[u]);
            km = max(km, (int)(r >> 63) * (int)(r & 63));
            const int j = dense ? ((4 * ck.c + u) << 5) + lane : col[128 * ck.c + 32 * u + lane];
            const unsigned long long key = (r & kKeyHi) | (unsigned long long)j;
            if ((ck.sel >> (2 * u + 1)) & 1u) {
                if (key < a1) { a2 = a1; a1 = key; va = ck.dv[u]; }
                else a2 = min(a2, key);
            } else {
                if (key < n1) { n2 = n1; n1 = key; vn = ck.dv[u]; }
                else n2 = min(n2, key);
            }
        }
        const unsigned long long la1 = a1, ln1 = n1;
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
        // keys carry the column id, so exactly one lane holds each winner
        if (a1 != kKeyNone && la1 == a1) out->va = va;
        if (n1 != kKeyNone && ln1 == n1) out->vn = vn;
        if (lane == 0) {
            out->a1 = a1; out->a2 = a2; out->n1 = n1; out->n2 = n2;
            out->km = km;
        }
    };
    // Rescan the listed rows inv[0..ni) (entry = row << 2 | stage mask), excluding
    // columns exA, exB. Warps < nmerge first run `merge` (the merge warps), then join.
    // Ends with every listed row's caches final (block-synchronous).
    auto rescan_rows = [&](int ni, int exA, int exB, auto&& merge, int nmerge) {
        const bool dense = 2 * S >= R0;
        const int nch = dense ? (Wr + 3) >> 2 : (S + 127) >> 7;
        const int rpb = nch > 0 ? max(1, RHSEG_APO_PARTS / nch) : 1;
        int r0 = 0;
        do {
            const int nrow = min(rpb, ni - r0);
            const int total = max(0, nrow) * max(nch, 0);
            if (r0 == 0 && warp < nmerge) merge();
            for (;;) {
                int t = 0;
                if (lane == 0) t = atomicAdd(&misc[kMiscIctr], 2);
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t >= total) break;
                const int k0 = t / nch, c0 = t - k0 * nch;
                const int e0 = inv[r0 + k0];
                Chunk x0, x1;
                chunk_load(x0, e0 >> 2, e0 & 3, c0, dense, exA, exB);
                const bool two = t + 1 < total;
                int e1 = 0, c1 = 0, k1 = 0;
                if (two) {
                    k1 = (t + 1) / nch;
                    c1 = t + 1 - k1 * nch;
                    e1 = inv[r0 + k1];
                    chunk_load(x1, e1 >> 2, e1 & 3, c1, dense, exA, exB);
                }
                chunk_fold(x0, dense, &part[t]);  // (t is batch-relative: the counter restarts per batch)
                if (two) chunk_fold(x1, dense, &part[t + 1]);
            }
            __syncthreads();  // partials (and the merge) complete
            // finalize: one warp per row combines its nch partials
            for (int k = warp; k < nrow; k += kWarps) {
                const int e = inv[r0 + k], i = e >> 2, mask = e & 3;
                RsPart p;
                if (lane < nch) p = part[k * nch + lane];
                else { p.a1 = p.a2 = p.n1 = p.n2 = kKeyNone; p.va = p.vn = 0.0; p.km = 0; }
                // (all 32 lanes end with the row's result: the slow path below is warp-wide)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const unsigned long long oa1 = __shfl_xor_sync(0xffffffffu, p.a1, o), oa2 = __shfl_xor_sync(0xffffffffu, p.a2, o);
                    const unsigned long long on1 = __shfl_xor_sync(0xffffffffu, p.n1, o), on2 = __shfl_xor_sync(0xffffffffu, p.n2, o);
                    const double ova = __shfl_xor_sync(0xffffffffu, p.va, o), ovn = __shfl_xor_sync(0xffffffffu, p.vn, o);
                    p.km = max(p.km, __shfl_xor_sync(0xffffffffu, p.km, o));
                    if (oa1 < p.a1) p.va = ova;
                    if (on1 < p.n1) p.vn = ovn;
                    p.a2 = min(min(p.a2, oa2), max(p.a1, oa1));
                    p.a1 = min(p.a1, oa1);
                    p.n2 = min(min(p.n2, on2), max(p.n1, on1));
                    p.n1 = min(p.n1, on1);
                }
                // unique iff the smallest key's upper bound lies below the lower bound of
                // every other entry (their centres >= the second key, truncated by 2^-37
                // relative, each interval within 2^(km-46) of its centre)
                auto unique = [&](unsigned long long k1, unsigned long long k2, double v1) {
                    if (k2 == kKeyNone) return true;
                    double l1, h1;
                    d_unpack(v1, l1, h1);
                    const double c2 = __longlong_as_double((long long)(k2 & kKeyHi));
                    const double rho = __longlong_as_double((long long)(p.km - 46 + 1023) << 52) + 0x1p-37;
                    return h1 < __dmul_rd(c2, __dsub_rd(1.0, rho));
                };
                int slow = 0;
                if ((mask & 1) && p.a1 != kKeyNone && !unique(p.a1, p.a2, p.va)) slow |= 1;
                if ((mask & 2) && p.n1 != kKeyNone && !unique(p.n1, p.n2, p.vn)) slow |= 2;
                if (lane == 0) {
                    if ((mask & 1) && !(slow & 1)) { bAd[i] = p.a1 == kKeyNone ? kInf : p.va; bAj[i] = p.a1 == kKeyNone ? -1 : (int)(p.a1 & 0x3fff); }
                    if ((mask & 2) && !(slow & 2)) { bNd[i] = p.n1 == kKeyNone ? kInf : p.vn; bNj[i] = p.n1 == kKeyNone ? -1 : (int)(p.n1 & 0x3fff); }
                }
                if (slow) rescan_exact(i, slow, exA, exB);
            }
            r0 += rpb;
            if (r0 < ni && tid == 0) misc[kMiscIctr] = 0;
            __syncthreads();  // caches final; partials free; claim counter reset
        } while (r0 < ni);
    };

    // ---- prologue: counts, column list, norm bound, versioned means, live set ----
    for (int i = tid; i < Rp; i += kThreads) {
        const uint32_t c = i < R0 ? bt.count[(size_t)sec * Rp + i] : 0u;
        cnt[i] = c;
        col[i] = (short)i;
        slot_of[i] = (short)i;
        ver[i] = (unsigned short)i;
        bAd[i] = kInf; bNd[i] = kInf; bAj[i] = -1; bNj[i] = -1;
    }
    if (tid < 32) misc[tid] = 0;
    __syncthreads();
    {
        // ||m|| bound for the whole loop: every later mean is a weighted average of the
        // initial ones (times (1 + u)^depth), so per band max_i |m_i[k]| bounds |m[k]|
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
        for (size_t e = tid; e < (size_t)R0 * B; e += kThreads) {
            const int i = (int)(e / B);
            if (cnt[i] != 0u) mr[e] = __ddiv_rn(sums[e], (double)cnt[i]);  // == the cached mean, bit for bit
        }
        for (int w = tid; w < W; w += kThreads) {
            uint32_t m = 0u;
            for (int t = 0; t < 32; ++t) m |= (cnt[(w << 5) + t] != 0u ? 1u : 0u) << t;
            livew[w] = m;
        }
        unsigned long long e = 0;
        for (size_t w = tid; w < (size_t)R0 * W; w += kThreads) e += __popc(adj[w]);
        atomicAdd(sE0, e);
    }
    __syncthreads();
    const double apoE = (double)(B + 8) * kU64 * 1.01;
    const double apoEe = sqrt(*sx * (1.0 + 1e-9)) * (10.0 * kU64 * 1.01);  // see apo_interval
    long long E = (long long)(*sE0 / 2);
    // initial per-row bests: every live row, both stages, through the chunk machinery
    {
        for (int i = tid; i < R0; i += kThreads)
            if (cnt[i] != 0u) inv[atomicAdd(&misc[kMiscNinv], 1)] = (i << 2) | 3;
        __syncthreads();
        const int ni = misc[kMiscNinv];
        rescan_rows(ni, -1, -1, [] {}, 0);
    }
    if (tid == 0) { misc[kMiscNinv] = 0; misc[kMiscIctr] = 0; }
    __syncthreads();

    int step = 0, conv = 0;
    long long pairs = 0, nresc = 0;
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
        if (tid == 0) {
            const long long R = R0 - step;
            pairs += R * (R - 1) / 2 - E;
        }
        // ---- (A) argmin over the row caches (engine.py:281-296), unique-or-exact ----
        Pair A = pair_none(), N = pair_none();
        {
            ArgSt xa = as_none(), xn = as_none();
            for (int i = tid; i < R0; i += kThreads) {
                if (cnt[i] == 0u) continue;
                const int ja = bAj[i], jn = bNj[i];
                if (ja >= 0) {
                    const double v = bAd[i];
                    double l2, h2;
                    d_unpack(v, l2, h2);
                    as_put(xa, l2, h2, ((unsigned)min(i, ja) << 16) | (unsigned)max(i, ja), v);
                }
                if (jn >= 0) {
                    const double v = bNd[i];
                    double l2, h2;
                    d_unpack(v, l2, h2);
                    as_put(xn, l2, h2, ((unsigned)min(i, jn) << 16) | (unsigned)max(i, jn), v);
                }
            }
            as_block2(xa, xn, red + par * kWarps * 2);
            const bool multA = xa.k1 != kPairNone && !as_unique(xa), multN = xn.k1 != kPairNone && !as_unique(xn);
            if (xa.k1 != kPairNone && !multA) A = Pair{xa.v1, (int)(xa.k1 >> 16), (int)(xa.k1 & 0xffffu)};
            if (xn.k1 != kPairNone && !multN) N = Pair{xn.v1, (int)(xn.k1 >> 16), (int)(xn.k1 & 0xffffu)};
            if (multA || multN) {
                // distinct pairs within each other's intervals: make the candidates exact
                // and take the lexicographic minimum (rare)
                unsigned short* clist = reinterpret_cast<unsigned short*>(inv);
                for (int i = tid; i < R0; i += kThreads) {
                    if (cnt[i] == 0u) continue;
#pragma unroll
                    for (int st = 0; st < 2; ++st) {
                        if (!(st ? multN : multA)) continue;
                        const int j = st ? bNj[i] : bAj[i];
                        if (j < 0) continue;
                        double l2, h2;
                        d_unpack(st ? bNd[i] : bAd[i], l2, h2);
                        if (l2 <= (st ? xn.u : xa.u)) clist[atomicAdd(&misc[kMiscNc], 1)] = (unsigned short)(i | (st << 14));
                    }
                }
                __syncthreads();
                const int nc = misc[kMiscNc];
                for (int t = warp; t < nc; t += kWarps) {
                    const int e = clist[t], i = e & 0x3fff, st = e >> 14;
                    const int j = st ? bNj[i] : bAj[i];
                    if (!d_is_interval(st ? bNd[i] : bAd[i])) continue;
                    const double d = exact_pair(i, j);
                    __syncwarp();
                    if (lane == 0) {
                        if (st) bNd[i] = d;
                        else bAd[i] = d;
                    }
                }
                __syncthreads();
                Pair ca = pair_none(), cn = pair_none();
                for (int t = tid; t < nc; t += kThreads) {
                    const int e = clist[t], i = e & 0x3fff;
                    if (e >> 14) pair_offer(cn, make_pair(bNd[i], i, bNj[i]));
                    else pair_offer(ca, make_pair(bAd[i], i, bAj[i]));
                }
                block_min_pair2(ca, cn, pscr);
                if (multA) A = ca;
                if (multN) N = cn;
                if (prof && tid == 0) atomicAdd(bt.prof + 9, (unsigned long long)nc);
                if (tid == 0) misc[kMiscNc] = 0;  // (read by every thread before the last barrier)
            }
        }
        mark(0);
        // ---- merge rule (engine.py:322-339): spectral iff d_s < w * d_a, strictly ----
        int a = -1, b = -1, kind = 0;
        double dch = 0.0;
        const bool hasA = A.hi != kNoJ;
        if (N.hi != kNoJ) {
            double nl, nh, al = kInf, ah = kInf;
            d_unpack(N.d, nl, nh);
            if (hasA) d_unpack(A.d, al, ah);
            int dec = nh < __dmul_rn(bt.weight, al) ? 1 : (nl >= __dmul_rn(bt.weight, ah) ? 0 : -1);
            if (dec < 0) {
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
        }
        if (a < 0 && hasA) { a = A.lo; b = A.hi; dch = A.d; kind = 0; }
        if (a < 0) { conv = 1; break; }
        const double na0 = (double)cnt[a], nb0 = (double)cnt[b];
        const double nn = __dadd_rn(na0, nb0);
        mark(1);

        // ---- (C) rows whose cached partner is a or b; D rows a, b -> shared memory ----
        {
            const int nchk = (R0 + 1) >> 1;  // 16-byte chunks per row
            for (int q = tid; q < 2 * nchk; q += kThreads) {
                const int r = q >= nchk, c = q - r * nchk;
                cp_async16((r ? rowB : rowA) + 2 * c, D + (size_t)(r ? b : a) * Rp + 2 * c);
            }
            cp_async_commit();
        }
        for (int i = tid; i < R0; i += kThreads) {
            if (cnt[i] == 0u || i == a || i == b) continue;
            int mask = 0;
            if (bAj[i] == a || bAj[i] == b) mask |= 1;
            if (bNj[i] == a || bNj[i] == b) mask |= 2;
            if (mask) inv[atomicAdd(&misc[kMiscNinv], 1)] = (i << 2) | mask;
        }
        __syncthreads();
        const int ni = misc[kMiscNinv];
        nresc += ni;
        if (prof && tid == 0) pc[5] += (unsigned long long)ni;

        // ---- (X) merge (graph.py:229-264) on the merge warps || rescans ----
        auto merge = [&]() {
            const double* sb = sums + (size_t)b * B;
            double* sa = sums + (size_t)a * B;
            for (int k = tid; k < B; k += kApoMergeThreads) {
                const double s = __dadd_rn(sa[k], sb[k]);
                sa[k] = s;
                mua[k] = __ddiv_rn(s, nn);
            }
            // adjacency union (A|B)\{a,b}; b's neighbours are re-pointed b -> a
            uint32_t* ra = adj + (size_t)a * W;
            uint32_t* rbw = adj + (size_t)b * W;
            const int wa = a >> 5, wb = b >> 5;
            const uint32_t ma = 1u << (a & 31), mb = 1u << (b & 31);
            auto repoint = [&](int n) {
                uint32_t* rn = adj + (size_t)n * W;
                if (wa == wb) rn[wa] = (rn[wa] | ma) & ~mb;
                else { rn[wa] |= ma; rn[wb] &= ~mb; }
            };
            int dE = 0;
            for (int w = tid; w < W; w += kApoMergeThreads) {
                const uint32_t oa = ra[w], ob = rbw[w];
                uint32_t nw = oa | ob;
                if (w == wa) nw &= ~ma;
                if (w == wb) nw &= ~mb;
                dE += __popc(nw) - __popc(oa) - __popc(ob);
                if (w == wb && (oa & mb)) dE += 1;
                ra[w] = nw;
                sra[w] = nw;
                rbw[w] = 0u;
                uint32_t bits = w == wa ? ob & ~ma : ob;
                while (bits) {
                    const int n = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int k = atomicAdd(&misc[kMiscNnb], 1);
                    if (k < kApoNbList) nbl[k] = (unsigned short)n;
                    else repoint(n);  // overflow (very high degree): in place
                }
            }
            if (dE) atomicAdd(&misc[kMiscDE], dE);
            bar_merge();
            const int nb = min(misc[kMiscNnb], kApoNbList);
            for (int k = tid; k < nb; k += kApoMergeThreads) repoint(nbl[k]);
        };
        rescan_rows(ni, a, b, merge, RHSEG_APO_MERGE_WARPS);
        E += misc[kMiscDE];
        mark(2);

        // ---- (R) row a': intervals from D rows a, b (parallelogram identity), written
        // to D and offered to every row's cache; a's own best (unique-or-exact) ----
        const ApoStep ap = apo_step<M>(na0, nb0, dch, apoE, apoEe);
        cp_async_wait_all();
        __syncthreads();  // every thread's cp.async chunks have landed
        unsigned short* l1 = reinterpret_cast<unsigned short*>(inv);  // exact offers
        unsigned short* l2 = l1 + Rp;                                 // a's candidates
        ArgSt pa = as_none(), pn = as_none();
        for (int sl = tid; sl < S; sl += kThreads) {
            const int j = col[sl];
            if (j < 0 || j == a || j == b || cnt[j] == 0u) continue;
            double dlo, dhi, v;
            apo_interval<M>(ap, rowA[j], rowB[j], (double)cnt[j], dlo, dhi);
            const bool aj = (sra[j >> 5] >> (j & 31)) & 1u;
            const unsigned short e = (unsigned short)(j | (aj ? 0 : 0x4000));
            if (!d_pack_interval(dlo, dhi, v)) {  // too wide to store: exact below
                l1[atomicAdd(&misc[kMiscN1], 1)] = (unsigned short)(e | 0x8000);
                as_put(aj ? pa : pn, dlo, dhi, (unsigned)j, RHSEG_UNPACKED);  // (never taken as is)
                continue;
            }
            D[(size_t)j * Rp + a] = v;
            D[(size_t)a * Rp + j] = v;
            as_put(aj ? pa : pn, dlo, dhi, (unsigned)j, v);
            double& bv = aj ? bAd[j] : bNd[j];
            int& bj = aj ? bAj[j] : bNj[j];
            if (bj < 0) {
                bv = v;
                bj = a;
            } else {
                double bl, bh;
                d_unpack(bv, bl, bh);
                if (dhi < bl) { bv = v; bj = a; }
                else if (!(dlo > bh)) l1[atomicAdd(&misc[kMiscN1], 1)] = e;
            }
        }
        as_block2(pa, pn, red + par * kWarps * 2 + 0);  // (the argmin's buffer: its readers passed two barriers)
        const int n1 = misc[kMiscN1];
        if (prof && tid == 0 && n1) atomicAdd(bt.prof + 8, (unsigned long long)n1);
        // overlaps with row j's cached best: exact d(a', j) and exact best
        for (int t = warp; t < n1; t += kWarps) {
            const int e = l1[t], j = e & 0x3fff;
            const bool aj = !(e & 0x4000);
            const double daj = warp_exact<M>(mua, mr + (size_t)ver[j] * B, nn, (double)cnt[j], B, lane);
            const int bj = aj ? bAj[j] : bNj[j];
            double db = aj ? bAd[j] : bNd[j];
            if (bj >= 0 && d_is_interval(db)) db = exact_pair(j, bj);
            __syncwarp();  // every lane has read row j's cache before lane 0 rewrites it
            if (lane == 0) {
                D[(size_t)j * Rp + a] = daj;
                D[(size_t)a * Rp + j] = daj;
                const bool take_a = bj < 0 || daj < db || (daj == db && a < bj);
                if (aj) { bAd[j] = take_a ? daj : db; bAj[j] = take_a ? a : bj; }
                else { bNd[j] = take_a ? daj : db; bNj[j] = take_a ? a : bj; }
            }
        }
        const bool uA = as_unique(pa) && !isnan(pa.v1), uN = as_unique(pn) && !isnan(pn.v1);
        const bool mA = pa.k1 != kPairNone && !uA, mN = pn.k1 != kPairNone && !uN;
        if (n1 || mA || mN) __syncthreads();  // (uniform) exact offers published
        RowBest pA = rb_none(), pN = rb_none();
        if (pa.k1 != kPairNone && uA) pA = RowBest{pa.v1, (int)pa.k1};
        if (pn.k1 != kPairNone && uN) pN = RowBest{pn.v1, (int)pn.k1};
        if (mA || mN) {
            // several columns within each other's intervals: the exact minimum of them
            for (int sl = tid; sl < S; sl += kThreads) {
                const int j = col[sl];
                if (j < 0 || j == a || j == b || cnt[j] == 0u) continue;
                const bool aj = (sra[j >> 5] >> (j & 31)) & 1u;
                if (!(aj ? mA : mN)) continue;
                double dlo, dhi;
                apo_interval<M>(ap, rowA[j], rowB[j], (double)cnt[j], dlo, dhi);
                if (dlo <= (aj ? pa.u : pn.u)) l2[atomicAdd(&misc[kMiscN2], 1)] = (unsigned short)(j | (aj ? 0 : 0x4000));
            }
            __syncthreads();
            const int n2 = misc[kMiscN2];
            if (prof && tid == 0) atomicAdd(bt.prof + 9, (unsigned long long)n2);
            RowBest cA = rb_none(), cN = rb_none();
            for (int t = warp; t < n2; t += kWarps) {
                const int e = l2[t], j = e & 0x3fff;
                const bool aj = !(e & 0x4000);
                double v = __ldcg(D + (size_t)a * Rp + j);
                if (d_is_interval(v)) {
                    v = warp_exact<M>(mua, mr + (size_t)ver[j] * B, nn, (double)cnt[j], B, lane);
                    if (lane == 0) {
                        D[(size_t)j * Rp + a] = v;
                        D[(size_t)a * Rp + j] = v;
                    }
                }
                if (lane == 0) {
                    if (aj) rb_offer(cA, v, j);
                    else rb_offer(cN, v, j);
                }
            }
            block_min_rb2(cA, cN, rscr);
            if (mA) pA = cA;
            if (mN) pN = cN;
        }
        mark(3);

        // ---- (E) publish the merge (one thread) + a's new mean version ----
        for (int k = tid; k < B; k += kThreads) mr[(size_t)(R0 + step) * B + k] = mua[k];
        if (tid == 0) {
            cnt[a] = (uint32_t)nn;
            cnt[b] = 0u;
            livew[b >> 5] &= ~(1u << (b & 31));
            if (d_is_interval(dch))  // exact value after the loop (mean versions of a and b)
                bt.apo_rec[(size_t)sec * Rp + step] = make_uint4(ver[a], ver[b], (unsigned)na0, (unsigned)nb0);
            ver[a] = (unsigned short)(R0 + step);
            bAd[a] = pA.d;
            bAj[a] = pA.j == kNoJ ? -1 : pA.j;
            bNd[a] = pN.d;
            bNj[a] = pN.j == kNoJ ? -1 : pN.j;
            bAd[b] = kInf; bAj[b] = -1;
            bNd[b] = kInf; bNj[b] = -1;
            const size_t o = (size_t)sec * Rp + step;
            bt.log_a[o] = a;
            bt.log_b[o] = b;
            bt.log_d[o] = dch;
            bt.log_k[o] = (uint8_t)kind;
            bt.parent[(size_t)sec * Rp + b] = a;
            col[slot_of[b]] = -1;
            slot_of[b] = -1;
            misc[kMiscNinv] = 0;
            misc[kMiscIctr] = 0;
            misc[kMiscNnb] = 0;
            misc[kMiscDE] = 0;
            misc[kMiscN1] = 0;
            misc[kMiscN2] = 0;
        }
        holes += 1;
        __syncthreads();
        if (S >= 64 && holes * RHSEG_APO_COMPACT >= S) {
            // stable compaction of the live-column list (ids stay ascending)
            int base = 0;
            for (int c0 = 0; c0 < S; c0 += kThreads) {
                const int s = c0 + tid;
                const int id = s < S ? col[s] : -1;
                const int v = id >= 0 ? 1 : 0;
                int x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                int* scr = misc + 16;
                if (lane == 31) scr[warp] = x;
                __syncthreads();
                int wbase = 0, tot = 0;
                for (int w = 0; w < kWarps; ++w) {
                    if (w < warp) wbase += scr[w];
                    tot += scr[w];
                }
                __syncthreads();  // every read of col[] / scr in this chunk precedes the writes
                const int np = base + wbase + x - v;
                if (id >= 0) {
                    col[np] = (short)id;
                    slot_of[id] = (short)np;
                }
                base += tot;
            }
            S = base;
            holes = 0;
            __syncthreads();
        }
        mark(4);
        ++step;
    }
    // the log's dissimilarities still held as intervals: exact values now, one thread
    // per step (the reference's ascending-band sum from the two mean versions)
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
    if (prof && tid == 0) {
        pc[7] = (unsigned long long)(clock64() - t_entry);
        for (int q = 0; q < 8; ++q) atomicAdd(bt.prof + q, pc[q]);
    }
    for (int i = tid; i < Rp; i += kThreads) bt.count[(size_t)sec * Rp + i] = cnt[i];
    if (tid == 0) {
        bt.nlog[sec] = step;
        bt.conv[sec] = conv;
        if (bt.pairs) bt.pairs[sec] = pairs;
        if (bt.nresc) bt.nresc[sec] = nresc;
    }
}

int launch_apo_loop(const SectionBatch& b, int nrun, cudaStream_t st) {
    if (nrun == 0) return 0;
    const size_t smem = apo_loop_smem(b.Rp, b.B);
    void (*kern)(SectionBatch) = b.measure == kEuclid ? hseg_apo_kernel<kEuclid> : hseg_apo_kernel<kBsmse>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<nrun, kThreads, smem, st>>>(b);
    return cudaGetLastError();
}

}  // namespace rhseg
