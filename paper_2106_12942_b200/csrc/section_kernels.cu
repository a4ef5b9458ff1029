// section_kernels.cu -- building and reassembling quadtree sections on device.
//
// Reference semantics replaced:
//   graph.py:161-183   init_region_graph (one region per pixel, row-major ids, 4/8 grid adjacency)
//   sections.py:57-79  partition (4^(L-1) leaves, row-major)
//   sections.py:82-163 _seam_pairs + stitch (dense renumber NW,NE,SW,SE; seam links)
//   graph.py:229-264   merge_regions pixel relabel -> deferred to a union-find resolve
//   graph.py:267-281   dense_renumber / label_map_from_graph (first row-major occurrence)
#include <cuda_runtime.h>

#include <algorithm>

#include "rhseg_batch.h"
#include "rhseg_device.cuh"

namespace rhseg {

// ---------------------------------------------------------------------------
// Leaf init: section `sec` of a rows x cols block of the leaf grid (origin
// row0, col0 in sections; the whole side x side partition for a full run)
// reads its e x e window of the BSQ float32 cube (image.py:59-62 subimage)
// straight from HBM.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
leaf_init_kernel(SectionBatch bt, const float* __restrict__ cube, int N, int cols, int row0, int col0, int conn) {
    const int sec = bt.sec0 + blockIdx.x;  // sections [sec0, sec0 + gridDim.x) of the level
    const int e = bt.edge, R0 = e * e, B = bt.B, Rp = bt.Rp, W = bt.W;
    const int orow = (row0 + sec / cols) * e, ocol = (col0 + sec % cols) * e;
    uint32_t* cnt = bt.count + (size_t)sec * Rp;
    int* parent = bt.parent + (size_t)sec * Rp;
    int* assign = bt.assign + (size_t)sec * bt.npx;
    double* mu = bt.mu + sec * bt.mu_stride();
    for (int p = threadIdx.x; p < Rp; p += kThreads) {
        cnt[p] = p < R0 ? 1u : 0u;
        parent[p] = -1;
        if (p < R0) assign[p] = p;
    }
    // one read of the window: 32 pixels x 32 bands tiles, coalesced along the pixels;
    // mu[k][p] (band-major) is written straight from the loads, sums[c][p][k]
    // (region-major) through a shared-memory transpose
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x kWarps
    for (int p0 = 0; p0 < R0; p0 += 32)
        for (int k0 = 0; k0 < B; k0 += 32) {
            for (int kk = ty; kk < 32; kk += kWarps) {
                const int p = p0 + tx, k = k0 + kk;
                double v = 0.0;
                if (p < R0 && k < B) {
                    const int r = p / e, c = p - r * e;
                    v = (double)cube[((size_t)k * N + orow + r) * N + ocol + c];
                    mu[(size_t)k * Rp + p] = v;
                }
                tile[kk][tx] = v;
            }
            __syncthreads();
            for (int pp = ty; pp < 32; pp += kWarps) {
                const int p = p0 + pp, k = k0 + tx;
                if (p < R0 && k < B)
                    for (int cc = 0; cc < bt.C; ++cc)
                        bt.sums[((size_t)sec * bt.C + cc) * bt.sums_copy() + (size_t)p * B + k] = tile[tx][pp];
            }
            __syncthreads();
        }
    if (bt.measure == kSam) {  // squared norms of the one-pixel means (sam only)
        __syncthreads();
        for (int p = threadIdx.x; p < R0; p += kThreads) bt.nrm2[(size_t)sec * Rp + p] = norm2_seq(mu + p, Rp, B);
    }
    // grid adjacency (graph.py:20-29 offsets), one writer per row; batch was zeroed
    for (int p = threadIdx.x; p < R0; p += kThreads) {
        const int r = p / e, c = p - r * e;
        for (int dr = -1; dr <= 1; ++dr)
            for (int dc = -1; dc <= 1; ++dc) {
                if (dr == 0 && dc == 0) continue;
                if (conn == 4 && dr != 0 && dc != 0) continue;
                const int rr = r + dr, c2 = c + dc;
                if (rr < 0 || rr >= e || c2 < 0 || c2 >= e) continue;
                const int q = rr * e + c2;
                for (int cc = 0; cc < bt.C; ++cc)
                    bt.adj[((size_t)sec * bt.C + cc) * bt.adj_copy() + (size_t)p * W + (q >> 5)] |= 1u << (q & 31);
            }
    }
}

void launch_leaf_init(const SectionBatch& b, const float* cube, int img_edge, int cols, int row0, int col0,
                      int connectivity, cudaStream_t st, int count) {
    const int n = count < 0 ? b.nsec - b.sec0 : count;
    if (n <= 0) return;
    leaf_init_kernel<<<n, kThreads, 0, st>>>(b, cube, img_edge, cols, row0, col0, connectivity);
}

// ---------------------------------------------------------------------------
// Resolve pixel -> live region through the absorbed->survivor links written by
// the merge loop (survivor id < absorbed id, so every chain terminates).
// ---------------------------------------------------------------------------
__global__ void resolve_kernel(SectionBatch bt) {
    const int sec = blockIdx.y;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= bt.npx) return;
    const int* parent = bt.parent + (size_t)sec * bt.Rp;
    int* assign = bt.assign + (size_t)sec * bt.npx;
    int x = assign[p];
    while (parent[x] >= 0) x = parent[x];
    assign[p] = x;
}

void launch_resolve(const SectionBatch& b, cudaStream_t st) {
    if (b.nsec == 0 || b.npx == 0) return;
    dim3 grid((b.npx + kThreads - 1) / kThreads, b.nsec);
    resolve_kernel<<<grid, kThreads, 0, st>>>(b);
}

// ---------------------------------------------------------------------------
// Stitch (sections.py:103-163): parent section P gathers children NW,NE,SW,SE.
// New ids: each child's live ids ascending, children in NW,NE,SW,SE order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int block_excl_scan(int v, int* scratch, int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    int wbase = 0, tot = 0;
    for (int w = 0; w < kWarps; ++w) {
        if (w < warp) wbase += scratch[w];
        tot += scratch[w];
    }
    __syncthreads();
    total = tot;
    return wbase + x - v;
}

__global__ void __launch_bounds__(kThreads)
stitch_kernel(SectionBatch ch, int ccols, SectionBatch pa, int pcols, int* cmap, int conn) {
    const int P = blockIdx.x;
    const int pr = P / pcols, pc = P % pcols;
    const int B = pa.B;
    __shared__ int scratch[kWarps];
    int cidx[4];
    for (int k = 0; k < 4; ++k) cidx[k] = (2 * pr + (k >> 1)) * ccols + (2 * pc + (k & 1));
    // 1. dense renumber maps; the parent's `parent` array doubles as the inverse
    //    list (parent id -> child k, child id) until step 5 resets it
    uint32_t* pcnt = pa.count + (size_t)P * pa.Rp;
    int* pparent = pa.parent + (size_t)P * pa.Rp;
    double* pmu = pa.mu + P * pa.mu_stride();
    int base = 0;
    for (int k = 0; k < 4; ++k) {
        const int c = cidx[k];
        const int R0c = ch.R0[c];
        const uint32_t* ccnt = ch.count + (size_t)c * ch.Rp;
        int* map = cmap + (size_t)c * ch.Rp;
        for (int i0 = 0; i0 < R0c; i0 += kThreads) {
            const int i = i0 + threadIdx.x;
            const int live = (i < R0c && ccnt[i] != 0u) ? 1 : 0;
            int tot;
            const int pre = block_excl_scan(live, scratch, tot);
            if (i < R0c) map[i] = live ? base + pre : -1;
            if (live) pparent[base + pre] = (k << 24) | i;
            base += tot;
        }
    }
    __syncthreads();
    // 2. counts, sums (all parent copies), mu, adjacency -- live regions only
    const int R = base;  // == pa.R0[P]
    for (int idx = threadIdx.x; idx < R * B; idx += kThreads) {
        const int m = idx / B, q = idx - m * B;
        const int src = pparent[m], k = src >> 24, i = src & 0xffffff, c = cidx[k];
        const double cn = (double)ch.count[(size_t)c * ch.Rp + i];
        if (q == 0) pcnt[m] = ch.count[(size_t)c * ch.Rp + i];
        const double s = ch.sums[(size_t)c * ch.C * ch.sums_copy() + (size_t)i * B + q];  // copy 0
        for (int cc = 0; cc < pa.C; ++cc)
            pa.sums[((size_t)P * pa.C + cc) * pa.sums_copy() + (size_t)m * B + q] = s;
        pmu[(size_t)q * pa.Rp + m] = __ddiv_rn(s, cn);
    }
    for (int idx = threadIdx.x; idx < R * ch.W; idx += kThreads) {
        const int m = idx / ch.W, w = idx - m * ch.W;
        const int src = pparent[m], k = src >> 24, i = src & 0xffffff, c = cidx[k];
        uint32_t bits = ch.adj[(size_t)c * ch.C * ch.adj_copy() + (size_t)i * ch.W + w];  // copy 0
        const int* map = cmap + (size_t)c * ch.Rp;
        while (bits) {
            const int j = (w << 5) + __ffs(bits) - 1;
            bits &= bits - 1;
            const int mj = map[j];
            for (int cc = 0; cc < pa.C; ++cc)
                atomicOr(&pa.adj[((size_t)P * pa.C + cc) * pa.adj_copy() + (size_t)m * pa.W + (mj >> 5)],
                         1u << (mj & 31));
        }
    }
    if (pa.measure == kSam) {
        __syncthreads();
        const int R = pa.R0[P];  // = live regions over the four children
        for (int m = threadIdx.x; m < R; m += kThreads)
            pa.nrm2[(size_t)P * pa.Rp + m] = norm2_seq(pmu + m, pa.Rp, B);
    }
    // 5. union-find links start empty (the inverse list lived here); the parent's pixel
    //    assignment and the seam links follow as two grid-wide kernels (a level near the
    //    root has one or four parents of up to 2048^2 pixels: one CTA per parent took
    //    8.7 ms at C4's root, profiles/r02_ncu_stitch)
    __syncthreads();
    for (int i = threadIdx.x; i < pa.Rp; i += kThreads) pparent[i] = -1;
}

// 3. parent pixel assignment over every pixel of every parent of the level (grid-wide)
__global__ void __launch_bounds__(kThreads)
stitch_assign_kernel(SectionBatch ch, int ccols, SectionBatch pa, int pcols, const int* cmap) {
    const int P = blockIdx.y;
    const int pr = P / pcols, pc = P % pcols;
    const int e = ch.edge, E = pa.edge;
    int* passign = pa.assign + (size_t)P * pa.npx;
    for (int p = blockIdx.x * kThreads + threadIdx.x; p < E * E; p += gridDim.x * kThreads) {
        const int r = p / E, c = p - r * E;
        const int k = (r >= e ? 2 : 0) + (c >= e ? 1 : 0);
        const int cidx = (2 * pr + (k >> 1)) * ccols + (2 * pc + (k & 1));
        const int lr = r - (k >> 1) * e, lc = c - (k & 1) * e;
        const int cid = ch.assign[(size_t)cidx * ch.npx + lr * e + lc];
        passign[p] = cmap[(size_t)cidx * ch.Rp + cid];
    }
}

// 4. seam links (sections.py:82-100): straight + both diagonals under 8-conn; one thread
//    per seam position r of each parent (grid-wide, atomicOr: order-free)
__global__ void __launch_bounds__(kThreads) stitch_seam_kernel(SectionBatch ch, SectionBatch pa, int conn) {
    const int P = blockIdx.y;
    const int e = ch.edge, E = pa.edge;
    const int* passign = pa.assign + (size_t)P * pa.npx;
    auto link = [&](int r1, int c1, int r2, int c2) {
        const int a = passign[r1 * E + c1], b = passign[r2 * E + c2];
        if (a == b) return;
        for (int cc = 0; cc < pa.C; ++cc) {
            uint32_t* A = pa.adj + ((size_t)P * pa.C + cc) * pa.adj_copy();
            atomicOr(&A[(size_t)a * pa.W + (b >> 5)], 1u << (b & 31));
            atomicOr(&A[(size_t)b * pa.W + (a >> 5)], 1u << (a & 31));
        }
    };
    const int r = blockIdx.x * kThreads + threadIdx.x;
    if (r >= E) return;
    link(r, e - 1, r, e);
    if (conn == 8 && r + 1 < E) {
        link(r, e - 1, r + 1, e);
        link(r, e, r + 1, e - 1);
    }
    link(e - 1, r, e, r);
    if (conn == 8 && r + 1 < E) {
        link(e - 1, r, e, r + 1);
        link(e - 1, r + 1, e, r);
    }
}

void launch_stitch(const SectionBatch& child, int child_cols, const SectionBatch& parent, int parent_cols,
                   int* child_map, int connectivity, cudaStream_t st) {
    if (parent.nsec == 0) return;
    stitch_kernel<<<parent.nsec, kThreads, 0, st>>>(child, child_cols, parent, parent_cols, child_map,
                                                     connectivity);
    const int npx = parent.edge * parent.edge;
    const int bx = std::max(1, std::min((npx + kThreads - 1) / kThreads, (4 * 148 + parent.nsec - 1) / parent.nsec * 4));
    stitch_assign_kernel<<<dim3(bx, parent.nsec), kThreads, 0, st>>>(child, child_cols, parent, parent_cols, child_map);
    stitch_seam_kernel<<<dim3((parent.edge + kThreads - 1) / kThreads, parent.nsec), kThreads, 0, st>>>(
        child, parent, connectivity);
}

// ---------------------------------------------------------------------------
// Standalone graph (hseg_run drop-in, engine.py:345): dense ascending-id regions
// with counts, region-major sums and CSR adjacency, as built by engine.snapshot
// (engine.py:167-191).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
graph_init_kernel(SectionBatch bt, const double* __restrict__ counts, const double* __restrict__ sums_rm,
                  const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices) {
    const int R0 = bt.R0[0], B = bt.B, Rp = bt.Rp, W = bt.W;
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= Rp) return;
    bt.parent[i] = -1;
    if (i >= R0) { bt.count[i] = 0u; return; }
    const double n = counts[i];
    bt.count[i] = (uint32_t)n;
    for (int k = 0; k < B; ++k) {
        const double s = sums_rm[(size_t)i * B + k];
        bt.mu[(size_t)k * Rp + i] = __ddiv_rn(s, n);
        for (int cc = 0; cc < bt.C; ++cc) bt.sums[cc * bt.sums_copy() + (size_t)i * B + k] = s;
    }
    if (bt.measure == kSam) bt.nrm2[i] = norm2_seq(bt.mu + i, Rp, B);
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
        const int j = (int)indices[p];
        for (int cc = 0; cc < bt.C; ++cc) bt.adj[cc * bt.adj_copy() + (size_t)i * W + (j >> 5)] |= 1u << (j & 31);
    }
}

void launch_graph_init(const SectionBatch& b, const double* counts, const double* sums_rm, const int64_t* indptr,
                       const int64_t* indices, cudaStream_t st) {
    graph_init_kernel<<<(b.Rp + kThreads - 1) / kThreads, kThreads, 0, st>>>(b, counts, sums_rm, indptr, indices);
}

// ---------------------------------------------------------------------------
// Dense labels by first row-major occurrence (graph.py:267-275).
// ---------------------------------------------------------------------------
constexpr int kFirstNone = 0x7f7f7f7f;  // memset(0x7f) sentinel

// first occurrence of every label: lanes holding the same label elect the lowest lane
// (the smallest pixel index of the group) for the one atomicMin -- a root with ~16
// regions over 4M pixels otherwise serialises on 16 addresses (2.7 ms at C4)
__global__ void first_occ_kernel(const int* assign, int npx, int* first) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = p < npx;
    const int lab = in ? assign[p] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, lab);
    if (in && (threadIdx.x & 31) == __ffs(grp) - 1) atomicMin(&first[lab], p);
}
__global__ void rank_kernel(const int* first, int R, int* rank) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const int f = first[r];
    if (f == kFirstNone) { rank[r] = -1; return; }
    int k = 0;
    for (int q = 0; q < R; ++q) k += first[q] < f;
    rank[r] = k;
}
__global__ void label_kernel(const int* assign, int npx, const int* rank, int* labels) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < npx) labels[p] = rank[assign[p]];
}

void launch_dense_labels(const int* assign, int npx, int R, int* first, int* rank, int* labels, cudaStream_t st) {
    cudaMemsetAsync(first, 0x7f, sizeof(int) * (size_t)R, st);  // 0x7f7f7f7f > any pixel index
    const int g = (npx + kThreads - 1) / kThreads;
    first_occ_kernel<<<g, kThreads, 0, st>>>(assign, npx, first);
    rank_kernel<<<(R + kThreads - 1) / kThreads, kThreads, 0, st>>>(first, R, rank);
    label_kernel<<<g, kThreads, 0, st>>>(assign, npx, rank, labels);
}

}  // namespace rhseg
