// rhseg_batch.h -- the HBM layout of one batch of independent HSEG sections
// (one quadtree level, or one standalone region graph). Shared by the host
// orchestration (rhseg_api.cu) and the kernels.
//
// Per section s (all arrays padded to Rp = roundup(R0max, 32) region slots):
//   count [Rp]          u32   pixel counts (0 = dead)      -- graph.py:86-92 pixel_count
//   mu    [B][Rp]       f64   band-major mean cache        -- sums/count (Appendix A.3)
//   mu2   [B][Rp]       f64   stream loop: ping-pong copy (each CTA's live columns compacted,
//                             ascending ids, in mu / mu2 and streamed); APO loop: [2 Rp][B]
//                             versioned region-major means (row R0 + t = mean made by step t)
//   D     [Rp][Rp]      f64   dissimilarity matrix (exact values; APO sections may hold
//                             encoded intervals around them) for every live pair
//                             (w > 0) or every adjacent pair (w = 0)
//   sums  [C][Rp][B]    f64   band sums, one private copy per cluster CTA
//   adj   [C][Rp][W]    u32   symmetric adjacency bitset, one private copy per CTA
//   parent[Rp]          i32   absorbed -> survivor (union-find for labels), -1 = root
//   assign[npx]         i32   pixel -> section-local region id
//   log_{a,b,d,k}[Rp]         merge records (survivor, absorbed, dissim, kind)
#pragma once

#include <stddef.h>
#include <stdint.h>

#include <vector_types.h>

namespace rhseg {

struct SectionBatch {
    int nsec;      // sections in the batch
    int B;         // bands
    int Rp;        // padded region capacity (multiple of 32)
    int W;         // Rp / 32 bitset words per row
    int C;         // CTAs per section (thread-block cluster size)
    int edge;      // section edge in pixels (0 for a standalone graph)
    int npx;       // edge * edge
    int spec;      // spectral stage on (weight > 0)
    int measure;   // 0 sqrt-bsmse (reference), 1 euclidean, 2 sam (extensions)
    int stage_bytes;  // merge-loop stream ring stage size (host-chosen)
    int nstages;      // merge-loop stream ring depth (host-chosen)
    int apo;          // merge loop bounds d(a', j) from D rows a, b (no mean stream; see hseg_kernels.cu)
    void* l2_window_base;    // L2-persisting access window of the loop launch (0 bytes = none)
    size_t l2_window_bytes;
    double weight; // spectral_weight (engine.py:33)
    const int* R0;       // [nsec] initial live regions
    const int* target;   // [nsec] stopping count (recursive.py:49-52)
    double* mu;
    double* nrm2;        // [nsec][Rp] squared norm of each mean vector (sam only, else nullptr)
    uint4* apo_rec;      // APO: [nsec][Rp] (mean versions of a, b; counts) of steps logged as intervals
    double* mu2;         // second mean buffer: the loop kernel compacts live columns into it (w > 0)
    double* D;
    double* sums;
    uint32_t* adj;
    uint32_t* count;
    int* parent;
    int* assign;
    int* log_a;
    int* log_b;
    double* log_d;
    uint8_t* log_k;
    int* nlog;
    int* conv;
    long long* pairs;    // [nsec] reference-equivalent spectral pairs, sum_steps R(R-1)/2 - E
    long long* nresc;    // [nsec] rows rescanned from D by the merge loop (traffic accounting)
    int sec0;            // first section covered by D (D is allocated per launch chunk)
    unsigned long long* prof;  // [5] per-phase cycles summed over CTAs (nullptr = off)
    int G;               // grid loop (grid_loop.cu): CTAs per section (0 = cluster/CTA loops)
    void* gscr;          // grid loop: per-section scratch (group barrier, slots, pending, live bits)

    __host__ __device__ size_t mu_stride() const { return (size_t)B * Rp; }
    __host__ __device__ size_t d_stride() const { return (size_t)Rp * Rp; }
    __host__ __device__ size_t sums_copy() const { return (size_t)Rp * B; }
    __host__ __device__ size_t adj_copy() const { return (size_t)Rp * W; }
};

// Per-section scratch of the grid loop (grid_loop.cu), G CTAs per section; every CTA's
// slot is written to kGridSlotRep replicas (128 bytes each, flag-carrying words).
constexpr int kGridSlotRep = 16;
struct GridScrLayout {
    size_t bar, slots, pend, pend_each, live, acc, bytes;
};
__host__ __device__ inline GridScrLayout grid_scr_layout(int G, int B, int W) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    GridScrLayout L;
    size_t o = 0;
    L.bar = o;
    o += 256;
    L.slots = o;
    o += al((size_t)2 * kGridSlotRep * G * 128);
    L.pend_each = al(16 + (size_t)8 * B);
    L.pend = o;
    o += 2 * L.pend_each;
    L.live = o;
    o += al((size_t)4 * W);
    L.acc = o;
    o += 256;
    L.bytes = o;
    return L;
}

// Kernel launchers (hseg_kernels.cu / section_kernels.cu). All stream-ordered.
void launch_dinit(const SectionBatch& b, int nrun, int R0max, cudaStream_t st);
int launch_hseg_loop(const SectionBatch& b, int nrun, cudaStream_t st);  // returns cudaError_t
int launch_apo_loop(const SectionBatch& b, int nrun, cudaStream_t st);   // apo_loop.cu (b.apo sections)
size_t apo_loop_smem(int Rp, int B);
int launch_adj_loop(const SectionBatch& b, int nrun, int nsm, cudaStream_t st);   // adj_loop.cu (w = 0, C = 1)
size_t adj_loop_smem(int Rp, int B, int nwarps);
int launch_grid_loop(const SectionBatch& b, int nrun, int nsm, cudaStream_t st, int* G_used);  // grid_loop.cu
size_t grid_loop_scratch_bytes(int nsm, int B, int W);                            // per section
size_t hseg_loop_smem(int Rp, int C, int B, bool spec, int measure, int stage_bytes, int nstages);
int hseg_loop_max_stages();
int hseg_loop_default_stages();
int hseg_loop_stage_bytes(bool spec, int C, int measure);  // default ring stage size
int hseg_loop_max_rows();  // own rows per CTA the loop kernel supports
bool hseg_apo_capable(bool spec, int C, int measure);  // the loop can run without the mean stream
// sections [b.sec0, b.sec0 + count) of the leaf level (count < 0: through the end)
void launch_leaf_init(const SectionBatch& b, const float* cube, int img_edge, int cols, int row0,
                      int col0, int connectivity, cudaStream_t st, int count = -1);
void launch_resolve(const SectionBatch& b, cudaStream_t st);
// Parent grid rows x pcols, child grid (2 rows) x (2 pcols), both row-major.
void launch_stitch(const SectionBatch& child, int child_cols, const SectionBatch& parent,
                   int parent_cols, int* child_map, int connectivity, cudaStream_t st);
void launch_dense_labels(const int* assign, int npx, int R, int* first, int* rank, int* labels,
                         cudaStream_t st);
void launch_graph_init(const SectionBatch& b, const double* counts, const double* sums_rm,
                       const int64_t* indptr, const int64_t* indices, cudaStream_t st);

}  // namespace rhseg
