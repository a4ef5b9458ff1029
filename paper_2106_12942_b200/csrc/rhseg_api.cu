// rhseg_api.cu -- host orchestration behind the C ABI (include/rhseg_b200.h).
//
// Drives the quadtree exactly like SequentialExecutor.execute (recursive.py:173-209):
// leaves (level L, row-major) -> stitch + HSEG per level L-1..1 -> assemble. Every
// level is ONE batch: all of its sections run concurrently on the device (one
// thread-block cluster per section, persistent merge loop), so the host only
// launches ~5 kernels per level and synchronises once per level to size the
// parent level (its region counts depend on how far the children merged).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rhseg_b200.h"
#include "rhseg_batch.h"
#include "rhseg_device.cuh"

namespace rhseg {
void launch_scan_prep(int n, int nb, int ld, int W, const double* counts, const double* sums,
                      const int64_t* indptr, const int64_t* indices, double* mu, uint32_t* bits,
                      bool need_bits, cudaStream_t st);
void launch_scan_adjacent(int row_start, int row_stop, int ld, int nb, const double* counts, const double* mu,
                          const int64_t* indptr, const int64_t* indices, double* out_d, int64_t* out_j,
                          cudaStream_t st);
int scan_nonadj_splits(int n, int rows, int nsm);
void launch_scan_nonadjacent(int row_start, int row_stop, int n, int ld, int nb, int W, int nsplit,
                             const double* counts, const double* mu, const uint32_t* bits, void* part,
                             double* out_d, int64_t* out_j, cudaStream_t st);

// ---------------------------------------------------------------------------
// small device helpers owned by the host layer
// ---------------------------------------------------------------------------
__global__ void compact_log_kernel(const int* la, const int* lb, const double* ld, const uint8_t* lk,
                                   const int* nlog, const long long* off, int Rp, int* oa, int* ob,
                                   double* od, uint8_t* ok) {
    const int s = blockIdx.x;
    const int n = nlog[s];
    const long long o = off[s];
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const size_t src = (size_t)s * Rp + k;
        oa[o + k] = la[src];
        ob[o + k] = lb[src];
        od[o + k] = ld[src];
        ok[o + k] = lk[src];
    }
}

__global__ void fp64_probe_kernel(double* out, int iters) {
    double x[8], y[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        x[q] = 1.0 + 1e-3 * (threadIdx.x + q);
        y[q] = 0.0;
    }
    const double m = 1.0000001;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] = bsmse_step(y[q], x[q], m);  // sub, mul, add
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += y[q];
    if (s == 12345.0) out[threadIdx.x] = s;  // keep the loop alive
}

__global__ void fp64_fma_probe_kernel(double* out, int iters) {
    double x[8], y[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        x[q] = 1.0 + 1e-3 * (threadIdx.x + q);
        y[q] = 0.0;
    }
    const double m = 1.0000001;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] = __fma_rn(x[q], m, y[q]);  // one DFMA = 2 flops
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += y[q];
    if (s == 12345.0) out[threadIdx.x] = s;
}

}  // namespace rhseg

using namespace rhseg;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;
static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
// for the library's other translation units (outputs.cu)
namespace rhseg {
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace rhseg
#define CK(expr)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(RHSEG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));  \
    } while (0)

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
// Largest section the shared-memory loops hold (one CTA, or a cluster of up to 16 CTAs;
// 14-bit region ids in the loop kernel's lists and keys, hseg_kernels.cu). Larger sections
// run on the grid loop (grid_loop.cu), limited only by D's R^2 fp64 in HBM
// (rhseg_ctx::max_regions).
constexpr long long kMaxSectionRegions = 16384;

#ifndef RHSEG_L2_PERSIST_MB
#define RHSEG_L2_PERSIST_MB 0  // off: no gain on C2, C4 3% slower with a 64 MB set-aside
#endif

// ---------------------------------------------------------------------------
// one batch of sections (a quadtree level or a standalone graph)
// ---------------------------------------------------------------------------
struct Level {
    // the batch is a rows x cols block of this level's side x side section grid
    // starting at section (row0, col0); a full run covers the whole grid
    int level = 0, rows = 0, cols = 0, row0 = 0, col0 = 0, nsec = 0, edge = 0, Rp = 0, W = 0, C = 1, B = 0,
        R0max = 0;
    bool imported = false;  // state received from other ranks: not part of this ctx's logs
    bool grid = false;      // merge loop on a group of co-resident CTAs (grid_loop.cu)
    int gridG = 0;          // CTAs per section of the grid loop's last launch
    int measure = 0;        // 0 sqrt-bsmse, 1 euclidean, 2 sam
    std::vector<int> R0h, tgth, nlogh, convh;
    std::vector<long long> pairsh, rescsh;
    SectionBatch sb{};
    void* keep = nullptr;
    void* work = nullptr;
    int* map = nullptr;    // dense-renumber scratch used when this level is stitched
    size_t work_zero = 0;  // bytes at the start of `work` that must be zeroed (adjacency)
    bool done = false;
};

struct rhseg_ctx {
    int device = 0;
    int nsm = 148;
    long long max_regions = kMaxSectionRegions;  // largest section D fits (set from the HBM size)
    cudaStream_t stream = nullptr;
    std::vector<Level> levels;  // processing order == log order (L .. 1)
    bool have = false;
    int edge = 0, bands = 0, L = 0;
    int top = 1;  // highest level processed by the last run (1 = a complete RHSEG with a root)
    // root snapshots (copy 0 of the private per-CTA state)
    void* snap = nullptr;
    uint32_t* init_count = nullptr;
    double* init_sums = nullptr;
    uint32_t* init_adj = nullptr;
    int* init_assign = nullptr;
    int root_initial_live = 0;
    int* labels = nullptr;  // [edge*edge]
    int* lab_first = nullptr;
    int* lab_rank = nullptr;
    void* dmat = nullptr;
    size_t dmat_bytes = 0;
    rhseg_result_info info{};
    float phase_ms[4] = {0, 0, 0, 0};
    bool phases_valid = false;
    long long launches = 0;  // kernels launched by the last run (+ result copies since)
    // Device buffers cached across runs (grown, never shrunk, freed with the ctx):
    // repeated runs of one shape allocate nothing, so no run waits on the driver.
    std::map<int, std::pair<void*, size_t>> bufs;
    size_t dmat_budget = 0;  // bytes the D matrix may use (measured once per ctx)
    size_t l2_persist_bytes = 0;  // persisting-L2 set-aside granted at ctx creation
    // host-input pipeline (rhseg_run_host): a copy stream and per-chunk streams/events
    cudaStream_t copy_stream = nullptr;
    cudaStream_t pstream[8] = {};
    cudaEvent_t ready[8] = {}, done[9] = {};
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> evs;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
};

static cudaEvent_t ev_get(rhseg_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}
struct PhaseTimer {
    rhseg_ctx* c;
    int phase;
    cudaStream_t st;
    cudaEvent_t a;
    PhaseTimer(rhseg_ctx* c_, int p, cudaStream_t s) : c(c_), phase(p), st(s) {
        a = ev_get(c);
        cudaEventRecord(a, st);
    }
    ~PhaseTimer() {
        cudaEvent_t b = ev_get(c);
        cudaEventRecord(b, st);
        c->evs.push_back({phase, {a, b}});
    }
};

enum BufKey { kBufSnap = 1, kBufDmat = 2, kBufLog = 3, kBufCube = 4, kBufLogOff = 5, kBufLevel = 100 };

// Cached device buffer `key` with at least `bytes` (contents undefined).
static int get_buf(rhseg_ctx* c, int key, size_t bytes, void** out) {
    auto& b = c->bufs[key];
    if (b.second < bytes) {
        if (b.first) CK(cudaFree(b.first));
        b.first = nullptr;
        b.second = 0;
        CK(cudaMalloc(&b.first, std::max<size_t>(bytes, 256)));
        b.second = std::max<size_t>(bytes, 256);
    }
    *out = b.first;
    return RHSEG_OK;
}

static void free_level(Level& lv, cudaStream_t) { lv.work = lv.keep = nullptr; }  // buffers stay cached
static void free_work(Level& lv, cudaStream_t) { lv.work = nullptr; }

static void reset_ctx(rhseg_ctx* c, cudaStream_t st) {
    for (auto& lv : c->levels) free_level(lv, st);
    c->levels.clear();
    c->snap = nullptr;
    c->have = false;
    c->top = 1;
    c->phases_valid = false;
    c->launches = 0;
    c->evs.clear();
    c->ev_used = 0;
    memset(&c->info, 0, sizeof(c->info));
}

static int choose_cluster(const rhseg_ctx* c, int nsec, int R0max, int forced, bool apo_ok) {
    if (forced > 0) return forced;
    if (R0max < 512) return 1;
    // sections the one-CTA APO loop can hold run there even when few: C2's 16 leaves of
    // 1296 regions, 46.5 ms on 4-CTA clusters (mean stream) -> 33.1 ms (profiles/r02_experiments)
    if (apo_ok && R0max <= hseg_loop_max_rows()) return 1;
    int C = 1;
    while (C * 2 <= kMaxCluster && nsec * C * 2 <= c->nsm && R0max / (C * 2) >= 128) C *= 2;
    return C;
}

// Allocate and zero one level's device state. R0h/tgth must be filled.
// Grid loop selection: sections a cluster cannot hold, and a level that is ONE
// multi-CTA section (the whole GPU for it: C1's 4096-region HSEG, 88.6 ms on a 16-CTA
// cluster -> 69.8 ms); RHSEG_GRID=1 also every other multi-CTA section, RHSEG_GRID=0 only
// the sections a cluster cannot hold. A forced cluster size (rhseg_params.cluster) keeps
// the cluster loop.
static int grid_env() {
    static const int v = [] {
        const char* e = getenv("RHSEG_GRID");
        return e && *e ? atoi(e) : -1;
    }();
    return v;
}

static int alloc_level(rhseg_ctx* c, Level& lv, double weight, cudaStream_t st, int forced_C, int slot) {
    lv.R0max = 0;
    for (int r : lv.R0h) lv.R0max = std::max(lv.R0max, r);
    if (lv.R0max > c->max_regions)
        return fail(RHSEG_E_TOO_LARGE, "section with " + std::to_string(lv.R0max) + " regions: its " +
                                           "dissimilarity matrix exceeds device memory (max " +
                                           std::to_string(c->max_regions) + " regions)");
    lv.Rp = std::max(64, (lv.R0max + 63) / 64 * 64);
    lv.W = lv.Rp / 32;
    const bool spec = weight > 0.0;
    {
        const char* apo_env = getenv("RHSEG_APO");
        const bool apo_ok = hseg_apo_capable(spec, 1, lv.measure) && !(apo_env && apo_env[0] == '0');
        lv.C = choose_cluster(c, lv.nsec, lv.R0max, forced_C, apo_ok);
    }
    auto fits = [&](int C) {
        return hseg_loop_smem(lv.Rp, C, lv.B, spec, lv.measure, hseg_loop_stage_bytes(spec, C, lv.measure),
                              hseg_loop_default_stages()) <=
                   220 * 1024 &&
               (lv.Rp + C - 1) / C <= hseg_loop_max_rows();
    };
    // grow the cluster until the per-CTA row slice fits shared memory; sections no
    // cluster holds (or every cluster section under RHSEG_GRID=1) run on the grid loop
    while (lv.C < kMaxCluster && !fits(lv.C)) lv.C *= 2;
    lv.grid = !fits(lv.C) || lv.R0max > kMaxSectionRegions || (grid_env() == 1 && lv.C > 1) ||
              (grid_env() != 0 && forced_C <= 0 && lv.C > 1 && lv.nsec == 1);
    if (lv.grid) lv.C = 1;
    // stream ring geometry (runtime knobs). Deeper (4 x 32 KB) or bigger (2 x 96 KB)
    // rings for levels with at most one CTA per SM were both measured slower on C2
    // (47 -> 87 / 82 ms): the shared-memory carveout takes the L1 that the
    // adjacency and sums accesses live in.
    // APO (default where capable; RHSEG_APO=0 selects the mean-stream loop): row a' is
    // bounded from D rows a and b: no stream ring; the second mean buffer holds the
    // region-major means the exact re-evaluations read
    const char* apo_env = getenv("RHSEG_APO");
    const bool apo = !lv.grid && hseg_apo_capable(spec, lv.C, lv.measure) && !(apo_env && apo_env[0] == '0');
    const int stage_bytes = hseg_loop_stage_bytes(spec, lv.C, lv.measure);
    const int nstages = (apo || lv.grid) ? 0 : hseg_loop_default_stages();
    const size_t ns = (size_t)lv.nsec, Rp = (size_t)lv.Rp, B = (size_t)lv.B, W = (size_t)lv.W,
                 C = (size_t)lv.C, npx = (size_t)lv.edge * lv.edge;
    // keep block
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = o;
        o = align256(o + bytes);
        return at;
    };
    const size_t oR0 = take(ns * 4), oT = take(ns * 4), oCnt = take(ns * Rp * 4), oPar = take(ns * Rp * 4),
                 oAs = take(ns * npx * 4), oMap = take(ns * Rp * 4), oLa = take(ns * Rp * 4),
                 oLb = take(ns * Rp * 4), oLd = take(ns * Rp * 8), oLk = take(ns * Rp), oN = take(ns * 4),
                 oCv = take(ns * 4), oPr = take(ns * 8), oRs = take(ns * 8), oN2 = take(lv.measure == 2 ? ns * Rp * 8 : 0);
    const size_t keep_bytes = o;
    {
        int rc = get_buf(c, kBufLevel + 2 * slot, keep_bytes, &lv.keep);
        if (rc) return rc;
    }
    CK(cudaMemsetAsync(lv.keep, 0, keep_bytes, st));
    o = 0;
    const size_t oAdj = take(ns * C * Rp * W * 4);
    lv.work_zero = o;
    // w = 0 (adj_loop.cu, one CTA per section) keeps region-major means in mu2
    const bool adjl = !spec && lv.C == 1 && !lv.grid;
    const size_t oMu = take(ns * B * Rp * 8),
                 oMu2 = take(lv.grid ? 0 : spec ? (apo ? 2 : 1) * ns * B * Rp * 8 : (adjl ? ns * B * Rp * 8 : 0)),  // APO: versioned means
                 oRec = take(apo ? ns * Rp * 16 : 0),
                 oGs = take(lv.grid ? ns * grid_loop_scratch_bytes(c->nsm, lv.B, lv.W) : 0),
                 oSums = take(ns * C * Rp * B * 8);
    const size_t work_bytes = o;
    {
        int rc = get_buf(c, kBufLevel + 2 * slot + 1, work_bytes, &lv.work);
        if (rc) return rc;
    }
    CK(cudaMemsetAsync(lv.work, 0, lv.work_zero, st));
    char* K = static_cast<char*>(lv.keep);
    char* Wk = static_cast<char*>(lv.work);
    SectionBatch& b = lv.sb;
    b = SectionBatch{};
    b.nsec = lv.nsec;
    b.B = lv.B;
    b.Rp = lv.Rp;
    b.W = lv.W;
    b.C = lv.C;
    b.edge = lv.edge;
    b.npx = (int)npx;
    b.spec = spec ? 1 : 0;
    b.stage_bytes = stage_bytes;
    b.nstages = nstages;
    b.apo = apo ? 1 : 0;
    // a level whose streamed means fit the persisting L2 set-aside keeps them there
    b.l2_window_base = nullptr;
    b.l2_window_bytes = 0;
    if (spec && c->l2_persist_bytes > 0) {
        const size_t mub = (size_t)(oSums - oMu);  // mu (+ mu2 / fp32 copies) are contiguous
        if (mub <= c->l2_persist_bytes) {
            b.l2_window_base = Wk + oMu;
            b.l2_window_bytes = mub;
        }
    }
    b.measure = lv.measure;
    b.nrm2 = lv.measure == 2 ? reinterpret_cast<double*>(K + oN2) : nullptr;
    b.weight = weight;
    b.R0 = reinterpret_cast<int*>(K + oR0);
    b.target = reinterpret_cast<int*>(K + oT);
    b.count = reinterpret_cast<uint32_t*>(K + oCnt);
    b.parent = reinterpret_cast<int*>(K + oPar);
    b.assign = reinterpret_cast<int*>(K + oAs);
    b.log_a = reinterpret_cast<int*>(K + oLa);
    b.log_b = reinterpret_cast<int*>(K + oLb);
    b.log_d = reinterpret_cast<double*>(K + oLd);
    b.log_k = reinterpret_cast<uint8_t*>(K + oLk);
    b.nlog = reinterpret_cast<int*>(K + oN);
    b.conv = reinterpret_cast<int*>(K + oCv);
    b.pairs = reinterpret_cast<long long*>(K + oPr);
    b.nresc = reinterpret_cast<long long*>(K + oRs);
    b.adj = reinterpret_cast<uint32_t*>(Wk + oAdj);
    b.mu = reinterpret_cast<double*>(Wk + oMu);
    b.mu2 = (!lv.grid && (spec || adjl)) ? reinterpret_cast<double*>(Wk + oMu2) : nullptr;
    b.gscr = lv.grid ? reinterpret_cast<void*>(Wk + oGs) : nullptr;
    if (lv.grid) {
        const char* e = getenv("RHSEG_GRID_CTAS");  // cap on CTAs per section (experiments)
        b.G = e && *e ? std::max(0, atoi(e)) : 0;
    }
    b.apo_rec = apo ? reinterpret_cast<uint4*>(Wk + oRec) : nullptr;
    b.sums = reinterpret_cast<double*>(Wk + oSums);
    lv.map = reinterpret_cast<int*>(K + oMap);
    CK(cudaMemcpyAsync(const_cast<int*>(b.R0), lv.R0h.data(), ns * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(const_cast<int*>(b.target), lv.tgth.data(), ns * 4, cudaMemcpyHostToDevice, st));
    return RHSEG_OK;
}
// dinit + merge loop over D-sized chunks of sections, then union-find resolve.
static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static bool profiling();
static double g_t0 = 0.0;
#define RHSEG_TRACE(...)                                                          \
    do {                                                                          \
        if (profiling()) {                                                        \
            fprintf(stderr, "[rhseg trace] %8.3f ms  ", now_ms() - g_t0);         \
            fprintf(stderr, __VA_ARGS__);                                         \
            fputc('\n', stderr);                                                  \
        }                                                                         \
    } while (0)

static bool profiling() {
    static const bool on = [] {
        const char* e = getenv("RHSEG_PROFILE");
        return e && *e && *e != '0';
    }();
    return on;
}

// Leaf level fed chunk by chunk from host memory: chunk k (a band of leaf rows)
// becomes runnable when its upload (event ready[k]) lands; its leaf init, all-pairs
// D and merge loop then run on stream pstream[k], concurrently with the other
// chunks and with the remaining uploads.
struct LeafPipe {
    int K;
    const float* d_samples;
    int edge, cols, row0, col0, conn;
};

static int run_level(rhseg_ctx* c, Level& lv, cudaStream_t st, const LeafPipe* pipe = nullptr) {
    unsigned long long* prof = nullptr;
    if (profiling()) {
        CK(cudaMallocAsync(&prof, 16 * 8, st));
        CK(cudaMemsetAsync(prof, 0, 16 * 8, st));
    }
    lv.sb.prof = prof;
    const double t_enter = prof ? now_ms() : 0.0;
    const size_t dsec = (size_t)lv.Rp * lv.Rp * 8;
    RHSEG_TRACE("run_level %d: enter", lv.level);
    size_t chunk = (size_t)lv.nsec;
    if (c->dmat_bytes < chunk * dsec) {
        // D for every section of the level at once if it fits 60% of what is free
        // (queried only when the cached D is too small)
        size_t freeb = 0, totalb = 0;
        CK(cudaMemGetInfo(&freeb, &totalb));
        const size_t budget = (size_t)(0.6 * (double)(freeb + c->dmat_bytes));
        chunk = std::max<size_t>(1, std::min<size_t>(lv.nsec, budget / dsec));
        if (c->dmat_bytes < chunk * dsec) {
            int rc = get_buf(c, kBufDmat, chunk * dsec, &c->dmat);
            if (rc) return rc;
            c->dmat_bytes = chunk * dsec;
        }
        chunk = std::max<size_t>(1, std::min<size_t>(lv.nsec, c->dmat_bytes / dsec));
    }
    lv.sb.D = static_cast<double*>(c->dmat);
    if (pipe && chunk == (size_t)lv.nsec) {
        const int per = lv.nsec / pipe->K;
        PhaseTimer t(c, 2, st);
        CK(cudaEventRecord(c->done[pipe->K], st));  // level buffers are initialised on st
        for (int k = 0; k < pipe->K; ++k) {
            cudaStream_t sk = c->pstream[k];
            CK(cudaStreamWaitEvent(sk, c->done[pipe->K], 0));
            CK(cudaStreamWaitEvent(sk, c->ready[k], 0));
            SectionBatch b = lv.sb;
            b.sec0 = k * per;
            launch_leaf_init(b, pipe->d_samples, pipe->edge, pipe->cols, pipe->row0, pipe->col0, pipe->conn, sk,
                             per);
            b.D = lv.sb.D + (size_t)k * per * (dsec / 8);
            launch_dinit(b, per, lv.R0max, sk);
            int e = lv.grid ? launch_grid_loop(b, per, c->nsm, sk, &lv.gridG) : launch_hseg_loop(b, per, sk);
            if (e != cudaSuccess)
                return fail(RHSEG_E_CUDA, std::string("hseg loop launch: ") + cudaGetErrorString((cudaError_t)e));
            c->launches += 3;
            CK(cudaEventRecord(c->done[k], sk));
            CK(cudaStreamWaitEvent(st, c->done[k], 0));
        }
        CK(cudaGetLastError());
    } else {
        if (pipe) {  // D does not fit every section at once: upload everything, then chunk
            for (int k = 0; k < pipe->K; ++k) CK(cudaStreamWaitEvent(st, c->ready[k], 0));
            SectionBatch b = lv.sb;
            launch_leaf_init(b, pipe->d_samples, pipe->edge, pipe->cols, pipe->row0, pipe->col0, pipe->conn, st);
            c->launches += 1;
        }
        for (size_t s0 = 0; s0 < (size_t)lv.nsec; s0 += chunk) {
            const int n = (int)std::min(chunk, (size_t)lv.nsec - s0);
            SectionBatch b = lv.sb;
            b.sec0 = (int)s0;
            b.D = lv.sb.D;
            {
                PhaseTimer t(c, 1, st);
                launch_dinit(b, n, lv.R0max, st);
                c->launches += 1;
            }
            CK(cudaGetLastError());
            {
                PhaseTimer t(c, 2, st);
                int e = lv.grid ? launch_grid_loop(b, n, c->nsm, st, &lv.gridG) : launch_hseg_loop(b, n, st);
                c->launches += 1;
                if (e != cudaSuccess)
                    return fail(RHSEG_E_CUDA, std::string("hseg loop launch: ") + cudaGetErrorString((cudaError_t)e));
            }
            CK(cudaGetLastError());
        }
    }
    {
        PhaseTimer t(c, 3, st);
        launch_resolve(lv.sb, st);
        c->launches += 1;
    }
    CK(cudaGetLastError());
    RHSEG_TRACE("run_level %d: launched", lv.level);
    lv.nlogh.resize(lv.nsec);
    lv.convh.resize(lv.nsec);
    lv.pairsh.resize(lv.nsec);
    lv.rescsh.resize(lv.nsec);
    CK(cudaMemcpyAsync(lv.nlogh.data(), lv.sb.nlog, 4 * (size_t)lv.nsec, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(lv.convh.data(), lv.sb.conv, 4 * (size_t)lv.nsec, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(lv.pairsh.data(), lv.sb.pairs, 8 * (size_t)lv.nsec, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(lv.rescsh.data(), lv.sb.nresc, 8 * (size_t)lv.nsec, cudaMemcpyDeviceToHost, st));
    unsigned long long ph[16] = {0};
    if (prof) CK(cudaMemcpyAsync(ph, prof, 16 * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (lv.sb.l2_window_bytes) cudaCtxResetPersistingL2Cache();  // hand the set-aside back
    RHSEG_TRACE("run_level %d: synced", lv.level);
    if (prof) {
        long long steps = 0;
        for (int s = 0; s < lv.nsec; ++s) steps += lv.nlogh[s];
        const double tot = (double)(ph[0] + ph[1] + ph[2] + ph[3] + ph[4]) + 1e-9;
        fprintf(stderr,
                "[rhseg profile] level %d: %d sections x C=%d, Rp=%d, %lld steps, %.0f cycles/step (per CTA): "
                "%s %.1f%% %s %.1f%% %s %.1f%% %s %.1f%% %s %.1f%%, %.2f rescans/step\n",
                lv.level, lv.nsec, lv.C, lv.Rp, steps, tot / (double)std::max(1LL, steps) / lv.C,
                "argmin", 100 * ph[0] / tot, lv.sb.apo ? "rule" : "combine", 100 * ph[1] / tot,
                lv.sb.apo ? "merge||rescans" : "merge", 100 * ph[2] / tot, lv.sb.apo ? "row-a'+offers" : "row-a",
                100 * ph[3] / tot, lv.sb.apo ? "publish" : "rescan", 100 * ph[4] / tot,
                (double)ph[5] / (double)std::max(1LL, steps));
        if (ph[8] + ph[9] + ph[11])
            fprintf(stderr, "[rhseg profile] level %d APO per step: %.2f exact offers, %.2f a-candidates, "
                    "%.2f rescan exact pairs (%.0f cycles each)\n", lv.level, (double)ph[8] / std::max(1LL, steps),
                    (double)ph[9] / std::max(1LL, steps), (double)ph[11] / std::max(1LL, steps),
                    (double)ph[12] / std::max(1ULL, ph[11]));
        if (ph[10])
            fprintf(stderr, "[rhseg profile] level %d APO row-a' intervals (inside the last phase): %.0f cycles/step\n",
                    lv.level, (double)ph[10] / (double)std::max(1LL, steps));
        if (ph[14])
            fprintf(stderr, "[rhseg profile] level %d APO rescans: %.0f cycles per rescan (warp view), max warp %.0f\n",
                    lv.level, (double)ph[13] / ph[14], (double)ph[15]);
        cudaFree(prof);
        fprintf(stderr, "[rhseg profile] level %d host wall in run_level %.2f ms; per CTA: prologue %.0f cycles, "
                "kernel %.0f cycles\n", lv.level, now_ms() - t_enter, (double)ph[6] / (lv.nsec * lv.C),
                (double)ph[7] / (lv.nsec * lv.C));
    }
    lv.done = true;
    return RHSEG_OK;
}

static int snapshot_root(rhseg_ctx* c, Level& lv, cudaStream_t st) {
    const size_t Rp = lv.Rp, B = lv.B, W = lv.W, npx = (size_t)lv.edge * lv.edge;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = o;
        o = align256(o + bytes);
        return at;
    };
    const size_t oc = take(Rp * 4), os = take(Rp * B * 8), oa = take(Rp * W * 4), oas = take(npx * 4),
                 olab = take(npx * 4), of = take(Rp * 4), orank = take(Rp * 4);
    {
        int rc = get_buf(c, kBufSnap, o, &c->snap);
        if (rc) return rc;
    }
    char* S = static_cast<char*>(c->snap);
    c->init_count = reinterpret_cast<uint32_t*>(S + oc);
    c->init_sums = reinterpret_cast<double*>(S + os);
    c->init_adj = reinterpret_cast<uint32_t*>(S + oa);
    c->init_assign = reinterpret_cast<int*>(S + oas);
    c->labels = reinterpret_cast<int*>(S + olab);
    c->lab_first = reinterpret_cast<int*>(S + of);
    c->lab_rank = reinterpret_cast<int*>(S + orank);
    CK(cudaMemcpyAsync(c->init_count, lv.sb.count, Rp * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c->init_sums, lv.sb.sums, Rp * B * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c->init_adj, lv.sb.adj, Rp * W * 4, cudaMemcpyDeviceToDevice, st));
    if (npx) CK(cudaMemcpyAsync(c->init_assign, lv.sb.assign, npx * 4, cudaMemcpyDeviceToDevice, st));
    c->root_initial_live = lv.R0h[0];
    return RHSEG_OK;
}

static void finish_info(rhseg_ctx* c) {
    rhseg_result_info& I = c->info;
    I.n_records = 0;
    I.spectral_pairs = 0;
    I.n_sections = 0;
    I.converged_early = 0;
    for (auto& lv : c->levels) {
        if (lv.imported) continue;
        for (int s = 0; s < lv.nsec; ++s) {
            I.n_records += lv.nlogh[s];
            I.spectral_pairs += lv.pairsh[s];
            I.converged_early |= lv.convh[s] ? 1 : 0;
        }
        I.n_sections += lv.nsec;
    }
    I.levels = c->L;
    I.edge = c->edge;
    I.bands = c->bands;
    if (c->top == 1) {
        Level& root = c->levels.back();
        I.root_idspace = root.R0h[0];
        I.root_initial_regions = c->root_initial_live;
        I.root_regions = root.R0h[0] - root.nlogh[0];
    }
}

static void finish_phases(rhseg_ctx* c) {
    for (int p = 0; p < 4; ++p) c->phase_ms[p] = 0.f;
    for (auto& e : c->evs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e.second.first, e.second.second);
        c->phase_ms[e.first] += ms;
    }
    c->phases_valid = true;
}

static int validate(const rhseg_params* p, int edge, int bands, long long max_regions) {
    if (!p) return fail(RHSEG_E_INVALID, "params is NULL");
    if (!(p->spectral_weight >= 0.0 && p->spectral_weight <= 1.0))
        return fail(RHSEG_E_INVALID, "spectral_weight must be in [0, 1]");
    if (p->target_regions < 1) return fail(RHSEG_E_INVALID, "target_regions must be >= 1");
    if (p->section_target_regions < 0) return fail(RHSEG_E_INVALID, "section_target_regions must be >= 1");
    if (p->levels < 1) return fail(RHSEG_E_INVALID, "levels must be >= 1");
    if (p->connectivity != 4 && p->connectivity != 8) return fail(RHSEG_E_INVALID, "connectivity must be 4 or 8");
    if (p->measure < 0 || p->measure > 2)
        return fail(RHSEG_E_INVALID, "unknown measure; available: ['euclidean', 'sam', 'sqrt-bsmse']");
    if (edge < 1 || bands < 1) return fail(RHSEG_E_INVALID, "width and bands must be >= 1");
    if (p->levels > 30) return fail(RHSEG_E_INVALID, "levels too large");
    const long long side = 1LL << (p->levels - 1);
    if (edge % side != 0)
        return fail(RHSEG_E_INDIVISIBLE, "edge " + std::to_string(edge) + " not divisible by " +
                                             std::to_string(side) + " (levels=" + std::to_string(p->levels) + ")");
    if (p->cluster != 0 && p->cluster != 1 && p->cluster != 2 && p->cluster != 4 && p->cluster != 8 &&
        p->cluster != 16)
        return fail(RHSEG_E_INVALID, "cluster must be 0 (auto) or one of 1,2,4,8,16");
    // Worst-case section sizes, checked before anything is launched: a leaf holds e*e
    // regions and a parent the live regions of its four children, at most
    // 4 * min(child size, section target) -- image sections are connected grids, so no
    // section stops above its target (RHSEG_E_TOO_LARGE is a documented deviation).
    {
        const long long e = edge / side, sect = p->section_target_regions > 0 ? p->section_target_regions
                                                                            : p->target_regions;
        long long R = e * e;
        if (R > max_regions)
            return fail(RHSEG_E_TOO_LARGE, "leaf sections of " + std::to_string(e) + "x" + std::to_string(e) +
                                               " pixels exceed " + std::to_string(max_regions) +
                                               " regions (the dissimilarity matrix would not fit device memory)");
        for (int level = p->levels - 1; level >= 1; --level) {
            R = 4 * std::min(R, sect);
            if (R > max_regions)
                return fail(RHSEG_E_TOO_LARGE, "level-" + std::to_string(level) + " sections can hold " +
                                                   std::to_string(R) + " regions (section_target_regions " +
                                                   std::to_string(sect) + "), above the " +
                                                   std::to_string(max_regions) + "-region limit of device memory");
        }
    }
    return RHSEG_OK;
}

// Stitch the back level into its parents and run HSEG on them, level by level,
// until `stop_level` has been processed (recursive.py:145-170 run_upper_levels).
static int upper_levels(rhseg_ctx* c, const rhseg_params* p, int stop_level, cudaStream_t st) {
    const int sect = p->section_target_regions > 0 ? p->section_target_regions : p->target_regions;
    for (int level = c->levels.back().level - 1; level >= stop_level; --level) {
        Level& ch = c->levels.back();
        Level pa;
        pa.level = level;
        pa.rows = ch.rows / 2;
        pa.cols = ch.cols / 2;
        pa.row0 = ch.row0 / 2;
        pa.col0 = ch.col0 / 2;
        pa.nsec = pa.rows * pa.cols;
        pa.edge = ch.edge * 2;
        pa.B = c->bands;
        pa.measure = p->measure;
        pa.R0h.assign(pa.nsec, 0);
        for (int P = 0; P < pa.nsec; ++P) {
            const int pr = P / pa.cols, pc = P % pa.cols;
            for (int k = 0; k < 4; ++k) {
                const int ci = (2 * pr + (k >> 1)) * ch.cols + (2 * pc + (k & 1));
                pa.R0h[P] += ch.R0h[ci] - ch.nlogh[ci];
            }
        }
        pa.tgth.assign(pa.nsec, level == 1 ? p->target_regions : sect);
        RHSEG_TRACE("level %d: alloc", level);
        int rc = alloc_level(c, pa, p->spectral_weight, st, p->cluster, (int)c->levels.size());
        RHSEG_TRACE("level %d: alloc done", level);
        if (rc) return rc;
        {
            PhaseTimer t(c, 0, st);
            launch_stitch(ch.sb, ch.cols, pa.sb, pa.cols, ch.map, p->connectivity, st);
            c->launches += 3;  // stitch, pixel assignment, seam links
        }
        CK(cudaGetLastError());
        if (ch.imported) free_level(ch, st);
        else free_work(ch, st);
        c->levels.push_back(std::move(pa));
        Level& lv = c->levels.back();
        if (level == 1) {
            rc = snapshot_root(c, lv, st);
            if (rc) return rc;
        }
        rc = run_level(c, lv, st);
        if (rc) return rc;
    }
    return RHSEG_OK;
}

static int finish_run(rhseg_ctx* c, cudaStream_t st) {
    RHSEG_TRACE("finish");
    if (c->top == 1) {
        Level& root = c->levels.back();
        PhaseTimer t(c, 3, st);
        launch_dense_labels(root.sb.assign, c->edge * c->edge, root.Rp, c->lab_first, c->lab_rank, c->labels, st);
        c->launches += 3;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    c->have = true;
    finish_info(c);
    finish_phases(c);
    return RHSEG_OK;
}

// Levels L..top over the block [r0, r0+nr) x [c0, c0+nc) of the level-`top`
// section grid; top = 1 with the 1x1 block is SequentialExecutor.execute
// (recursive.py:173-209). A block of level-`top` subtrees is the unit a rank
// owns under multi-GPU sharding.
static int ensure_pipeline(rhseg_ctx* c) {
    if (c->copy_stream) return RHSEG_OK;
    CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 8; ++k) {
        CK(cudaStreamCreateWithFlags(&c->pstream[k], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ready[k], cudaEventDisableTiming));
    }
    for (int k = 0; k < 9; ++k) CK(cudaEventCreateWithFlags(&c->done[k], cudaEventDisableTiming));
    return RHSEG_OK;
}

// h_samples (optional): the same cube in host memory; the leaf level is then fed
// chunk by chunk while it uploads into d_samples (rhseg_run_host).
static int run_device_impl(rhseg_ctx* c, const float* d_samples, int edge, int bands, const rhseg_params* p,
                           int top, int r0, int c0, int nr, int nc, cudaStream_t st,
                           const float* h_samples = nullptr) {
    int rc = validate(p, edge, bands, c->max_regions);
    if (rc) return rc;
    const int L = p->levels;
    if (top < 1 || top > L) return fail(RHSEG_E_INVALID, "top_level must be in [1, levels]");
    const int tside = 1 << (top - 1);
    if (nr < 1 || nc < 1 || r0 < 0 || c0 < 0 || r0 + nr > tside || c0 + nc > tside)
        return fail(RHSEG_E_INVALID, "subtree block outside the level grid");
    CK(cudaSetDevice(c->device));
    g_t0 = now_ms();
    RHSEG_TRACE("run start");
    reset_ctx(c, st);
    RHSEG_TRACE("reset done");
    c->edge = edge;
    c->bands = bands;
    c->L = L;
    c->top = top;
    const int sect = p->section_target_regions > 0 ? p->section_target_regions : p->target_regions;
    const int side = 1 << (L - 1);
    const int e = edge / side;
    c->levels.reserve(L);
    // ---- leaves ----
    {
        c->levels.emplace_back();
        Level& lv = c->levels.back();
        const int scale = 1 << (L - top);
        lv.level = L;
        lv.rows = nr * scale;
        lv.cols = nc * scale;
        lv.row0 = r0 * scale;
        lv.col0 = c0 * scale;
        lv.nsec = lv.rows * lv.cols;
        lv.edge = e;
        lv.B = bands;
        lv.measure = p->measure;
        lv.R0h.assign(lv.nsec, e * e);
        lv.tgth.assign(lv.nsec, L == 1 ? p->target_regions : sect);
        RHSEG_TRACE("leaves: alloc");
        rc = alloc_level(c, lv, p->spectral_weight, st, p->cluster, 0);
        RHSEG_TRACE("leaves: alloc done");
        if (rc) return rc;
        // RHSEG_DEV_PIPE=1: the device-resident path runs the leaf level in the same chunks
        // on concurrent streams (the FP64-bound all-pairs init of one chunk beside the
        // latency-bound merge loops of the others)
        static const bool dev_pipe = [] {
            const char* e = getenv("RHSEG_DEV_PIPE");
            return e && e[0] == '1';
        }();
        const bool piped = (h_samples || dev_pipe) && L >= 2 && top == 1;
        if (piped) {
            // upload in K bands of leaf rows on the copy stream; chunk k starts as soon
            // as its rows land (run_level / LeafPipe)
            rc = ensure_pipeline(c);
            if (rc) return rc;
            LeafPipe pipe{std::min(8, lv.rows), d_samples, edge, lv.cols, lv.row0, lv.col0, p->connectivity};
            const size_t rows = (size_t)edge / pipe.K, plane = (size_t)edge * edge;
            for (int k = 0; k < pipe.K; ++k) {
                const size_t off = (size_t)k * rows * edge;
                if (h_samples) {
                    CK(cudaMemcpy2DAsync(const_cast<float*>(d_samples) + off, plane * 4, h_samples + off, plane * 4,
                                         rows * edge * 4, (size_t)bands, cudaMemcpyHostToDevice, c->copy_stream));
                    CK(cudaEventRecord(c->ready[k], c->copy_stream));
                } else {
                    CK(cudaEventRecord(c->ready[k], st));  // (resident: ready now)
                }
            }
            rc = run_level(c, lv, st, &pipe);
            if (rc) return rc;
        } else {
            {
                PhaseTimer t(c, 0, st);
                launch_leaf_init(lv.sb, d_samples, edge, lv.cols, lv.row0, lv.col0, p->connectivity, st);
                c->launches += 1;
            }
            CK(cudaGetLastError());
            if (L == 1) {
                rc = snapshot_root(c, lv, st);
                if (rc) return rc;
            }
            rc = run_level(c, lv, st);
            if (rc) return rc;
        }
    }
    rc = upper_levels(c, p, top, st);
    if (rc) return rc;
    return finish_run(c, st);
}

// ---- section state exchange (multi-GPU reassembly) -------------
// One packed section: count u32[rp] | sums f64[rp][B] | adjacency u32[rp][rp/32]
// | assignment i32[e*e], each segment 256-byte aligned.
struct PackLayout {
    size_t cnt, sums, adj, asg, bytes;
};
static PackLayout pack_layout(int rp, int B, int e) {
    PackLayout P;
    size_t o = 0;
    P.cnt = o;
    o = align256(o + 4 * (size_t)rp);
    P.sums = o;
    o = align256(o + 8 * (size_t)rp * B);
    P.adj = o;
    o = align256(o + 4 * (size_t)rp * (rp / 32));
    P.asg = o;
    o = align256(o + 4 * (size_t)e * e);
    P.bytes = o;
    return P;
}

// ===========================================================================
// exported C ABI
// ===========================================================================
extern "C" {

int rhseg_abi_version(void) { return RHSEG_ABI_VERSION; }
const char* rhseg_last_error(void) { return g_err.c_str(); }

int rhseg_ctx_create(int device, rhseg_ctx** out) {
    if (!out) return fail(RHSEG_E_INVALID, "out is NULL");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(RHSEG_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(RHSEG_E_INVALID, "bad device index");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(RHSEG_E_CUDA, std::string("librhseg_b200 is built for sm_100a; device is ") + prop.name);
    rhseg_ctx* c = new rhseg_ctx();
    c->device = device;
    c->nsm = prop.multiProcessorCount;
    {   // the largest section whose D (R^2 fp64) plus adjacency bitset takes at most 75% of HBM
        const double per2 = 8.0 + 1.0 / 8.0;
        long long r = (long long)std::sqrt(0.75 * (double)prop.totalGlobalMem / per2);
        c->max_regions = std::max<long long>(kMaxSectionRegions, r / 64 * 64);
    }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    {   // persisting-L2 set-aside for small levels' streamed means (best effort)
        int maxp = 0;
        if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device) == cudaSuccess && maxp > 0) {
            const size_t want = std::min<size_t>((size_t)maxp, (size_t)RHSEG_L2_PERSIST_MB << 20);
            if (want > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess)
                c->l2_persist_bytes = want;
        }
        cudaGetLastError();
    }
    *out = c;
    return RHSEG_OK;
}

int rhseg_ctx_destroy(rhseg_ctx* c) {
    if (!c) return RHSEG_OK;
    cudaSetDevice(c->device);
    reset_ctx(c, c->stream);
    cudaStreamSynchronize(c->stream);
    for (auto& kv : c->bufs)
        if (kv.second.first) cudaFree(kv.second.first);
    c->bufs.clear();
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->copy_stream) {
        cudaStreamDestroy(c->copy_stream);
        for (int k = 0; k < 8; ++k) {
            cudaStreamDestroy(c->pstream[k]);
            cudaEventDestroy(c->ready[k]);
        }
        for (int k = 0; k < 9; ++k) cudaEventDestroy(c->done[k]);
    }
    cudaStreamDestroy(c->stream);
    delete c;
    return RHSEG_OK;
}

int rhseg_run_device(rhseg_ctx* c, const float* d_samples, int32_t edge, int32_t bands, const rhseg_params* p,
                     void* stream) {
    if (!c) return fail(RHSEG_E_INVALID, "ctx is NULL");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    return run_device_impl(c, d_samples, edge, bands, p, 1, 0, 0, 1, 1, st);
}

int rhseg_run_subtrees(rhseg_ctx* c, const float* d_samples, int32_t edge, int32_t bands, const rhseg_params* p,
                       int32_t top_level, int32_t r0, int32_t c0, int32_t nr, int32_t nc, void* stream) {
    if (!c) return fail(RHSEG_E_INVALID, "ctx is NULL");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    return run_device_impl(c, d_samples, edge, bands, p, top_level, r0, c0, nr, nc, st);
}

int rhseg_top_info(rhseg_ctx* c, int32_t* nsec, int32_t* rp, int32_t* sec_edge, int32_t* R0, int32_t* nlog) {
    if (!c || !c->have) return fail(RHSEG_E_STATE, "no result");
    const Level& lv = c->levels.back();
    if (nsec) *nsec = lv.nsec;
    if (rp) *rp = lv.Rp;
    if (sec_edge) *sec_edge = lv.edge;
    for (int s = 0; s < lv.nsec; ++s) {
        if (R0) R0[s] = lv.R0h[s];
        if (nlog) nlog[s] = lv.nlogh[s];
    }
    return RHSEG_OK;
}

int rhseg_pack_bytes(int32_t rp, int32_t bands, int32_t sec_edge, int64_t* bytes) {
    if (!bytes || rp < 32 || rp % 32 || bands < 1 || sec_edge < 1) return fail(RHSEG_E_INVALID, "bad pack shape");
    *bytes = (int64_t)pack_layout(rp, bands, sec_edge).bytes;
    return RHSEG_OK;
}

int rhseg_export_top(rhseg_ctx* c, int32_t rp, void* d_pack, void* stream) {
    if (!c || !c->have) return fail(RHSEG_E_STATE, "no result");
    const Level& lv = c->levels.back();
    if (lv.imported || lv.work == nullptr) return fail(RHSEG_E_STATE, "top level state is not resident");
    if (rp < lv.Rp || rp % 32) return fail(RHSEG_E_INVALID, "rp must be a multiple of 32 and >= the level's Rp");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    const PackLayout P = pack_layout(rp, lv.B, lv.edge);
    const size_t B = lv.B, W = lv.W, Wo = rp / 32, npx = (size_t)lv.edge * lv.edge;
    char* out = static_cast<char*>(d_pack);
    CK(cudaMemsetAsync(out, 0, P.bytes * lv.nsec, st));
    for (int s = 0; s < lv.nsec; ++s) {
        char* o = out + P.bytes * s;
        const size_t R0 = lv.R0h[s];
        CK(cudaMemcpyAsync(o + P.cnt, lv.sb.count + (size_t)s * lv.Rp, 4 * R0, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(o + P.sums, lv.sb.sums + (size_t)s * lv.C * lv.sb.sums_copy(), 8 * R0 * B,
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpy2DAsync(o + P.adj, 4 * Wo, lv.sb.adj + (size_t)s * lv.C * lv.sb.adj_copy(), 4 * W, 4 * W, R0,
                             cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(o + P.asg, lv.sb.assign + (size_t)s * npx, 4 * npx, cudaMemcpyDeviceToDevice, st));
    }
    return RHSEG_OK;
}

int rhseg_run_upper(rhseg_ctx* c, const void* d_pack, int32_t top_level, int32_t rp, const int32_t* R0,
                    const int32_t* nlog, int32_t edge, int32_t bands, const rhseg_params* p, void* stream) {
    if (!c) return fail(RHSEG_E_INVALID, "ctx is NULL");
    int rc = validate(p, edge, bands, c->max_regions);
    if (rc) return rc;
    if (top_level < 2 || top_level > p->levels) return fail(RHSEG_E_INVALID, "top_level must be in [2, levels]");
    if (rp < 32 || rp % 32) return fail(RHSEG_E_INVALID, "rp must be a positive multiple of 32");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    reset_ctx(c, st);
    c->edge = edge;
    c->bands = bands;
    c->L = p->levels;
    c->top = 1;
    const int tside = 1 << (top_level - 1);
    c->levels.reserve(top_level + 1);
    c->levels.emplace_back();
    Level& lv = c->levels.back();
    lv.level = top_level;
    lv.rows = lv.cols = tside;
    lv.nsec = tside * tside;
    lv.edge = edge / tside;
    lv.B = bands;
    lv.measure = p->measure;
    lv.imported = true;
    lv.R0h.assign(R0, R0 + lv.nsec);
    lv.nlogh.assign(nlog, nlog + lv.nsec);
    lv.convh.assign(lv.nsec, 0);
    lv.pairsh.assign(lv.nsec, 0);
    lv.rescsh.assign(lv.nsec, 0);
    lv.tgth.assign(lv.nsec, 1);
    int rpmax = 0;
    for (int r : lv.R0h) rpmax = std::max(rpmax, r);
    if (rpmax > rp) return fail(RHSEG_E_INVALID, "a section's R0 exceeds rp");
    rc = alloc_level(c, lv, p->spectral_weight, st, 1, 0);
    if (rc) return rc;
    const PackLayout P = pack_layout(rp, bands, lv.edge);
    const size_t B = bands, W = lv.W, Wi = rp / 32, npx = (size_t)lv.edge * lv.edge;
    const char* in = static_cast<const char*>(d_pack);
    for (int s = 0; s < lv.nsec; ++s) {
        const char* o = in + P.bytes * s;
        const size_t r0 = lv.R0h[s];
        CK(cudaMemcpyAsync(lv.sb.count + (size_t)s * lv.Rp, o + P.cnt, 4 * r0, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(lv.sb.sums + (size_t)s * lv.sb.sums_copy(), o + P.sums, 8 * r0 * B,
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpy2DAsync(lv.sb.adj + (size_t)s * lv.sb.adj_copy(), 4 * W, o + P.adj, 4 * Wi,
                             4 * std::min(W, Wi), r0, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(lv.sb.assign + (size_t)s * npx, o + P.asg, 4 * npx, cudaMemcpyDeviceToDevice, st));
    }
    lv.done = true;
    rc = upper_levels(c, p, 1, st);
    if (rc) return rc;
    return finish_run(c, st);
}

int rhseg_result_info_get(rhseg_ctx* c, rhseg_result_info* info) {
    if (!c || !c->have) return fail(RHSEG_E_STATE, "no result");
    *info = c->info;
    info->device_ms = c->phase_ms[0] + c->phase_ms[1] + c->phase_ms[2] + c->phase_ms[3];
    return RHSEG_OK;
}

int rhseg_result_phase_ms(rhseg_ctx* c, float* ms4) {
    if (!c || !c->phases_valid) return fail(RHSEG_E_STATE, "no timed run");
    for (int p = 0; p < 4; ++p) ms4[p] = c->phase_ms[p];
    return RHSEG_OK;
}

int rhseg_result_rescans(rhseg_ctx* c, int32_t level, int64_t* n) {
    if (!c || !n) return fail(RHSEG_E_INVALID, "NULL argument");
    long long t = 0;
    for (auto& lv : c->levels)
        if (!lv.imported && (level <= 0 || lv.level == level))
            for (long long x : lv.rescsh) t += x;
    *n = t;
    return RHSEG_OK;
}

int rhseg_result_level_info(rhseg_ctx* c, int32_t level, int32_t* nsec, int32_t* rp, int32_t* cluster,
                            int32_t* loop_variant, int64_t* merges) {
    if (!c) return fail(RHSEG_E_INVALID, "NULL argument");
    for (auto& lv : c->levels) {
        if (lv.imported || lv.level != level) continue;
        if (nsec) *nsec = lv.nsec;
        if (rp) *rp = lv.Rp;
        if (cluster) *cluster = lv.grid ? lv.gridG : lv.C;
        if (loop_variant) {
            static const bool recut = [] {
                const char* e = getenv("RHSEG_APO_V2");
                return e && e[0] == '1';
            }();
            *loop_variant = lv.grid ? RHSEG_LOOP_GRID
                            : !lv.sb.spec ? RHSEG_LOOP_ADJACENT
                            : lv.sb.apo ? (recut ? RHSEG_LOOP_APO_RECUT : RHSEG_LOOP_APO)
                                        : RHSEG_LOOP_STREAM;
        }
        if (merges) {
            long long t = 0;
            for (int x : lv.nlogh) t += x;
            *merges = t;
        }
        return RHSEG_OK;
    }
    return fail(RHSEG_E_INVALID, "level " + std::to_string(level) + " was not run by this context");
}

int rhseg_result_launches(rhseg_ctx* c, int64_t* n) {
    if (!c || !n) return fail(RHSEG_E_INVALID, "NULL argument");
    *n = c->launches;
    return RHSEG_OK;
}

int rhseg_result_sections(rhseg_ctx* c, int32_t* level, int32_t* row, int32_t* col, int64_t* offset,
                          int64_t* count) {
    if (!c || !c->have) return fail(RHSEG_E_STATE, "no result");
    int64_t off = 0;
    int k = 0;
    for (auto& lv : c->levels) {
        if (lv.imported) continue;
        for (int s = 0; s < lv.nsec; ++s, ++k) {
            if (level) level[k] = lv.level;
            if (row) row[k] = lv.row0 + s / lv.cols;
            if (col) col[k] = lv.col0 + s % lv.cols;
            if (offset) offset[k] = off;
            if (count) count[k] = lv.nlogh[s];
            off += lv.nlogh[s];
        }
    }
    return RHSEG_OK;
}

// Concatenate the per-section device logs in log order (level L..top,
// row-major) into device arrays of n_records entries.
static int compact_log(rhseg_ctx* c, int32_t* da, int32_t* db, double* dd, uint8_t* dk, cudaStream_t st) {
    std::vector<long long> off;
    std::vector<size_t> first;
    for (auto& lv : c->levels) {
        first.push_back(off.size());
        if (lv.imported) continue;
        for (int s = 0; s < lv.nsec; ++s) off.push_back(0);
    }
    long long base = 0;
    {
        size_t k = 0;
        for (auto& lv : c->levels) {
            if (lv.imported) continue;
            for (int s = 0; s < lv.nsec; ++s, ++k) {
                off[k] = base;
                base += lv.nlogh[s];
            }
        }
    }
    if (base == 0) return RHSEG_OK;
    long long* doff = nullptr;
    {
        void* p = nullptr;
        int rc = get_buf(c, kBufLogOff, 8 * off.size(), &p);
        if (rc) return rc;
        doff = static_cast<long long*>(p);
    }
    CK(cudaMemcpyAsync(doff, off.data(), 8 * off.size(), cudaMemcpyHostToDevice, st));
    for (size_t L = 0; L < c->levels.size(); ++L) {
        Level& lv = c->levels[L];
        if (lv.imported) continue;
        compact_log_kernel<<<lv.nsec, 256, 0, st>>>(lv.sb.log_a, lv.sb.log_b, lv.sb.log_d, lv.sb.log_k, lv.sb.nlog,
                                                    doff + first[L], lv.Rp, da, db, dd, dk);
        CK(cudaGetLastError());
        c->launches += 1;
    }
    CK(cudaStreamSynchronize(st));  // `off` must outlive the async H2D copy
    return RHSEG_OK;
}

static int copy_log(rhseg_ctx* c, int32_t* sa, int32_t* sb, double* sd, uint8_t* sk, cudaStream_t st) {
    const int64_t n = c->info.n_records;
    if (n == 0) return RHSEG_OK;
    int* da = nullptr;
    {
        void* p = nullptr;
        int rc = get_buf(c, kBufLog, (size_t)n * 17 + 1024, &p);
        if (rc) return rc;
        da = static_cast<int*>(p);
    }
    int* db = da + n;
    double* dd = reinterpret_cast<double*>(db + n);  // 2n ints: 8-byte aligned
    uint8_t* dk = reinterpret_cast<uint8_t*>(dd + n);
    int rc = compact_log(c, da, db, dd, dk, st);
    if (rc) return rc;
    if (sa) CK(cudaMemcpyAsync(sa, da, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
    if (sb) CK(cudaMemcpyAsync(sb, db, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
    if (sd) CK(cudaMemcpyAsync(sd, dd, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
    if (sk) CK(cudaMemcpyAsync(sk, dk, (size_t)n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return RHSEG_OK;
}

int rhseg_result_log_device(rhseg_ctx* c, int32_t* survivor, int32_t* absorbed, double* dissim, uint8_t* kind,
                            void* stream) {
    if (!c || !c->have) return fail(RHSEG_E_STATE, "no result");
    if (!survivor || !absorbed || !dissim || !kind) return fail(RHSEG_E_INVALID, "NULL device buffer");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    return compact_log(c, survivor, absorbed, dissim, kind, st);
}

int rhseg_result_log(rhseg_ctx* c, int32_t* survivor, int32_t* absorbed, double* dissim, uint8_t* kind) {
    if (!c || !c->have) return fail(RHSEG_E_STATE, "no result");
    CK(cudaSetDevice(c->device));
    return copy_log(c, survivor, absorbed, dissim, kind, c->stream);
}

int rhseg_result_labels(rhseg_ctx* c, int32_t* labels, int32_t* assignment) {
    if (!c || !c->have) return fail(RHSEG_E_STATE, "no result");
    if (c->top != 1) return fail(RHSEG_E_STATE, "partial (subtree) run has no root labels");
    CK(cudaSetDevice(c->device));
    const size_t npx = (size_t)c->edge * c->edge;
    if (labels) CK(cudaMemcpyAsync(labels, c->labels, npx * 4, cudaMemcpyDeviceToHost, c->stream));
    if (assignment)
        CK(cudaMemcpyAsync(assignment, c->levels.back().sb.assign, npx * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return RHSEG_OK;
}

int rhseg_result_root(rhseg_ctx* c, int32_t which, int64_t* counts, double* sums, uint32_t* adjacency,
                      int32_t* assignment) {
    if (!c || !c->have) return fail(RHSEG_E_STATE, "no result");
    if (c->top != 1) return fail(RHSEG_E_STATE, "partial (subtree) run has no root graph");
    CK(cudaSetDevice(c->device));
    Level& root = c->levels.back();
    const size_t R = (size_t)root.R0h[0], B = (size_t)root.B, Rp = root.Rp, W = root.W;
    const size_t Wo = (R + 31) / 32, npx = (size_t)c->edge * c->edge;
    const uint32_t* cnt = which == 0 ? c->init_count : root.sb.count;
    const double* sm = which == 0 ? c->init_sums : root.sb.sums;
    const uint32_t* ad = which == 0 ? c->init_adj : root.sb.adj;
    const int* as = which == 0 ? c->init_assign : root.sb.assign;
    std::vector<uint32_t> hc(Rp);
    CK(cudaMemcpyAsync(hc.data(), cnt, Rp * 4, cudaMemcpyDeviceToHost, c->stream));
    if (sums) CK(cudaMemcpyAsync(sums, sm, R * B * 8, cudaMemcpyDeviceToHost, c->stream));
    if (adjacency)
        CK(cudaMemcpy2DAsync(adjacency, Wo * 4, ad, W * 4, Wo * 4, R, cudaMemcpyDeviceToHost, c->stream));
    if (assignment) CK(cudaMemcpyAsync(assignment, as, npx * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (counts)
        for (size_t i = 0; i < R; ++i) counts[i] = hc[i];
    return RHSEG_OK;
}

int rhseg_run_host(rhseg_ctx* c, const float* h_samples, int32_t edge, int32_t bands, const rhseg_params* p,
                   void* stream, int32_t* log_survivor, int32_t* log_absorbed, double* log_dissim,
                   uint8_t* log_kind, int32_t* labels, rhseg_result_info* info) {
    if (!c) return fail(RHSEG_E_INVALID, "ctx is NULL");
    int rc = validate(p, edge, bands, c->max_regions);
    if (rc) return rc;
    CK(cudaSetDevice(c->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    const size_t bytes = (size_t)edge * edge * bands * sizeof(float);
    float* d = nullptr;
    {
        void* p = nullptr;
        rc = get_buf(c, kBufCube, bytes, &p);
        if (rc) return rc;
        d = static_cast<float*>(p);
    }
    if (p->levels >= 2) {  // leaf chunks start while the rest of the cube uploads
        rc = run_device_impl(c, d, edge, bands, p, 1, 0, 0, 1, 1, st, h_samples);
    } else {
        CK(cudaMemcpyAsync(d, h_samples, bytes, cudaMemcpyHostToDevice, st));
        rc = run_device_impl(c, d, edge, bands, p, 1, 0, 0, 1, 1, st);
    }
    if (rc) return rc;
    rc = copy_log(c, log_survivor, log_absorbed, log_dissim, log_kind, st);
    if (rc) return rc;
    if (labels) {
        CK(cudaMemcpyAsync(labels, c->labels, (size_t)edge * edge * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    if (info) rhseg_result_info_get(c, info);
    return RHSEG_OK;
}

int rhseg_hseg_graph(rhseg_ctx* c, int64_t n, int64_t nbands, const double* counts, const double* sums,
                     const int64_t* indptr, const int64_t* indices, double weight, int64_t target, int32_t cluster,
                     int32_t measure,
                     int32_t* log_survivor, int32_t* log_absorbed, double* log_dissim, uint8_t* log_kind,
                     int64_t* n_records, int32_t* converged_early) {
    if (!c) return fail(RHSEG_E_INVALID, "ctx is NULL");
    if (!(weight >= 0.0 && weight <= 1.0)) return fail(RHSEG_E_INVALID, "spectral_weight must be in [0, 1]");
    if (measure < 0 || measure > 2)
        return fail(RHSEG_E_INVALID, "unknown measure; available: ['euclidean', 'sam', 'sqrt-bsmse']");
    if (target < 1) return fail(RHSEG_E_INVALID, "target_regions must be >= 1");
    if (n < 0 || nbands < 1) return fail(RHSEG_E_INVALID, "bad graph shape");
    if (n > c->max_regions)
        return fail(RHSEG_E_TOO_LARGE, "graph of " + std::to_string(n) + " regions: its dissimilarity matrix " +
                                           "exceeds device memory (max " + std::to_string(c->max_regions) + ")");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    reset_ctx(c, st);
    if (n == 0) {
        *n_records = 0;
        *converged_early = 0;
        return RHSEG_OK;
    }
    c->levels.emplace_back();
    Level& lv = c->levels.back();
    lv.level = 1;
    lv.rows = lv.cols = 1;
    lv.nsec = 1;
    lv.edge = 0;
    lv.B = (int)nbands;
    lv.measure = measure;
    lv.R0h.assign(1, (int)n);
    lv.tgth.assign(1, (int)std::min<int64_t>(target, INT32_MAX));
    int rc = alloc_level(c, lv, weight, st, cluster, 0);
    if (rc) return rc;
    const int64_t nnz = indptr[n];
    void* tmp = nullptr;
    const size_t b_counts = align256(8 * (size_t)n), b_sums = align256(8 * (size_t)n * nbands),
                 b_ptr = align256(8 * (size_t)(n + 1)), b_idx = align256(8 * (size_t)std::max<int64_t>(nnz, 1));
    CK(cudaMallocAsync(&tmp, b_counts + b_sums + b_ptr + b_idx, st));
    char* T = static_cast<char*>(tmp);
    double* dc = reinterpret_cast<double*>(T);
    double* ds = reinterpret_cast<double*>(T + b_counts);
    int64_t* dp = reinterpret_cast<int64_t*>(T + b_counts + b_sums);
    int64_t* di = reinterpret_cast<int64_t*>(T + b_counts + b_sums + b_ptr);
    CK(cudaMemcpyAsync(dc, counts, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ds, sums, 8 * (size_t)n * nbands, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dp, indptr, 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, st));
    if (nnz) CK(cudaMemcpyAsync(di, indices, 8 * (size_t)nnz, cudaMemcpyHostToDevice, st));
    {
        PhaseTimer t(c, 0, st);
        launch_graph_init(lv.sb, dc, ds, dp, di, st);
        c->launches += 1;
    }
    CK(cudaGetLastError());
    CK(cudaFreeAsync(tmp, st));
    rc = run_level(c, lv, st);
    if (rc) return rc;
    const int nrec = lv.nlogh[0];
    if (nrec) {
        if (log_survivor) CK(cudaMemcpyAsync(log_survivor, lv.sb.log_a, 4 * (size_t)nrec, cudaMemcpyDeviceToHost, st));
        if (log_absorbed) CK(cudaMemcpyAsync(log_absorbed, lv.sb.log_b, 4 * (size_t)nrec, cudaMemcpyDeviceToHost, st));
        if (log_dissim) CK(cudaMemcpyAsync(log_dissim, lv.sb.log_d, 8 * (size_t)nrec, cudaMemcpyDeviceToHost, st));
        if (log_kind) CK(cudaMemcpyAsync(log_kind, lv.sb.log_k, (size_t)nrec, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    *n_records = nrec;
    *converged_early = lv.convh[0];
    finish_phases(c);
    return RHSEG_OK;
}

// ---- B3 ---------------------------------------------------------------------
struct ScanState {
    std::mutex mu;
    bool init = false;
    int device = 0, nsm = 148;
    cudaStream_t st = nullptr;
    void* buf = nullptr;
    size_t cap = 0;
};
static ScanState g_scan;

static int scan_common(int64_t row_start, int64_t row_stop, int64_t n, int64_t nb, const double* counts,
                       const double* sums, const int64_t* indptr, const int64_t* indices, double* out_d,
                       int64_t* out_j, bool nonadj) {
    if (row_start < 0 || row_stop > n || row_start > row_stop) return fail(RHSEG_E_INVALID, "bad row range");
    if (n > INT32_MAX / 2 || nb < 0) return fail(RHSEG_E_INVALID, "bad shape");
    if (row_start == row_stop) return RHSEG_OK;
    std::lock_guard<std::mutex> lock(g_scan.mu);
    if (!g_scan.init) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(RHSEG_E_CUDA, "no CUDA device");
        CK(cudaGetDevice(&g_scan.device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, g_scan.device));
        if (prop.major != 10) return fail(RHSEG_E_CUDA, "librhseg_b200 is built for sm_100a");
        g_scan.nsm = prop.multiProcessorCount;
        CK(cudaStreamCreateWithFlags(&g_scan.st, cudaStreamNonBlocking));
        g_scan.init = true;
    }
    CK(cudaSetDevice(g_scan.device));
    cudaStream_t st = g_scan.st;
    const int ni = (int)n, nbi = (int)nb, ld = std::max(64, (ni + 63) / 64 * 64), W = ld / 32;
    const int64_t nnz = indptr[n];
    const int rows = (int)(row_stop - row_start);
    const int nsplit = nonadj ? scan_nonadj_splits(ni, rows, g_scan.nsm) : 1;
    const size_t b_c = align256(8 * (size_t)n), b_s = align256(8 * (size_t)n * std::max<int64_t>(nb, 1)),
                 b_p = align256(8 * (size_t)(n + 1)), b_i = align256(8 * (size_t)std::max<int64_t>(nnz, 1)),
                 b_mu = align256(8 * (size_t)ld * std::max<int64_t>(nb, 1)),
                 b_bits = nonadj ? align256(4 * (size_t)ni * W) : 0,
                 b_part = nonadj ? align256(sizeof(RowBest) * (size_t)nsplit * ld) : 0, b_od = align256(8 * (size_t)n),
                 b_oj = align256(8 * (size_t)n);
    const size_t total = b_c + b_s + b_p + b_i + b_mu + b_bits + b_part + b_od + b_oj;
    if (g_scan.cap < total) {
        if (g_scan.buf) CK(cudaFree(g_scan.buf));
        g_scan.buf = nullptr;
        CK(cudaMalloc(&g_scan.buf, total));
        g_scan.cap = total;
    }
    char* P = static_cast<char*>(g_scan.buf);
    double* dc = reinterpret_cast<double*>(P);
    P += b_c;
    double* ds = reinterpret_cast<double*>(P);
    P += b_s;
    int64_t* dp = reinterpret_cast<int64_t*>(P);
    P += b_p;
    int64_t* di = reinterpret_cast<int64_t*>(P);
    P += b_i;
    double* dmu = reinterpret_cast<double*>(P);
    P += b_mu;
    uint32_t* dbits = reinterpret_cast<uint32_t*>(P);
    P += b_bits;
    void* dpart = P;
    P += b_part;
    double* dod = reinterpret_cast<double*>(P);
    P += b_od;
    int64_t* doj = reinterpret_cast<int64_t*>(P);
    CK(cudaMemcpyAsync(dc, counts, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
    if (nb) CK(cudaMemcpyAsync(ds, sums, 8 * (size_t)n * nb, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dp, indptr, 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, st));
    if (nnz) CK(cudaMemcpyAsync(di, indices, 8 * (size_t)nnz, cudaMemcpyHostToDevice, st));
    launch_scan_prep(ni, nbi, ld, W, dc, ds, dp, di, dmu, dbits, nonadj, st);
    if (nonadj)
        launch_scan_nonadjacent((int)row_start, (int)row_stop, ni, ld, nbi, W, nsplit, dc, dmu, dbits, dpart, dod, doj,
                                st);
    else
        launch_scan_adjacent((int)row_start, (int)row_stop, ld, nbi, dc, dmu, dp, di, dod, doj, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_d + row_start, dod + row_start, 8 * (size_t)rows, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out_j + row_start, doj + row_start, 8 * (size_t)rows, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return RHSEG_OK;
}

int rhseg_scan_adjacent(int64_t row_start, int64_t row_stop, int64_t n, int64_t nbands, const double* counts,
                        const double* sums, const int64_t* indptr, const int64_t* indices, double* out_d,
                        int64_t* out_j) {
    return scan_common(row_start, row_stop, n, nbands, counts, sums, indptr, indices, out_d, out_j, false);
}

int rhseg_scan_nonadjacent(int64_t row_start, int64_t row_stop, int64_t col_tile, int64_t n, int64_t nbands,
                           const double* counts, const double* sums, const int64_t* indptr, const int64_t* indices,
                           double* out_d, int64_t* out_j) {
    (void)col_tile;  // result-invariant in the reference (_kernels.py:66-72)
    return scan_common(row_start, row_stop, n, nbands, counts, sums, indptr, indices, out_d, out_j, true);
}

int rhseg_fp64_peak(rhseg_ctx* c, double* ops_per_s) {
    if (!c) return fail(RHSEG_E_INVALID, "ctx is NULL");
    CK(cudaSetDevice(c->device));
    double* out = nullptr;
    CK(cudaMalloc(&out, 1024 * sizeof(double)));
    const int blocks = c->nsm * 8, threads = 256, iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    fp64_probe_kernel<<<blocks, threads, 0, c->stream>>>(out, 100);
    cudaEventRecord(a, c->stream);
    fp64_probe_kernel<<<blocks, threads, 0, c->stream>>>(out, iters);
    cudaEventRecord(b, c->stream);
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    *ops_per_s = (double)blocks * threads * iters * 8.0 * 3.0 / (ms * 1e-3);
    return RHSEG_OK;
}

int rhseg_fp64_fma_peak(rhseg_ctx* c, double* flops_per_s) {
    if (!c) return fail(RHSEG_E_INVALID, "ctx is NULL");
    CK(cudaSetDevice(c->device));
    double* out = nullptr;
    CK(cudaMalloc(&out, 1024 * sizeof(double)));
    const int blocks = c->nsm * 8, threads = 256, iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    fp64_fma_probe_kernel<<<blocks, threads, 0, c->stream>>>(out, 100);
    cudaEventRecord(a, c->stream);
    fp64_fma_probe_kernel<<<blocks, threads, 0, c->stream>>>(out, iters);
    cudaEventRecord(b, c->stream);
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    *flops_per_s = (double)blocks * threads * iters * 8.0 * 2.0 / (ms * 1e-3);
    return RHSEG_OK;
}

}  // extern "C"
