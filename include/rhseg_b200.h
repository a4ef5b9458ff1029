/*
 * rhseg_b200.h -- C ABI of librhseg_b200.so, the sm_100a RHSEG hot path.
 *
 * Plain C: pointers, sizes and status codes; no torch or C++ types cross the
 * boundary. Every entry point returns RHSEG_OK (0) or an RHSEG_E_* status and
 * leaves a thread-local message in rhseg_last_error(). No C++ exception ever
 * crosses the boundary. There is no CPU fallback: without a usable sm_100a
 * device every compute entry point returns RHSEG_E_CUDA.
 *
 * The reference (rhseg, pure Python + numba) has no FFI of its own; the seams it
 * exposes for this path, and which these entry points replace, are:
 *
 *   B3 kernel seam  rhseg/_kernels.py:31-33  scan_adjacent(row_start, row_stop, counts,
 *                   sums, indptr, indices, out_d, out_j)           -> rhseg_scan_adjacent
 *                   rhseg/_kernels.py:62-65  scan_nonadjacent(row_start, row_stop,
 *                   col_tile, ...)                                  -> rhseg_scan_nonadjacent
 *                   (looked up as module attributes by engine._scan, engine.py:213-218)
 *   B2 engine seam  rhseg/engine.py:345-371  hseg_run(graph, params, strategy, ...)
 *                                                                    -> rhseg_hseg_graph
 *   B1 executor     rhseg/recursive.py:179-209 executor.execute(image, params, strategy,
 *                   profile) -> RhsegResult; rhseg_run recursive.py:212-223
 *                                                    -> rhseg_run_device / rhseg_run_host
 *                   + rhseg_result_* accessors for the RhsegResult fields
 *                   (recursive.py:62-92: section_logs, root_initial, root_hierarchy,
 *                   graph, labels, converged_early).
 *
 * Arithmetic contract: fp64, IEEE div/sqrt, no FMA, ascending-band accumulation,
 * strict-< / lexicographic (d, min id, max id) tie-breaks -- merge logs, dissimilarities
 * and labels are bit-identical to the reference CPU path.
 */
#ifndef RHSEG_B200_H
#define RHSEG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RHSEG_ABI_VERSION 1

#define RHSEG_OK 0
#define RHSEG_E_INVALID 1     /* ValueError in the reference (engine.py:37-42, recursive.py:41-47) */
#define RHSEG_E_INDIVISIBLE 2 /* errors.IndivisibleImage (sections.py:61-65) */
#define RHSEG_E_CUDA 3        /* CUDA failure / no sm_100a device */
#define RHSEG_E_TOO_LARGE 4   /* a section's dissimilarity matrix (R0^2 fp64) exceeds device memory */
#define RHSEG_E_STATE 5       /* no result available / wrong call order */
#define RHSEG_E_TOO_MANY_LABELS 6 /* errors.TooManyLabels: label above 65535 in a PGM (hsio.py:85-101) */
#define RHSEG_E_IO 7          /* OSError: an output file cannot be opened or written */

typedef struct rhseg_ctx rhseg_ctx;

/* RhsegParams + HsegParams (recursive.py:30-59, engine.py:29-42). */
typedef struct {
    double spectral_weight;         /* w in [0, 1] */
    int32_t target_regions;         /* >= 1; the root's stopping count */
    int32_t section_target_regions; /* >= 1; every section above the root (0 = target) */
    int32_t levels;                 /* >= 1 recursion levels */
    int32_t connectivity;           /* 4 or 8 */
    int32_t measure;                /* 0 = "sqrt-bsmse" (the reference's only measure, dissim.py:45);
                                       1 = "euclidean", 2 = "sam" (north-star extensions, same fp64
                                       conventions; parity pinned to the oracle only) */
    int32_t cluster;                /* 0 = auto; else CTAs per section in {1,2,4,8,16} */
} rhseg_params;

typedef struct {
    int64_t n_records;              /* merge records over all sections (log order) */
    int64_t spectral_pairs;         /* reference-equivalent sum_steps (R(R-1)/2 - E), w > 0 */
    int32_t n_sections;             /* sections over all levels */
    int32_t levels, edge, bands;
    int32_t root_idspace;           /* region id space of the root section */
    int32_t root_initial_regions;   /* live regions of root_initial */
    int32_t root_regions;           /* live regions after the root HSEG */
    int32_t converged_early;        /* any section converged early (recursive.py:208) */
    float device_ms;                /* device time of the last run (CUDA events) */
    float pad_;
} rhseg_result_info;

int rhseg_abi_version(void);
const char *rhseg_last_error(void);

int rhseg_ctx_create(int device, rhseg_ctx **out);
int rhseg_ctx_destroy(rhseg_ctx *ctx);

/* ---- B1: full RHSEG (SequentialExecutor.execute, recursive.py:173-209) ----------- */
/* d_samples: DEVICE pointer, float32 BSQ [bands][edge][edge] (image.py:12-52).
 * stream: a cudaStream_t (NULL = legacy default). Results stay in the context. */
int rhseg_run_device(rhseg_ctx *ctx, const float *d_samples, int32_t edge, int32_t bands,
                     const rhseg_params *params, void *stream);
/* Same from a HOST cube (pinned or pageable): H2D, run, D2H of the merge log (SoA,
 * capacity edge*edge records each) and dense labels (edge*edge). Any output
 * pointer may be NULL. */
int rhseg_run_host(rhseg_ctx *ctx, const float *h_samples, int32_t edge, int32_t bands,
                   const rhseg_params *params, void *stream, int32_t *log_survivor,
                   int32_t *log_absorbed, double *log_dissim, uint8_t *log_kind,
                   int32_t *labels, rhseg_result_info *info);

/* ---- B1 sharded: subtree blocks + reassembly --------------------- */
/* Levels L..top_level over the block [r0, r0+nr) x [c0, c0+nc) of the level-top
 * section grid (2^(top-1) sections a side). top_level = 1, block 1x1 is exactly
 * rhseg_run_device. Each rank of a multi-GPU run owns one block of level-top
 * subtrees (the quadrant recursion of recursive.py:145-170 below top is local to
 * it). d_samples is the full cube on this device. */
int rhseg_run_subtrees(rhseg_ctx *ctx, const float *d_samples, int32_t edge, int32_t bands,
                       const rhseg_params *params, int32_t top_level, int32_t r0, int32_t c0,
                       int32_t nr, int32_t nc, void *stream);
/* Top level of the last run: sections, their region capacity (multiple of 32),
 * section edge; R0[nsec] initial regions and nlog[nsec] merges (either may be NULL). */
int rhseg_top_info(rhseg_ctx *ctx, int32_t *nsec, int32_t *rp, int32_t *sec_edge, int32_t *R0,
                   int32_t *nlog);
/* Bytes of one packed section state with capacity rp (stitch input, sections.py:103-163):
 * count u32[rp] | sums f64[rp][bands] | adjacency u32[rp][rp/32] | assignment i32[e*e]. */
int rhseg_pack_bytes(int32_t rp, int32_t bands, int32_t sec_edge, int64_t *bytes);
/* Pack the top level's sections (row-major within the block) into a DEVICE buffer
 * of nsec * rhseg_pack_bytes(rp, ...) bytes, rp >= the level's own capacity. */
int rhseg_export_top(rhseg_ctx *ctx, int32_t rp, void *d_pack, void *stream);
/* Rank 0 after the gather: the packed states of ALL 4^(top-1) level-top sections
 * (row-major over the whole grid) -> stitch + HSEG of levels top-1..1 + root labels.
 * R0/nlog: host arrays of 4^(top-1) entries. The result covers levels < top_level;
 * the other levels' logs come from the ranks (rhseg_result_log_device). */
int rhseg_run_upper(rhseg_ctx *ctx, const void *d_pack, int32_t top_level, int32_t rp,
                    const int32_t *R0, const int32_t *nlog, int32_t edge, int32_t bands,
                    const rhseg_params *params, void *stream);

int rhseg_result_info_get(rhseg_ctx *ctx, rhseg_result_info *info);
/* Sections in log order (level L..1, row-major, recursive.py:95-104): n_sections entries. */
int rhseg_result_sections(rhseg_ctx *ctx, int32_t *level, int32_t *row, int32_t *col,
                          int64_t *offset, int64_t *count);
/* Flat merge log, n_records entries each (host buffers). */
int rhseg_result_log(rhseg_ctx *ctx, int32_t *survivor, int32_t *absorbed, double *dissim,
                     uint8_t *kind);
/* Same into DEVICE buffers of n_records entries, stream-ordered (for NCCL gathers). */
int rhseg_result_log_device(rhseg_ctx *ctx, int32_t *survivor, int32_t *absorbed, double *dissim,
                            uint8_t *kind, void *stream);
/* labels: dense, first row-major occurrence (graph.py:267-281); assignment: root ids. */
int rhseg_result_labels(rhseg_ctx *ctx, int32_t *labels, int32_t *assignment);
/* Root graph state, which = 0: root_initial (pre-root-HSEG, recursive.py:166-167),
 * which = 1: final. counts[idspace] (0 = dead), sums[idspace][bands] f64,
 * adjacency bitset[idspace][ceil(idspace/32)] u32, assignment[edge*edge]. */
int rhseg_result_root(rhseg_ctx *ctx, int32_t which, int64_t *counts, double *sums,
                      uint32_t *adjacency, int32_t *assignment);

/* ---- B2: hseg_run on one region graph (engine.py:345-371) ---------------------- */
/* Dense ascending-id graph as built by engine.snapshot (engine.py:167-191): counts[n]
 * f64, sums[n][nbands] f64 row-major, CSR indptr[n+1]/indices int64 (host). Writes up
 * to n-1 records; *n_records receives the count. */
int rhseg_hseg_graph(rhseg_ctx *ctx, int64_t n, int64_t nbands, const double *counts,
                     const double *sums, const int64_t *indptr, const int64_t *indices,
                     double spectral_weight, int64_t target_regions, int32_t cluster,
                     int32_t measure, int32_t *log_survivor, int32_t *log_absorbed, double *log_dissim,
                     uint8_t *log_kind, int64_t *n_records, int32_t *converged_early);

/* ---- B3: per-row best-partner tables (_kernels.py:31-115), HOST buffers --------- */
/* Rows [row_start, row_stop) of out_d/out_j are written, nothing else. n = rows of
 * counts/sums; nbands = columns of sums. Reentrant (serialised internally). */
int rhseg_scan_adjacent(int64_t row_start, int64_t row_stop, int64_t n, int64_t nbands,
                        const double *counts, const double *sums, const int64_t *indptr,
                        const int64_t *indices, double *out_d, int64_t *out_j);
int rhseg_scan_nonadjacent(int64_t row_start, int64_t row_stop, int64_t col_tile, int64_t n,
                           int64_t nbands, const double *counts, const double *sums,
                           const int64_t *indptr, const int64_t *indices, double *out_d,
                           int64_t *out_j);

/* ---- output files at scale (cli.py:386-390, hsio.py:85-101, manifest.py:22-27) ---- */
/* Python repr of a double (shortest round trip, repr layout; json.dumps spelling of
 * inf/nan) into buf (cap >= 32). Host-only, no device needed. */
int rhseg_format_float(double x, char *buf, int32_t cap);
/* sha256 of n bytes as 64 hex chars + NUL (hex65). Host-only. */
int rhseg_sha256_hex(const void *data, int64_t n, char *hex65);
/* Labels PGM + merge-log JSONL byte-identical to the reference CLI's files, from
 * host arrays (rhseg_result_sections / _log / _labels); content_hash_hex65 =
 * sha256(pgm || jsonl) = the reference manifest's content_hash. Host-only. */
int rhseg_write_outputs_host(const char *pgm_path, const char *jsonl_path, int32_t width, int32_t height,
                             const int32_t *labels, int32_t n_sections, const int32_t *sec_level,
                             const int32_t *sec_row, const int32_t *sec_col, const int64_t *sec_count,
                             const int32_t *survivor, const int32_t *absorbed, const double *dissim,
                             const uint8_t *kind, char *content_hash_hex65, int64_t *jsonl_bytes);

/* ---- measurement helpers ------------------------------------------------------ */
/* Per-kernel device time of the last run: [0] leaf/graph init, [1] all-pairs D init,
 * [2] merge loops, [3] stitch+resolve+labels (ms, CUDA events on the run stream). */
int rhseg_result_phase_ms(rhseg_ctx *ctx, float *ms4);
/* Kernels this library launched for the last run_* call, plus result copies
 * (rhseg_result_log) made since (the bench's gpu_launches evidence). */
int rhseg_result_launches(rhseg_ctx *ctx, int64_t *n);
/* Rows the merge loops of the last run rescanned from D (level <= 0: all levels) --
 * the traffic model of the loop's roofline (bench.py). */
int rhseg_result_rescans(rhseg_ctx *ctx, int32_t level, int64_t *n);
/* Which merge loop ran on one level of the last run (the roofline model follows it):
 * RHSEG_LOOP_ADJACENT (w = 0), RHSEG_LOOP_STREAM (mean-stream loop: SAM, thread-block
 * clusters, RHSEG_APO=0), RHSEG_LOOP_APO (the APO loop, hseg_kernels.cu), RHSEG_LOOP_APO_RECUT
 * (apo_loop.cu, RHSEG_APO_V2=1); plus sections, padded capacity, CTAs per section, merges.
 * Any output pointer may be NULL. */
#define RHSEG_LOOP_ADJACENT 0
#define RHSEG_LOOP_STREAM 1
#define RHSEG_LOOP_APO 2
#define RHSEG_LOOP_APO_RECUT 3
#define RHSEG_LOOP_GRID 4 /* grid_loop.cu: sections above a cluster's capacity (cluster = CTAs per section) */
int rhseg_result_level_info(rhseg_ctx *ctx, int32_t level, int32_t *nsec, int32_t *rp, int32_t *cluster,
                            int32_t *loop_variant, int64_t *merges);
/* FP64 DADD/DMUL issue-rate probe: returns achieved fp64 ops/s of a pure
 * sub/mul/add loop over the whole GPU (roofline denominator). */
int rhseg_fp64_peak(rhseg_ctx *ctx, double *ops_per_s);
/* FP64 fused multiply-add probe: achieved fp64 flops/s (2 per DFMA) of a pure DFMA
 * loop over the whole GPU -- the FP64 flop roofline of the all-pairs D init. */
int rhseg_fp64_fma_peak(rhseg_ctx *ctx, double *flops_per_s);

#ifdef __cplusplus
}
#endif
#endif
