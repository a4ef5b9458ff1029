// scan_kernels.cu -- from-scratch per-row best-partner tables on a CSR snapshot:
// the device versions of the reference's two numba kernels, with their exact
// signature semantics (rows [row_start, row_stop) written, nothing else):
//   _kernels.py:31-59  scan_adjacent    -> scan_adjacent_kernel (warp per row, lane per neighbour)
//   _kernels.py:62-115 scan_nonadjacent -> scan_nonadj_kernel   (64x64 fp64 pair tiles, 4x4
//                                          register blocks, per-row lexicographic (d, j) min,
//                                          column splits combined in ascending order)
// Means are divided once (mu = sums / count, IEEE) -- bit-identical to the
// reference dividing inside the inner loop (_kernels.py:43, 52).
#include <cuda_runtime.h>

#include "rhseg_device.cuh"

namespace rhseg {

__global__ void scan_means_kernel(int n, int nb, int ld, const double* __restrict__ counts,
                                  const double* __restrict__ sums, double* __restrict__ mu) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * nb) return;
    const int i = idx / nb, k = idx - i * nb;
    mu[(size_t)k * ld + i] = __ddiv_rn(sums[idx], counts[i]);
}

__global__ void scan_bitset_kernel(int n, int W, const int64_t* __restrict__ indptr,
                                   const int64_t* __restrict__ indices, uint32_t* __restrict__ bits) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
        const int j = (int)indices[p];
        bits[(size_t)i * W + (j >> 5)] |= 1u << (j & 31);
    }
}

// One warp per row; each lane owns one CSR neighbour at a time.
__global__ void scan_adjacent_kernel(int row_start, int row_stop, int ld, int nb,
                                     const double* __restrict__ counts, const double* __restrict__ mu,
                                     const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices,
                                     double* __restrict__ out_d, int64_t* __restrict__ out_j) {
    const int warps = blockDim.x >> 5;
    const int i = row_start + blockIdx.x * warps + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= row_stop) return;
    const double ni = counts[i];
    RowBest best = rb_none();
    for (int64_t p = indptr[i] + lane; p < indptr[i + 1]; p += 32) {
        const int j = (int)indices[p];
        double s = 0.0;
        for (int k = 0; k < nb; ++k) s = bsmse_step(s, mu[(size_t)k * ld + i], mu[(size_t)k * ld + j]);
        rb_offer(best, bsmse_finish(ni, counts[j], s), j);
    }
    best = warp_min_rb(best);
    if (lane == 0) {
        out_d[i] = best.d;
        out_j[i] = best.j == kNoJ ? -1 : best.j;
    }
}

constexpr int kST = 64;   // pair tile
constexpr int kSKB = 16;  // bands per smem stage

// grid (row tiles covering [row_start,row_stop), column splits). Each CTA folds its
// column range into per-row (d, j) minima -> part[split][row].
__global__ void __launch_bounds__(256)
scan_nonadj_kernel(int row_start, int row_stop, int n, int ld, int nb, int W, int cols_per_split,
                   const double* __restrict__ counts, const double* __restrict__ mu,
                   const uint32_t* __restrict__ bits, RowBest* __restrict__ part) {
    const int i0 = row_start + blockIdx.x * kST;
    const int c_begin = blockIdx.y * cols_per_split;
    const int c_end = min(n, c_begin + cols_per_split);
    __shared__ double sA[kSKB][kST];
    __shared__ double sB[kSKB][kST];
    __shared__ RowBest red[16][kST + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    RowBest best[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) best[p] = rb_none();
    for (int j0 = c_begin; j0 < c_end; j0 += kST) {
        double acc[4][4];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
        for (int k0 = 0; k0 < nb; k0 += kSKB) {
            const int kn = min(kSKB, nb - k0);
            for (int e = threadIdx.x; e < kSKB * kST; e += 256) {
                const int kk = e / kST, r = e % kST;
                const bool in = kk < kn;
                sA[kk][r] = (in && i0 + r < n) ? mu[(size_t)(k0 + kk) * ld + i0 + r] : 0.0;
                sB[kk][r] = (in && j0 + r < n) ? mu[(size_t)(k0 + kk) * ld + j0 + r] : 0.0;
            }
            __syncthreads();
            for (int kk = 0; kk < kn; ++kk) {
                double a[4], b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a[q] = sA[kk][ty + 16 * q];
                    b[q] = sB[kk][tx + 16 * q];
                }
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[p][q] = bsmse_step(acc[p][q], a[p], b[q]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int i = i0 + ty + 16 * p;
            if (i >= row_stop) continue;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = j0 + tx + 16 * q;
                if (j >= c_end || j == i) continue;
                if ((bits[(size_t)i * W + (j >> 5)] >> (j & 31)) & 1u) continue;
                rb_offer(best[p], bsmse_finish(counts[i], counts[j], acc[p][q]), j);
            }
        }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) red[tx][ty + 16 * p] = best[p];
    __syncthreads();
    if (threadIdx.x < kST) {
        const int r = threadIdx.x;
        RowBest b = red[0][r];
        for (int t = 1; t < 16; ++t) {
            const RowBest c = red[t][r];
            if (c.d < b.d || (c.d == b.d && c.j < b.j)) b = c;
        }
        const int i = i0 + r;
        if (i < row_stop) part[(size_t)blockIdx.y * ld + i] = b;
    }
}

__global__ void scan_combine_kernel(int row_start, int row_stop, int ld, int nsplit, const RowBest* part,
                                    double* out_d, int64_t* out_j) {
    const int i = row_start + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= row_stop) return;
    RowBest b = rb_none();
    for (int s = 0; s < nsplit; ++s) {
        const RowBest c = part[(size_t)s * ld + i];
        if (c.d < b.d || (c.d == b.d && c.j < b.j)) b = c;
    }
    out_d[i] = b.d;
    out_j[i] = b.j == kNoJ ? -1 : b.j;
}

// Host launchers (device buffers already populated by the caller).
void launch_scan_prep(int n, int nb, int ld, int W, const double* counts, const double* sums,
                      const int64_t* indptr, const int64_t* indices, double* mu, uint32_t* bits,
                      bool need_bits, cudaStream_t st) {
    if (n == 0) return;
    if (nb > 0) scan_means_kernel<<<(n * nb + 255) / 256, 256, 0, st>>>(n, nb, ld, counts, sums, mu);
    if (need_bits) {
        cudaMemsetAsync(bits, 0, sizeof(uint32_t) * (size_t)n * W, st);
        scan_bitset_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, W, indptr, indices, bits);
    }
}

void launch_scan_adjacent(int row_start, int row_stop, int ld, int nb, const double* counts, const double* mu,
                          const int64_t* indptr, const int64_t* indices, double* out_d, int64_t* out_j,
                          cudaStream_t st) {
    const int rows = row_stop - row_start;
    if (rows <= 0) return;
    scan_adjacent_kernel<<<(rows + 7) / 8, 256, 0, st>>>(row_start, row_stop, ld, nb, counts, mu, indptr, indices,
                                                         out_d, out_j);
}

int scan_nonadj_splits(int n, int rows, int nsm) {
    const int rt = (rows + kST - 1) / kST;
    int s = (2 * nsm + rt - 1) / rt;
    const int max_s = (n + kST - 1) / kST;
    if (s > max_s) s = max_s;
    return s < 1 ? 1 : s;
}

void launch_scan_nonadjacent(int row_start, int row_stop, int n, int ld, int nb, int W, int nsplit,
                             const double* counts, const double* mu, const uint32_t* bits, void* part,
                             double* out_d, int64_t* out_j, cudaStream_t st) {
    const int rows = row_stop - row_start;
    if (rows <= 0) return;
    int cps = (n + nsplit - 1) / nsplit;
    cps = (cps + kST - 1) / kST * kST;
    const int ns = (n + cps - 1) / cps;
    dim3 grid((rows + kST - 1) / kST, ns);
    scan_nonadj_kernel<<<grid, 256, 0, st>>>(row_start, row_stop, n, ld, nb, W, cps, counts, mu, bits,
                                                  static_cast<RowBest*>(part));
    scan_combine_kernel<<<(rows + 255) / 256, 256, 0, st>>>(row_start, row_stop, ld, ns,
                                                            static_cast<const RowBest*>(part), out_d, out_j);
}

}  // namespace rhseg
