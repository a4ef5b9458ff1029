// Microbenchmark: latency of one exact ascending-band fp64 pair evaluation by one warp
// (the APO loop's exact re-evaluation), three formulations. Build + run on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/es tools/micro/exact_sum.cu && /tmp/es
#include <cstdio>
#include <cuda_runtime.h>

__device__ __noinline__ double v_shfl(const double* mi, const double* mj, int B, int lane) {
    double s = 0.0;
    for (int k0 = 0; k0 < B; k0 += 256) {
        double term[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + 32 * u + lane;
            const double vi = k < B ? mi[k] : 0.0, vj = k < B ? __ldcg(mj + k) : 0.0;
            const double t = __dsub_rn(vi, vj);
            term[u] = __dmul_rn(t, t);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int kn = min(32, B - (k0 + 32 * u));
            if (kn <= 0) break;
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
                const double tk = __shfl_sync(0xffffffffu, term[u], kk);
                if (kk < kn) s = __dadd_rn(s, tk);
            }
        }
    }
    return s;
}
__device__ __noinline__ double v_smem(const double* mi, const double* mj, int B, int lane, double* scr) {
    for (int k = lane; k < B; k += 32) {
        const double t = __dsub_rn(mi[k], __ldcg(mj + k));
        scr[k] = __dmul_rn(t, t);
    }
    __syncwarp();
    double s = 0.0;
    if (lane == 0) {
        int k = 0;
        for (; k + 8 <= B; k += 8) {
            double x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = scr[k + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) s = __dadd_rn(s, x[u]);
        }
        for (; k < B; ++k) s = __dadd_rn(s, scr[k]);
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    __syncwarp();
    return s;
}
__device__ __noinline__ double v_chain(int B, double x) {  // pure dependent DADD chain
    double s = 0.0;
    for (int k = 0; k < B; ++k) s = __dadd_rn(s, x * k);
    return s;
}
__global__ void bench(const double* m, int B, long long* out, double* sink) {
    __shared__ double scr[8][256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double* mi = m + (size_t)(blockIdx.x * 64 + w) * B;
    const double* mj = m + (size_t)(blockIdx.x * 64 + 32 + w) * B;
    double acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < 4; ++r) acc += v_shfl(mi + r, mj, B, lane);
    long long t1 = clock64();
    for (int r = 0; r < 4; ++r) acc += v_smem(mi + r, mj, B, lane, scr[w]);
    long long t2 = clock64();
    acc += v_chain(B, acc);
    long long t3 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = (t1 - t0) / 4; out[1] = (t2 - t1) / 4; out[2] = t3 - t2; }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    const int B = 224, nb = 296;
    double* m; long long* out; double* sink;
    cudaMalloc(&m, (size_t)nb * 64 * B * 8 + 4096);
    cudaMemset(m, 0, (size_t)nb * 64 * B * 8 + 4096);
    cudaMallocManaged(&out, 64);
    cudaMalloc(&sink, nb * 256 * 8);
    for (int blocks : {1, nb}) {
        for (int it = 0; it < 3; ++it) bench<<<blocks, 256>>>(m, B, out, sink);
        cudaDeviceSynchronize();
        printf("blocks %d: shfl %lld cyc, smem %lld cyc, %d-DADD chain %lld cyc\n", blocks, out[0], out[1], B, out[2]);
    }
    return 0;
}
