// fp64 CUDA-core throughput on one SM: DFMA issue rate with 8 warps x 8 independent chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_tput dfma_tput.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, int n) {
    double x[8];
    for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-3 + q;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = fma(x[q], 0.9999999, 1e-7);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int q = 0; q < 8; ++q) s += x[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void kf(float *out, long long *cyc, int n) {
    float x[8];
    for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-3f + q;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = fmaf(x[q], 0.9999999f, 1e-7f);
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int q = 0; q < 8; ++q) s += x[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double *out; float *outf; long long *cyc, h;
    cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&outf, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    const int n = 4096;
    for (int th : {32, 128, 256, 512}) {
        k<<<148, th>>>(out, cyc, n);
        k<<<148, th>>>(out, cyc, n);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        std::printf("DFMA threads/SM %4d: %.2f DFMA lane-ops per clock per SM\n", th, (double)th * 8 * n / h);
        kf<<<148, th>>>(outf, cyc, n);
        kf<<<148, th>>>(outf, cyc, n);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        std::printf("FFMA threads/SM %4d: %.2f FFMA lane-ops per clock per SM\n", th, (double)th * 8 * n / h);
    }
    return 0;
}
