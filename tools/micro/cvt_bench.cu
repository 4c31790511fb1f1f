// Microbenchmark: bf16 -> fp64 conversion + DFMA dot throughput on one SM-full grid.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double cvt_f2f(uint32_t w, int hi) {
    return (double)__uint_as_float(hi ? (w & 0xffff0000u) : (w << 16));
}
__device__ __forceinline__ double cvt_int(uint32_t w, int hi) {
    // bf16 -> fp64 bit construction (normal numbers; zero -> 2^-127)
    const uint32_t x = hi ? w : (w << 16);
    const uint32_t h = (((x >> 3) & 0x0FFFE000u) + 0x38000000u) | (x & 0x80000000u);
    return __hiloint2double((int)h, 0);
}
template <int MODE>
__global__ void k(const uint4 *in, const double *kc, double *out, int iters) {
    __shared__ double s[128];
    for (int j = threadIdx.x; j < 128; j += blockDim.x) s[j] = kc[j];
    __syncthreads();
    uint4 v[16];
    for (int q = 0; q < 16; ++q) v[q] = in[(blockIdx.x * blockDim.x + threadIdx.x) * 16 + q];
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const uint32_t wd[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const double x = MODE == 0 ? cvt_f2f(wd[e >> 1], e & 1)
                                 : MODE == 1 ? cvt_int(wd[e >> 1], e & 1)
                                 : ((e & 1) ? cvt_int(wd[e >> 1], 1) : cvt_f2f(wd[e >> 1], 0));
                double &a = (e & 3) == 0 ? acc0 : (e & 3) == 1 ? acc1 : (e & 3) == 2 ? acc2 : acc3;
                a = fma(x, s[q * 8 + e], a);
            }
        }
        v[it & 15].x ^= 0x10001;  // keep loop-variant
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
int main() {
    const int blocks = 148, iters = 200;
    for (int threads = 256; threads <= 256; threads *= 2) {
    uint4 *in; double *kc, *out;
    cudaMalloc(&in, sizeof(uint4) * 16 * blocks * threads);
    cudaMemset(in, 0x3f, sizeof(uint4) * 16 * blocks * threads);
    cudaMalloc(&kc, 128 * 8); cudaMemset(kc, 0, 128 * 8);
    cudaMalloc(&out, 8 * blocks * threads);
    for (int mode = 0; mode < 3; ++mode) {
        for (int warm = 0; warm < 2; ++warm) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, threads>>>(in, kc, out, iters);
            else if (mode == 1) k<1><<<blocks, threads>>>(in, kc, out, iters);
            else k<2><<<blocks, threads>>>(in, kc, out, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double elems = (double)blocks * threads * iters * 128;
            if (warm) printf("threads %d mode %s: %.3f ms, %.2f elem/clk/SM (at 1.965 GHz)\n", threads, mode == 2 ? "mix" : mode ? "int" : "f2f", ms,
                             elems / (ms * 1e-3) / 1.965e9 / 148);
        }
    }
    }
    return 0;
}
