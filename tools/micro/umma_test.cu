// Probe: one 128 x N x K bf16 GEMM on tcgen05 (K-major SW128 smem operands, fp32 TMEM accum).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../../paper_2602_10056_b200/csrc/umma.cuh"
using namespace wc;
template <int N, int K>
__global__ void __launch_bounds__(128) gemm_probe(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *C) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *sa = sm, *sb = sm + 128 * K * 2;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int e = tid; e < 128 * K; e += 128) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<__nv_bfloat16 *>(sa + umma::sw128_offset(r, k, 128)) = A[r * K + k];
    }
    for (int e = tid; e < N * K; e += 128) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<__nv_bfloat16 *>(sb + umma::sw128_offset(r, k, N)) = B[r * K + k];
    }
    if (w == 0) umma::tmem_alloc(&tbase, 256);
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t t0 = tbase;
    if (tid == 0) {
        umma::gemm_128xNxK(t0, smem_u32(sa), smem_u32(sb), N, K, false);
        umma::commit(&bar);
    }
    mbar_wait(&bar, 0);
    umma::fence_after_sync();
    for (int c0 = 0; c0 < N; c0 += 32) {
        float v[32];
        umma::ld32(t0 + ((uint32_t)(w * 32) << 16) + c0, v);
        for (int i = 0; i < 32; ++i) C[(w * 32 + lane) * N + c0 + i] = v[i];
    }
    umma::fence_before_sync();
    __syncthreads();
    if (w == 0) umma::tmem_dealloc(t0, 256);
}
template <int N, int K> int run() {
    std::vector<__nv_bfloat16> hA(128 * K), hB(N * K);
    std::vector<float> fA(128 * K), fB(N * K);
    srand(1);
    for (int i = 0; i < 128 * K; ++i) { float x = (rand() % 2001 - 1000) / 500.f; hA[i] = __float2bfloat16(x); fA[i] = __bfloat162float(hA[i]); }
    for (int i = 0; i < N * K; ++i) { float x = (rand() % 2001 - 1000) / 500.f; hB[i] = __float2bfloat16(x); fB[i] = __bfloat162float(hB[i]); }
    __nv_bfloat16 *dA, *dB; float *dC;
    cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dC, 128 * N * 4);
    cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
    const int smem = (128 + N) * K * 2 + 1024;
    cudaFuncSetAttribute(gemm_probe<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    gemm_probe<N, K><<<1, 128, smem>>>(dA, dB, dC);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e)); return 1; }
    std::vector<float> hC(128 * N);
    cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
        double ref = 0; for (int k = 0; k < K; ++k) ref += (double)fA[m * K + k] * fB[n * K + k];
        maxerr = fmax(maxerr, fabs(ref - hC[m * N + n])); maxref = fmax(maxref, fabs(ref));
    }
    printf("N=%d K=%d: max abs err %.3e (max |ref| %.3e) %s\n", N, K, maxerr, maxref, maxerr < 1e-3 * maxref ? "OK" : "MISMATCH");
    return 0;
}
int main() { run<256, 128>(); run<128, 64>(); run<64, 128>(); run<32, 64>(); run<16, 128>(); return 0; }
