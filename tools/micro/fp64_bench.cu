// fp64_bench.cu -- microbenchmarks for the blocked-selection GEMM design choice:
// fp64 FMA throughput on B200 as (a) pure DFMA, (b) DFMA fed by broadcast LDS.128 (1 key/thread),
// (c) the same with 2 keys/thread, (d) DMMA m8n8k4 tensor-core fp64 with register operands.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_bench fp64_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void pure_dfma(double *out, double s) {
    double acc[16];
#pragma unroll
    for (int x = 0; x < 16; ++x) acc[x] = threadIdx.x * 1e-3 + x;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int x = 0; x < 16; ++x) acc[x] = fma(acc[x], s, 1e-9);
    }
    double t = 0;
#pragma unroll
    for (int x = 0; x < 16; ++x) t += acc[x];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// 1 key per thread: per row 1 LDS.64 (own column) + 8 LDS.128 broadcast + 16 DFMA
template <int KPT>
__global__ void lds_dfma(double *out, int rows) {
    extern __shared__ double sm[];
    double *ring = sm;                   // [64][256*KPT]
    double *fs = ring + 64 * 256 * KPT;  // [64][16]
    for (int i = threadIdx.x; i < 64 * 256 * KPT; i += blockDim.x) ring[i] = i * 1e-6;
    for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) fs[i] = i * 1e-5;
    __syncthreads();
    double acc[KPT][16];
#pragma unroll
    for (int k = 0; k < KPT; ++k)
#pragma unroll
        for (int x = 0; x < 16; ++x) acc[k][x] = 0;
    for (int it = 0; it < rows; ++it) {
        const int r = it & 63;
        double xv[KPT];
#pragma unroll
        for (int k = 0; k < KPT; ++k) xv[k] = ring[r * 256 * KPT + k * 256 + threadIdx.x];
        const double2 *fr = reinterpret_cast<const double2 *>(fs + r * 16);
#pragma unroll
        for (int x2 = 0; x2 < 8; ++x2) {
            const double2 f = fr[x2];
#pragma unroll
            for (int k = 0; k < KPT; ++k) {
                acc[k][2 * x2] = fma(xv[k], f.x, acc[k][2 * x2]);
                acc[k][2 * x2 + 1] = fma(xv[k], f.y, acc[k][2 * x2 + 1]);
            }
        }
    }
    double t = 0;
#pragma unroll
    for (int k = 0; k < KPT; ++k)
#pragma unroll
        for (int x = 0; x < 16; ++x) t += acc[k][x];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void dmma_bench(double *out, double s) {
    double a = threadIdx.x * 1e-3 + s, b = threadIdx.x * 2e-3;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1])
                         : "d"(a), "d"(b));
    }
    double t = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += c[k][0] + c[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *out;
    cudaMalloc(&out, sizeof(double) * sms * 4 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    auto report = [&](const char *name, double fmas) {
        const double per_clk_sm = fmas / (ms * 1e-3) / sms / (clk * 1e3);
        std::printf("%-28s %8.3f ms  %7.1f TFLOP/s  %6.1f FMA/clk/SM (clk %d MHz nominal)\n", name, ms,
                    2 * fmas / (ms * 1e-3) / 1e12, per_clk_sm, clk / 1000);
    };
    for (int warps : {8, 16}) {
        const int th = warps * 32;
        pure_dfma<<<sms, th>>>(out, 1.0000001);
        cudaEventRecord(e0);
        pure_dfma<<<sms, th>>>(out, 1.0000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        char nm[64];
        std::snprintf(nm, 64, "pure DFMA, %d warps", warps);
        report(nm, (double)sms * th * kIters * 16);
    }
    const int rows = 8192;
    {
        const size_t smem = (64 * 256 * 1 + 64 * 16) * 8;
        cudaFuncSetAttribute(lds_dfma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        lds_dfma<1><<<sms, 256, smem>>>(out, rows);
        cudaEventRecord(e0);
        lds_dfma<1><<<sms, 256, smem>>>(out, rows);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        report("LDS.128 bcast + DFMA, 1 key", (double)sms * 256 * rows * 16);
    }
    {
        const size_t smem = (64 * 256 * 2 + 64 * 16) * 8;
        cudaFuncSetAttribute(lds_dfma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        lds_dfma<2><<<sms, 256, smem>>>(out, rows);
        cudaEventRecord(e0);
        lds_dfma<2><<<sms, 256, smem>>>(out, rows);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        report("LDS.128 bcast + DFMA, 2 keys", (double)sms * 256 * rows * 32);
    }
    for (int warps : {4, 8, 16}) {
        const int th = warps * 32;
        dmma_bench<<<sms, th>>>(out, 1.0);
        cudaEventRecord(e0);
        dmma_bench<<<sms, th>>>(out, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        char nm[64];
        std::snprintf(nm, 64, "DMMA m8n8k4, %d warps", warps);
        report(nm, (double)sms * warps * (kIters / 4) * 8 * 256);
    }
    cudaError_t e = cudaGetLastError();
    std::printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
