// Latency of the dependent fp64 chains that dominate the blocked selection's serial phases
// (DADD, DFMA, DSETP+select, shfl+DADD, LDS+DADD, MUFU rsqrt + Newton), single warp, clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_bench lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double *out, long long *cyc, double x0, int n) {
    __shared__ double sm[64];
    const int lane = threadIdx.x;
    sm[lane] = x0 + lane;
    sm[lane + 32] = x0 - lane;
    __syncwarp();
    double x = x0 + lane * 1e-3;
    long long t0, t1;
    // 1: dependent DADD
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + 1.0000001;
    t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    // 2: dependent DFMA
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 0.9999999, 1e-7);
    t1 = clock64();
    if (lane == 0) cyc[1] = t1 - t0;
    // 3: shfl + DADD (one step of a warp scan)
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + __shfl_xor_sync(0xffffffffu, x, 1);
    t1 = clock64();
    if (lane == 0) cyc[2] = t1 - t0;
    // 4: LDS + DADD (dependent address)
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const double y = sm[idx];
        x = x + y;
        idx = ((int)x & 31) + (i & 1) * 32;
    }
    t1 = clock64();
    if (lane == 0) cyc[3] = t1 - t0;
    // 5: DSETP + select chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = (x > 0.5) ? x - 0.25 : x + 0.3;
    t1 = clock64();
    if (lane == 0) cyc[4] = t1 - t0;
    // 6: FP32 FFMA chain for reference
    float f = (float)x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) f = fmaf(f, 0.9999999f, 1e-7f);
    t1 = clock64();
    if (lane == 0) cyc[5] = t1 - t0;
    // 7: DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x * 1.0000001;
    t1 = clock64();
    if (lane == 0) cyc[6] = t1 - t0;
    // 8: F2F.F64.F32 conversion chain (float -> double -> float)
    t0 = clock64();
    for (int i = 0; i < n; ++i) f = (float)((double)f * 1.0000001);
    t1 = clock64();
    if (lane == 0) cyc[7] = t1 - t0;
    out[lane] = x + f;
}

int main() {
    double *out;
    long long *cyc, h[8];
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMalloc(&cyc, 8 * sizeof(long long));
    const int n = 4096;
    lat<<<1, 32>>>(out, cyc, 0.3, n);
    lat<<<1, 32>>>(out, cyc, 0.3, n);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const char *names[] = {"DADD", "DFMA", "SHFL+DADD", "LDS+DADD+idx", "DSETP+sel+DADD", "FFMA(fp32)", "DMUL", "F2F64+DMUL+F2F32"};
    for (int k = 0; k < 8; ++k) std::printf("%-18s %.1f cycles/iter\n", names[k], (double)h[k] / n);
    return 0;
}
