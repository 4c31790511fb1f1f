// weights.cu -- A3 + A4 of the hot path: optimal Nystrom reweighting.
//   Y~ = h~(K_S, K) [V, 1_n]            (P:156-158 weights; Alg 2 "Compress values")
//   X  = h~(K_S,K_S)^{-1} Y~ = L^{-T} (L^{-1} Y~),   L from the selection (Z8)
// The e^{-mstar} scale of h~ cancels in X (h~(K_S,K_S)^{-1} h~(K_S,K) = W), so X = [V_S, w].
//
// A3 here is the CUDA-core exp-GEMM: per (n-split, 32-row coreset tile, unit) a CTA forms
// P = exp(g <kc_s, kc_l> - mstar) tile by tile in shared memory (fp32 dot of centred keys)
// and accumulates P [V, 1] in fp32 registers; the split partials are summed in fixed order
// in fp64 by the solve kernel.  A4 is a warp-per-RHS-column fp64 triangular solve.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace wc {

namespace {

constexpr int kWT = 256;  // threads
constexpr int kTA = 32;   // coreset rows per CTA
constexpr int kTL = 32;   // keys per smem tile

template <typename T, int D>
__global__ void __launch_bounds__(kWT) weights_partial_kernel(const T *__restrict__ K, const T *__restrict__ V,
                                                              const int32_t *__restrict__ S,
                                                              const int32_t *__restrict__ r_eff,
                                                              const double *__restrict__ stats, int64_t n,
                                                              int r, int splits, float *__restrict__ Ypart) {
    constexpr int DC = D + 1;
    constexpr int CPT = (DC + 7) / 8;  // accumulator columns per thread
    extern __shared__ double wsm[];
    double *kb = wsm;                                              // [D]
    float (*kcS)[D + 1] = reinterpret_cast<float (*)[D + 1]>(kb + D);  // [kTA][D+1]
    float (*kcL)[D + 1] = kcS + kTA;                                // [kTL][D+1]
    float (*vL)[D + 1] = kcL + kTL;                                 // [kTL][D+1]
    float (*Pm)[kTL + 1] = reinterpret_cast<float (*)[kTL + 1]>(&vL[kTL][0]);  // [kTA][kTL+1]

    const int split = blockIdx.x, a0 = blockIdx.y * kTA, u = blockIdx.z;
    const int re = r_eff[u];
    if (a0 >= re) return;  // whole tile beyond r_eff: partials unused by the solve
    const int tid = threadIdx.x;
    const double *st = stats + (int64_t)u * (8 + D);
    const float g = (float)st[1], mstar = (float)st[2];
    for (int j = tid; j < D; j += kWT) kb[j] = st[8 + j];
    __syncthreads();
    const T *Ku = K + (int64_t)u * n * D;
    const T *Vu = V + (int64_t)u * n * D;
    for (int e = tid; e < kTA * D; e += kWT) {
        const int a = e / D, j = e % D;
        float v = 0.f;
        if (a0 + a < re) {
            const int s = S[(int64_t)u * r + a0 + a];
            v = (float)(to_f64(Ku[(int64_t)s * D + j]) - kb[j]);
        }
        kcS[a][j] = v;
    }
    const int64_t rows = ceil_div(n, splits);
    const int64_t lo = (int64_t)split * rows, hi = std::min<int64_t>(n, lo + rows);

    const int ta = tid >> 3, cg = tid & 7;  // accumulator ownership: row ta, columns cg + 8k
    float acc[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) acc[k] = 0.f;

    for (int64_t l0 = lo; l0 < hi; l0 += kTL) {
        __syncthreads();
        for (int e = tid; e < kTL * D; e += kWT) {
            const int l = e / D, j = e % D;
            const int64_t gl = l0 + l;
            float kv = 0.f, vv = 0.f;
            if (gl < hi) {
                kv = (float)(to_f64(Ku[gl * D + j]) - kb[j]);
                vv = to_f32(Vu[gl * D + j]);
            }
            kcL[l][j] = kv;
            vL[l][j] = vv;
        }
        __syncthreads();
        // P tile: 32 x 32, 4 entries per thread
#pragma unroll
        for (int q = 0; q < (kTA * kTL) / kWT; ++q) {
            const int e = tid + q * kWT;
            const int a = e / kTL, l = e % kTL;
            float dot = 0.f;
#pragma unroll 16
            for (int j = 0; j < D; ++j) dot = fmaf(kcS[a][j], kcL[l][j], dot);
            const bool ok = (a0 + a < re) && (l0 + l < hi);
            Pm[a][l] = ok ? expf(fmaf(g, dot, -mstar)) : 0.f;
        }
        __syncthreads();
#pragma unroll 4
        for (int l = 0; l < kTL; ++l) {
            const float pv = Pm[ta][l];
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int cidx = cg + 8 * k;
                if (cidx < D) acc[k] = fmaf(pv, vL[l][cidx], acc[k]);
                else if (cidx == D) acc[k] += pv;
            }
        }
    }
    float *out = Ypart + (((int64_t)u * splits + split) * r + a0 + ta) * DC;
    if (a0 + ta < re) {
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int cidx = cg + 8 * k;
            if (cidx < DC) out[cidx] = acc[k];
        }
    }
}

// Reduce split partials (fixed order, fp64) and solve L L^T X = Y~ for 8 RHS columns per CTA.
// One warp per column: forward substitution reads rows of L (left-looking), backward
// substitution is right-looking so it also reads rows of L (coalesced).
template <int D>
__global__ void __launch_bounds__(256) weights_solve_kernel(const float *__restrict__ Ypart,
                                                            const double *__restrict__ L,
                                                            const int32_t *__restrict__ r_eff, int r,
                                                            int splits, float *__restrict__ X) {
    constexpr int DC = D + 1;
    extern __shared__ double zs[];  // [8][r]
    const int u = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col = blockIdx.x * 8 + w;
    const int q = r_eff[u];
    double *z = zs + w * r;
    const double *Lu = L + (int64_t)u * r * r;
    float *Xu = X + (int64_t)u * r * DC;
    if (col >= DC) return;
    for (int a = lane; a < q; a += 32) {
        double y = 0.0;
        for (int sp = 0; sp < splits; ++sp) y += (double)Ypart[(((int64_t)u * splits + sp) * r + a) * DC + col];
        z[a] = y;
    }
    __syncwarp();
    // forward: z_a = (y_a - sum_{b<a} L[a][b] z_b) / L[a][a]
    for (int a = 0; a < q; ++a) {
        const double *La = Lu + (int64_t)a * r;
        double t = 0.0;
        for (int b = lane; b < a; b += 32) t += La[b] * z[b];
        t = warp_sum(t);
        if (lane == 0) z[a] = (z[a] - t) / La[a];
        __syncwarp();
    }
    // backward (right-looking): x_a = z_a / L[a][a];  z_b -= L[a][b] x_a  for b < a
    for (int a = q - 1; a >= 0; --a) {
        const double *La = Lu + (int64_t)a * r;
        const double xa = z[a] / La[a];
        __syncwarp();
        for (int b = lane; b < a; b += 32) z[b] -= La[b] * xa;
        if (lane == 0) z[a] = xa;
        __syncwarp();
    }
    for (int a = lane; a < r; a += 32) Xu[(int64_t)a * DC + col] = a < q ? (float)z[a] : 0.f;
}

template <typename T, int D>
__global__ void gather_ks_kernel(const T *__restrict__ K, const int32_t *__restrict__ S,
                                 const int32_t *__restrict__ r_eff, int64_t n, int r, T *__restrict__ KS) {
    const int u = blockIdx.y, a = blockIdx.x;
    const int q = r_eff[u];
    const int s = a < q ? S[(int64_t)u * r + a] : -1;
    for (int j = threadIdx.x; j < D; j += blockDim.x)
        KS[((int64_t)u * r + a) * D + j] = s >= 0 ? K[((int64_t)u * n + s) * D + j] : from_f32<T>(0.f);
}

template <typename T, int D>
int launch_weights_td(const Dims &Dm, const void *K, const void *V, const int32_t *S, const int32_t *r_eff,
                      const double *L, const double *stats, float *Ypart, void *KS, float *X, cudaStream_t st) {
    const int units = Dm.units();
    const int splits = weights_num_splits(Dm);
    dim3 g1(splits, (Dm.r + kTA - 1) / kTA, units);
    const size_t smem1 = D * sizeof(double) + (size_t)(kTA + 2 * kTL) * (D + 1) * sizeof(float) +
                         (size_t)kTA * (kTL + 1) * sizeof(float);
    auto pk = weights_partial_kernel<T, D>;
    if (smem1 > 48 * 1024) cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    pk<<<g1, kWT, smem1, st>>>(static_cast<const T *>(K), static_cast<const T *>(V), S,
                                                      r_eff, stats, Dm.n, Dm.r, splits, Ypart);
    const size_t smem = (size_t)8 * Dm.r * sizeof(double);
    auto sk = weights_solve_kernel<D>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 g2((D + 1 + 7) / 8, units);
    sk<<<g2, 256, smem, st>>>(Ypart, L, r_eff, Dm.r, splits, X);
    dim3 g3(Dm.r, units);
    gather_ks_kernel<T, D><<<g3, 128, 0, st>>>(static_cast<const T *>(K), S, r_eff, Dm.n, Dm.r,
                                               static_cast<T *>(KS));
    return cudaPeekAtLastError() == cudaSuccess ? 3 : -1;
}

template <typename T>
int launch_weights_t(const Dims &Dm, const void *K, const void *V, const int32_t *S, const int32_t *r_eff,
                     const double *L, const double *stats, float *Ypart, void *KS, float *X, cudaStream_t st) {
    switch (Dm.d) {
        case 16: return launch_weights_td<T, 16>(Dm, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
        case 32: return launch_weights_td<T, 32>(Dm, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
        case 64: return launch_weights_td<T, 64>(Dm, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
        case 128: return launch_weights_td<T, 128>(Dm, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
    }
    return -1;
}

}  // namespace

int weights_num_splits(const Dims &D) {
    const int64_t tiles = (int64_t)D.units() * ((D.r + kTA - 1) / kTA);
    const int64_t want = std::max<int64_t>(1, (148 * 4 + tiles - 1) / tiles);
    const int64_t by_n = std::max<int64_t>(1, ceil_div(D.n, 256));
    return (int)std::min<int64_t>(std::min<int64_t>(want, by_n), 512);
}

int launch_weights(const Dims &D, const void *K, const void *V, const int32_t *S, const int32_t *r_eff,
                   const double *L, const double *stats, float *Ypart, void *KS, float *X, cudaStream_t st) {
    if (D.dtype == 0) return launch_weights_t<float>(D, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
    return launch_weights_t<__nv_bfloat16>(D, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
}

}  // namespace wc
