// attend.cu -- A5 of the hot path: weighted coreset attention, Alg 3 WtdAttn.
//   S = beta Q K_S^T (K_S uncentred);  P = exp(S - rowmax)
//   num = P X[:, :d],  den = P X[:, d]       (X = [V_S, w])
//   O = clip(num/den where den > 0 else 0, vmin, vmax)        (Z14, Z15)
// CUDA-core fp32 version: 64-query tiles, 32-row coreset tiles staged in shared memory,
// online max rescaling across coreset tiles (exact: the shift cancels in num/den).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace wc {

namespace {

constexpr int kAT = 256;
constexpr int kBM = 64;  // queries per CTA
constexpr int kRT = 32;  // coreset rows per tile

template <typename T, int D>
__global__ void __launch_bounds__(kAT) attend_kernel(const T *__restrict__ Q, const T *__restrict__ KS,
                                                     const float *__restrict__ X,
                                                     const int32_t *__restrict__ r_eff, const T *__restrict__ vmin,
                                                     const T *__restrict__ vmax, int64_t m, int r, int group,
                                                     int hq, int hkv, float beta, int clip, T *__restrict__ O) {
    constexpr int DC = D + 1;
    constexpr int CPT = (DC + 3) / 4;  // output columns per thread
    extern __shared__ float asmem[];
    float (*Qs)[D + 1] = reinterpret_cast<float (*)[D + 1]>(asmem);  // [kBM][D+1]
    float (*Ks)[D + 1] = Qs + kBM;                                   // [kRT][D+1]
    float (*Xs)[DC + 1] = reinterpret_cast<float (*)[DC + 1]>(&Ks[kRT][0]);  // [kRT][DC+1]
    float (*Ps)[kRT + 1] = reinterpret_cast<float (*)[kRT + 1]>(&Xs[kRT][0]);  // [kBM][kRT+1]
    float *den_s = &Ps[kBM][0];                                      // [kBM]

    const int b = blockIdx.z, h = blockIdx.y;
    const int64_t q0 = (int64_t)blockIdx.x * kBM;
    const int u = b * hkv + h / group;
    const int re = r_eff[u];
    const int tid = threadIdx.x;
    const T *Qh = Q + ((int64_t)b * hq + h) * m * D;
    T *Oh = O + ((int64_t)b * hq + h) * m * D;
    const T *KSu = KS + (int64_t)u * r * D;
    const float *Xu = X + (int64_t)u * r * DC;

    for (int e = tid; e < kBM * D; e += kAT) {
        const int qi = e / D, j = e % D;
        Qs[qi][j] = (q0 + qi < m) ? to_f32(Qh[(q0 + qi) * D + j]) * beta : 0.f;
    }
    const int row = tid >> 2, sub = tid & 3;  // thread owns query `row`, columns sub + 4k
    float acc[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) acc[k] = 0.f;
    float mrow = -INFINITY;

    for (int s0 = 0; s0 < re; s0 += kRT) {
        __syncthreads();
        for (int e = tid; e < kRT * D; e += kAT) {
            const int a = e / D, j = e % D;
            Ks[a][j] = (s0 + a < re) ? to_f32(KSu[(int64_t)(s0 + a) * D + j]) : 0.f;
        }
        for (int e = tid; e < kRT * DC; e += kAT) {
            const int a = e / DC, c = e % DC;
            Xs[a][c] = (s0 + a < re) ? Xu[(int64_t)(s0 + a) * DC + c] : 0.f;
        }
        __syncthreads();
        // scores for (row, keys sub + 4k), k < 8
        float sc[kRT / 4];
        float mloc = -INFINITY;
#pragma unroll
        for (int k = 0; k < kRT / 4; ++k) {
            const int a = sub + 4 * k;
            float dot = 0.f;
#pragma unroll 16
            for (int j = 0; j < D; ++j) dot = fmaf(Qs[row][j], Ks[a][j], dot);
            sc[k] = (s0 + a < re) ? dot : -INFINITY;
            mloc = fmaxf(mloc, sc[k]);
        }
        mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1));
        mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 2));
        const float mnew = fmaxf(mrow, mloc);
        const float scale = (mrow == -INFINITY) ? 0.f : expf(mrow - mnew);
        mrow = mnew;
#pragma unroll
        for (int k = 0; k < kRT / 4; ++k) Ps[row][sub + 4 * k] = expf(sc[k] - mnew);
#pragma unroll
        for (int k = 0; k < CPT; ++k) acc[k] *= scale;
        __syncwarp();
#pragma unroll 4
        for (int a = 0; a < kRT; ++a) {
            const float pv = Ps[row][a];
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int c = sub + 4 * k;
                if (c < DC) acc[k] = fmaf(pv, Xs[a][c], acc[k]);
            }
        }
    }
    // den lives in column D, owned by sub == D % 4 at slot D / 4
    if (sub == (D & 3)) den_s[row] = acc[D >> 2];
    __syncthreads();
    const float den = den_s[row];
    const int64_t qi = q0 + row;
    if (qi < m) {
        const T *vmn = vmin + (int64_t)u * D;
        const T *vmx = vmax + (int64_t)u * D;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int c = sub + 4 * k;
            if (c < D) {
                float o = den > 0.f ? acc[k] / den : 0.f;
                if (clip) o = fminf(fmaxf(o, to_f32(vmn[c])), to_f32(vmx[c]));
                Oh[qi * D + c] = from_f32<T>(o);
            }
        }
    }
}

template <typename T, int D>
int launch_attend_td(const Dims &Dm, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                     const void *vmin, const void *vmax, double beta, int clip, void *O, cudaStream_t st) {
    if (Dm.m == 0) return 0;
    constexpr int DC = D + 1;
    const size_t smem = ((size_t)kBM * (D + 1) + (size_t)kRT * (D + 1) + (size_t)kRT * (DC + 1) +
                         (size_t)kBM * (kRT + 1) + kBM) * sizeof(float);
    auto kern = attend_kernel<T, D>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)ceil_div(Dm.m, kBM), Dm.hq, Dm.batch);
    kern<<<grid, kAT, smem, st>>>(static_cast<const T *>(Q), static_cast<const T *>(KS), X, r_eff,
                                  static_cast<const T *>(vmin), static_cast<const T *>(vmax), Dm.m, Dm.r,
                                  Dm.group(), Dm.hq, Dm.hkv, (float)beta, clip, static_cast<T *>(O));
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T>
int launch_attend_t(const Dims &Dm, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                    const void *vmin, const void *vmax, double beta, int clip, void *O, cudaStream_t st) {
    switch (Dm.d) {
        case 16: return launch_attend_td<T, 16>(Dm, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, st);
        case 32: return launch_attend_td<T, 32>(Dm, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, st);
        case 64: return launch_attend_td<T, 64>(Dm, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, st);
        case 128: return launch_attend_td<T, 128>(Dm, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, st);
    }
    return -1;
}

}  // namespace

int launch_attend(const Dims &D, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                  const void *vmin, const void *vmax, double beta, int clip, void *O, cudaStream_t st) {
    if (D.dtype == 0) return launch_attend_t<float>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, st);
    return launch_attend_t<__nv_bfloat16>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, st);
}

}  // namespace wc
