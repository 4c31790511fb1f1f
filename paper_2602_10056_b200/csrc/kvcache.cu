// kvcache.cu -- KV-cache compression ("prefill phase"; E3 protocol P:667-669) around the
// CompressKV kernels, and the decode-shaped WtdAttn (Alg 3) for few queries per head.
//
// Reading Z24: the cache of a unit is the union of exact retained entries and the
// CompressKV coreset of the middle tokens.  Each cache row is a key row KC[a] plus a [value | weight]
// row XC[a]:
//   rows [0, kf)            first kf tokens,  (k_l, [v_l, 1])
//   rows [kf, kf + kl)      last kl tokens,   (k_l, [v_l, 1])
//   rows [kf + kl, c_eff)   coreset rows of the middle, (k_s, [V_S, w]_s) in Alg 2 order
//   rows [c_eff, C)         zero
// so WtdAttn over the cache adds the retained tokens' exact terms to the Nystrom estimate of the
// middle's unnormalised sums under one softmax shift.
//
//   kv_assemble_kernel:    writes KC / XC / c_eff / S (global token indices) from the retained rows of
//                          K, V and the middle's KS / X / S / r_eff.
//   attend_decode_kernel:  Alg 3 for m <= kDecodeMaxM queries per q-head (decode): the unit's query
//                          rows (contiguous: the q-heads of a kv-group are adjacent) in chunks of 16,
//                          the cache in chunks of 64 rows, one CTA per (chunk, unit, query chunk);
//                          scores and P.[V_S, w] in fp32 on CUDA cores (a 16-row tile would leave a
//                          128-row tcgen05 MMA 87 % idle; the step is bound by reading the cache);
//                          per-chunk (max, num, den) partials merged by the last CTA of the unit (an
//                          atomic ticket), which applies the shift, the division and the clip.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace wc {

namespace {

template <typename T>
__global__ void kv_assemble_kernel(const T *__restrict__ K, const T *__restrict__ V, int64_t n, int d, int kf, int kl,
                                   int R, const T *__restrict__ KS, const float *__restrict__ X,
                                   const int32_t *__restrict__ Smid, const int32_t *__restrict__ reff_mid,
                                   T *__restrict__ KC, float *__restrict__ XC, int32_t *__restrict__ c_eff,
                                   int32_t *__restrict__ S_out) {
    const int u = blockIdx.y, kept = kf + kl, C = kept + R, dc = d + 1;
    const int re = reff_mid ? reff_mid[u] : 0;
    const int rows_per_block = blockDim.x / 32;
    const int a = blockIdx.x * rows_per_block + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0) c_eff[u] = kept + re;
    if (a >= C) return;
    T *kc = KC + ((int64_t)u * C + a) * d;
    float *xc = XC + ((int64_t)u * C + a) * dc;
    if (a < kept) {  // retained token (k_l, [v_l, 1])
        const int64_t l = a < kf ? a : n - kl + (a - kf);
        const T *k = K + ((int64_t)u * n + l) * d, *v = V + ((int64_t)u * n + l) * d;
        for (int j = lane; j < d; j += 32) {
            kc[j] = k[j];
            xc[j] = to_f32(v[j]);
        }
        if (lane == 0) xc[d] = 1.f;
        return;
    }
    const int j0 = a - kept;  // coreset row j0 of the middle
    if (lane == 0 && S_out) S_out[(int64_t)u * R + j0] = j0 < re ? Smid[(int64_t)u * R + j0] + kf : -1;
    const bool ok = j0 < re;
    for (int j = lane; j < d; j += 32) kc[j] = ok ? KS[((int64_t)u * R + j0) * d + j] : from_f32<T>(0.f);
    for (int j = lane; j < dc; j += 32) xc[j] = ok ? X[((int64_t)u * R + j0) * dc + j] : 0.f;
}

constexpr int kDecQ = 16;   // query rows per CTA
constexpr int kDecC = 64;   // cache rows per CTA
constexpr int kDecT = 256;  // threads

template <int D> struct DecSmem {
    static constexpr int kQ = 0;                                // [kDecQ][D]    fp32, scaled by beta*log2(e)
    static constexpr int kK = kQ + kDecQ * D;                   // [kDecC][D+1]  fp32
    static constexpr int kX = kK + kDecC * (D + 1);             // [kDecC][D+1]  fp32 ([V_S, w] rows)
    static constexpr int kS = kX + kDecC * (D + 1);             // [kDecQ][kDecC] scores -> P
    static constexpr int kM = kS + kDecQ * kDecC;               // [kDecQ] chunk max
    static constexpr int kFloats = kM + kDecQ + 1;
    static constexpr size_t kBytes = (size_t)kFloats * 4;
};

// part: [units][qz][splits][kDecQ][D + 2] = (max, num[0..D-1], den) per (chunk, row), log2 domain.
template <typename T, int D>
__global__ void __launch_bounds__(kDecT) attend_decode_kernel(
    const T *__restrict__ Q, const T *__restrict__ KS, const float *__restrict__ X, const int32_t *__restrict__ r_eff,
    const T *__restrict__ vmin, const T *__restrict__ vmax, int64_t m, int r, int group, int hq, int hkv, float sl2,
    int clip, T *__restrict__ O, float *__restrict__ part, unsigned *__restrict__ tickets) {
    extern __shared__ float sm[];
    using L = DecSmem<D>;
    float *qs = sm + L::kQ, *ks = sm + L::kK, *xs = sm + L::kX, *ss = sm + L::kS, *mx = sm + L::kM;
    constexpr int DC = D + 1, PW = D + 2;
    const int split = blockIdx.x, u = blockIdx.y, z = blockIdx.z, splits = gridDim.x, qz = gridDim.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b = u / hkv, h = u % hkv;
    const int64_t rows = (int64_t)group * m;  // the unit's query rows are contiguous
    const int64_t qoff = ((int64_t)b * hq + (int64_t)h * group) * m;
    const int64_t t0 = (int64_t)z * kDecQ;
    const int nq = (int)(rows - t0 < kDecQ ? rows - t0 : kDecQ);
    const int re = r_eff[u];
    const int c0 = split * kDecC, nc = max(0, min(kDecC, re - c0));
    float *pp = part + ((((int64_t)u * qz + z) * splits + split) * kDecQ) * PW;

    if (nc > 0) {
        for (int e = tid; e < kDecQ * D; e += kDecT) {
            const int q = e / D, j = e % D;
            qs[e] = q < nq ? to_f32(Q[(qoff + t0 + q) * D + j]) * sl2 : 0.f;
        }
        const T *kr = KS + ((int64_t)u * r + c0) * D;
        for (int e = tid; e < nc * D; e += kDecT) ks[(e / D) * DC + e % D] = to_f32(kr[e]);
        const float *xr = X + ((int64_t)u * r + c0) * DC;
        for (int e = tid; e < nc * DC; e += kDecT) xs[e] = xr[e];
        __syncthreads();
        // scores: thread -> row q = tid / 16, cache rows c = tid % 16 + 16 k
        {
            const int q = tid >> 4, cl = tid & 15;
            float acc[kDecC / 16];
#pragma unroll
            for (int k = 0; k < kDecC / 16; ++k) acc[k] = 0.f;
#pragma unroll 8
            for (int j = 0; j < D; ++j) {
                const float qv = qs[q * D + j];
#pragma unroll
                for (int k = 0; k < kDecC / 16; ++k) acc[k] = fmaf(qv, ks[(cl + 16 * k) * DC + j], acc[k]);
            }
#pragma unroll
            for (int k = 0; k < kDecC / 16; ++k) ss[q * kDecC + cl + 16 * k] = cl + 16 * k < nc ? acc[k] : -INFINITY;
        }
        __syncthreads();
        // per row: chunk max, P = 2^(s - max); warp w owns rows 2w, 2w + 1
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int q = 2 * warp + rr;
            float a0 = ss[q * kDecC + lane], a1 = ss[q * kDecC + lane + 32];
            float mm = fmaxf(a0, a1);
#pragma unroll
            for (int o = 16; o; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
            ss[q * kDecC + lane] = lane < nc ? exp2f(a0 - mm) : 0.f;
            ss[q * kDecC + lane + 32] = lane + 32 < nc ? exp2f(a1 - mm) : 0.f;
            if (lane == 0) mx[q] = mm;
        }
        __syncthreads();
        // partial [num | den] = P . [V_S, w]: warp w rows 2w, 2w + 1, lane -> columns lane + 32 k
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int q = 2 * warp + rr;
            float acc[(DC + 31) / 32];
#pragma unroll
            for (int k = 0; k < (DC + 31) / 32; ++k) acc[k] = 0.f;
            for (int c = 0; c < nc; ++c) {
                const float p = ss[q * kDecC + c];
#pragma unroll
                for (int k = 0; k < (DC + 31) / 32; ++k) {
                    const int col = lane + 32 * k;
                    if (col < DC) acc[k] = fmaf(p, xs[c * DC + col], acc[k]);
                }
            }
            float *o = pp + (int64_t)q * PW;
            if (lane == 0) o[0] = mx[q];
#pragma unroll
            for (int k = 0; k < (DC + 31) / 32; ++k) {
                const int col = lane + 32 * k;
                if (col < DC) o[1 + col] = acc[k];
            }
        }
    } else {
        for (int e = tid; e < kDecQ * PW; e += kDecT) pp[e] = (e % PW) == 0 ? -INFINITY : 0.f;
    }
    // the last CTA of (unit, query chunk) merges the chunk partials
    __shared__ unsigned s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned t = atomicAdd(tickets + (int64_t)u * qz + z, 1u);
        s_last = (t == (unsigned)splits - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float *pu = part + (((int64_t)u * qz + z) * splits) * kDecQ * PW;
    for (int q = warp; q < nq; q += kDecT / 32) {
        float M = -INFINITY;
        for (int s = lane; s < splits; s += 32) M = fmaxf(M, __ldcg(pu + ((int64_t)s * kDecQ + q) * PW));
#pragma unroll
        for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        float acc[(DC + 31) / 32];
#pragma unroll
        for (int k = 0; k < (DC + 31) / 32; ++k) acc[k] = 0.f;
        if (M > -INFINITY) {
            for (int s = 0; s < splits; ++s) {
                const float *ps = pu + ((int64_t)s * kDecQ + q) * PW;
                const float ms = __ldcg(ps);
                if (!(ms > -INFINITY)) continue;
                const float f = exp2f(ms - M);
#pragma unroll
                for (int k = 0; k < (DC + 31) / 32; ++k) {
                    const int col = lane + 32 * k;
                    if (col < DC) acc[k] = fmaf(f, __ldcg(ps + 1 + col), acc[k]);
                }
            }
        }
        // den = column D: lane D % 32 of chunk k = D / 32
        const float den = __shfl_sync(0xffffffffu, acc[D / 32], D % 32);
        T *orow = O + (qoff + t0 + q) * D;
#pragma unroll
        for (int k = 0; k < (DC + 31) / 32; ++k) {
            const int col = lane + 32 * k;
            if (col < D) {
                float o = den > 0.f ? acc[k] / den : 0.f;
                if (clip) o = fminf(fmaxf(o, to_f32(vmin[(int64_t)u * D + col])), to_f32(vmax[(int64_t)u * D + col]));
                orow[col] = from_f32<T>(o);
            }
        }
    }
    if (tid == 0) tickets[(int64_t)u * qz + z] = 0u;  // reusable without a reset launch
}

template <typename T, int D>
int launch_decode_td(const Dims &Dm, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                     const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws, cudaStream_t st) {
    using L = DecSmem<D>;
    const int splits = (int)std::max<int64_t>(1, (Dm.r + kDecC - 1) / kDecC);
    const int qz = (int)(((int64_t)Dm.group() * Dm.m + kDecQ - 1) / kDecQ);
    float *part = static_cast<float *>(ws);
    unsigned *tickets = reinterpret_cast<unsigned *>(
        static_cast<char *>(ws) + (size_t)Dm.units() * qz * splits * kDecQ * (D + 2) * sizeof(float));
    if (cudaMemsetAsync(tickets, 0, (size_t)Dm.units() * qz * sizeof(unsigned), st) != cudaSuccess) return -1;
    auto kern = attend_decode_kernel<T, D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::kBytes);
    kern<<<dim3(splits, Dm.units(), qz), kDecT, L::kBytes, st>>>(
        static_cast<const T *>(Q), static_cast<const T *>(KS), X, r_eff, static_cast<const T *>(vmin),
        static_cast<const T *>(vmax), Dm.m, Dm.r, Dm.group(), Dm.hq, Dm.hkv, (float)(beta * 1.4426950408889634), clip,
        static_cast<T *>(O), part, tickets);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T>
int launch_decode_t(const Dims &Dm, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                    const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws, cudaStream_t st) {
    switch (Dm.d) {
        case 16: return launch_decode_td<T, 16>(Dm, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
        case 32: return launch_decode_td<T, 32>(Dm, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
        case 64: return launch_decode_td<T, 64>(Dm, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
        case 128: return launch_decode_td<T, 128>(Dm, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
    }
    return -1;
}

}  // namespace

size_t attend_decode_ws_bytes(const Dims &D) {
    const int64_t splits = std::max<int64_t>(1, (D.r + kDecC - 1) / kDecC);
    const int64_t qz = ((int64_t)D.group() * D.m + kDecQ - 1) / kDecQ;
    return (size_t)D.units() * qz * splits * kDecQ * (D.d + 2) * sizeof(float) + (size_t)D.units() * qz * 4 + 256;
}

int launch_attend_decode(const Dims &D, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                         const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws,
                         cudaStream_t st) {
    if (D.m == 0) return 0;
    if (!ws) return -1;
    if (D.dtype == 0) return launch_decode_t<float>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
    return launch_decode_t<__nv_bfloat16>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
}

int launch_kv_assemble(const Dims &D, const void *K, const void *V, int kf, int kl, int R, const void *KS,
                       const float *X, const int32_t *Smid, const int32_t *reff_mid, void *KC, float *XC,
                       int32_t *c_eff, int32_t *S_out, cudaStream_t st) {
    const int C = kf + kl + R;
    dim3 g((unsigned)std::max(1, (C + 7) / 8), D.units());
    if (D.dtype == 0)
        kv_assemble_kernel<float><<<g, 256, 0, st>>>(static_cast<const float *>(K), static_cast<const float *>(V), D.n,
                                                     D.d, kf, kl, R, static_cast<const float *>(KS), X, Smid, reff_mid,
                                                     static_cast<float *>(KC), XC, c_eff, S_out);
    else
        kv_assemble_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(
            static_cast<const __nv_bfloat16 *>(K), static_cast<const __nv_bfloat16 *>(V), D.n, D.d, kf, kl, R,
            static_cast<const __nv_bfloat16 *>(KS), X, Smid, reff_mid, static_cast<__nv_bfloat16 *>(KC), XC, c_eff,
            S_out);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace wc
