// kvcache.cu -- KV-cache compression ("prefill phase"; E3 protocol P:667-669) around the
// CompressKV kernels, and the decode-shaped WtdAttn (Alg 3) for few queries per head.
//
// Reading Z24: the cache of a unit is the union of exact retained entries and the
// CompressKV coreset of the middle tokens.  Each cache row is a key row KC[a], a value row VC[a] (the
// cache dtype: V_S rounded like the keys) and a weight WC[a] (fp32):
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
                                   T *__restrict__ KC, T *__restrict__ VC, float *__restrict__ WC,
                                   int32_t *__restrict__ c_eff, int32_t *__restrict__ S_out) {
    const int u = blockIdx.y, kept = kf + kl, C = kept + R, dc = d + 1;
    const int re = reff_mid ? reff_mid[u] : 0;
    const int rows_per_block = blockDim.x / 32;
    const int a = blockIdx.x * rows_per_block + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0) c_eff[u] = kept + re;
    if (a >= C) return;
    T *kc = KC + ((int64_t)u * C + a) * d;
    T *vc = VC + ((int64_t)u * C + a) * d;
    float *wc = WC + (int64_t)u * C + a;
    if (a < kept) {  // retained token (k_l, v_l, 1)
        const int64_t l = a < kf ? a : n - kl + (a - kf);
        const T *k = K + ((int64_t)u * n + l) * d, *v = V + ((int64_t)u * n + l) * d;
        for (int j = lane; j < d; j += 32) {
            kc[j] = k[j];
            vc[j] = v[j];
        }
        if (lane == 0) *wc = 1.f;
        return;
    }
    const int j0 = a - kept;  // coreset row j0 of the middle
    if (lane == 0 && S_out) S_out[(int64_t)u * R + j0] = j0 < re ? Smid[(int64_t)u * R + j0] + kf : -1;
    const bool ok = j0 < re;
    for (int j = lane; j < d; j += 32) {
        kc[j] = ok ? KS[((int64_t)u * R + j0) * d + j] : from_f32<T>(0.f);
        vc[j] = from_f32<T>(ok ? X[((int64_t)u * R + j0) * dc + j] : 0.f);  // V_S rounded to the cache dtype
    }
    if (lane == 0) *wc = ok ? X[((int64_t)u * R + j0) * dc + d] : 0.f;
}

constexpr int kDecC = 64;   // cache rows per tile
constexpr int kDecT = 256;  // threads: QR query rows x (256 / QR) threads
constexpr int kDecQmax = 16;

template <int D, int QR> struct DecSmem {
    static constexpr int kQ = 0;                                // [QR][D]       fp32, scaled by beta*log2(e)
    static constexpr int kKW = D + 1;                           // K row stride in 32-bit words (raw elements;
    static constexpr int kK = kQ + QR * D;                      //  bf16 rows use (D/2 + 1) of them)
    static constexpr int kX = kK + kDecC * kKW;                 // [kDecC][D+1]  fp32 ([V_S, w] rows)
    static constexpr int kS = kX + kDecC * (D + 1);             // [kDecC][QR]   P (row-major over cache rows)
    static constexpr int kF = kS + QR * kDecC;                  // [QR] this tile's rescale factors
    static constexpr int kDen = kF + QR;                        // [QR] running denominators
    static constexpr int kRed = kDen + QR;                      // [2][8] cross-warp max / den partials
                                                                //  (MMA scores: [2][8 warps][4] + run / new max)
    static constexpr int kR = kRed + 80;                        // [256/D][QR][D] row-group partial sums
    static constexpr int kFloats = kR + kDecT * QR;
    static constexpr size_t kBytes = (size_t)kFloats * 4;
};

// One cache tile (kDecC rows of KS and X) held in registers between its global load and its
// shared-memory store, so the next tile's loads are in flight while the current one is computed.
template <typename T, int D, bool COMPACT> struct DecTile {
    static constexpr int kKTot = kDecC * D * (int)sizeof(T) / 16;       // 16-byte K vectors per tile
    static constexpr int kKVec = (kKTot + kDecT - 1) / kDecT;             // ... per thread
    static constexpr int kXF = COMPACT ? 0 : kDecC * (D + 1) / kDecT;     // X floats per thread (exact)
    static constexpr int kXRem = COMPACT ? 0 : kDecC * (D + 1) - kXF * kDecT;
    uint4 k[kKVec];
    float x[kXF + 1];  // fp32 [V_S, w] path
    // [V_S, w] rows from the fp32 X rows, or (Xu == nullptr) from a compact KV cache: values VCu (dtype
    // [C][D]) and weights WCu (fp32 [C])
    __device__ __forceinline__ void load(const T *KSu, const float *Xu, const T *VCu, const float *WCu, int c0, int nc,
                                         int tid) {
        const uint4 *kv = reinterpret_cast<const uint4 *>(KSu + (int64_t)c0 * D);
        constexpr int kPerRow = D * (int)sizeof(T) / 16;
#pragma unroll
        for (int i = 0; i < kKVec; ++i) {
            const int e = tid + i * kDecT;
            k[i] = (e < kKTot && e / kPerRow < nc) ? __ldg(kv + e) : make_uint4(0, 0, 0, 0);
        }
        const int lim = nc * (D + 1);
        if constexpr (!COMPACT) {
            const float *xr = Xu + (int64_t)c0 * (D + 1);
#pragma unroll
            for (int i = 0; i < kXF; ++i) {
                const int e = tid + i * kDecT;
                x[i] = e < lim ? __ldg(xr + e) : 0.f;
            }
            if (kXRem) x[kXF] = (tid < kXRem && kXF * kDecT + tid < lim) ? __ldg(xr + kXF * kDecT + tid) : 0.f;
        } else {  // compact cache: 16-byte vectors of the value rows, one weight per thread
            const uint4 *vr = reinterpret_cast<const uint4 *>(VCu + (int64_t)c0 * D);
            constexpr int kPerRow = D * (int)sizeof(T) / 16;
#pragma unroll
            for (int i = 0; i < kVVec; ++i) {
                const int e = tid + i * kDecT;
                v[i] = (e < kVTot && e / kPerRow < nc) ? __ldg(vr + e) : make_uint4(0, 0, 0, 0);
            }
            w = tid < nc ? __ldg(WCu + c0 + tid) : 0.f;
        }
    }
    // compact cache: 16-byte value vectors and the weights of the tile (registers until the store)
    static constexpr int kVTot = COMPACT ? kDecC * D * (int)sizeof(T) / 16 : 0;
    static constexpr int kVVec = COMPACT ? (kVTot + kDecT - 1) / kDecT : 1;
    uint4 v[kVVec];
    float w;
    // K rows stay raw (bf16 pairs / fp32) in shared memory, row stride kW = D*sizeof(T)/4 + 1 words
    // (odd: the score loop's row-per-lane reads are conflict-free); 4 word stores per vector.
    static constexpr int kW = D * (int)sizeof(T) / 4 + 1;
    __device__ __forceinline__ void store(uint32_t *ks, float *xs, int tid) const {
        constexpr int kPerRow = D * (int)sizeof(T) / 16;
#pragma unroll
        for (int i = 0; i < kKVec; ++i) {
            const int e = tid + i * kDecT, row = e / kPerRow, c = e % kPerRow;
            if (kKTot % kDecT && e >= kKTot) break;
            uint32_t *dst = ks + row * kW + 4 * c;
            dst[0] = k[i].x; dst[1] = k[i].y; dst[2] = k[i].z; dst[3] = k[i].w;
        }
        if constexpr (!COMPACT) {
#pragma unroll
            for (int i = 0; i < kXF; ++i) xs[tid + i * kDecT] = x[i];
            if (kXRem && tid < kXRem) xs[kXF * kDecT + tid] = x[kXF];
        } else {  // [V_S, w] rows of the fp32 tile from the compact cache
            constexpr int kEl = 16 / (int)sizeof(T), kPerRow = D / kEl;
#pragma unroll
            for (int i = 0; i < kVVec; ++i) {
                const int e = tid + i * kDecT, row = e / kPerRow, c = (e % kPerRow) * kEl;
                if (kVTot % kDecT && e >= kVTot) break;
                const uint32_t wd[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
                float *dst = xs + row * (D + 1) + c;
                if constexpr (sizeof(T) == 2) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        dst[2 * k] = __uint_as_float(wd[k] << 16);
                        dst[2 * k + 1] = __uint_as_float(wd[k] & 0xffff0000u);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) dst[k] = __uint_as_float(wd[k]);
                }
            }
            if (tid < kDecC) xs[tid * (D + 1) + D] = w;
        }
    }
};

// bf16 tensor-core MMA m16n8k16 (fp32 accumulate): D = A B + C, A 16x16 row-major, B 16x8 column-major.
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Grid (splits, units, qz).  CTA (split, u, z) runs query rows [QR z, QR z + QR) of unit u over the
// cache tiles split, split + splits, ... (kDecC rows each) with an online max.
//   scores: thread (q = tid / TPR, g = tid % TPR), TPR = 256 / QR, computes query row q's scores of
//           cache rows g + TPR k, the tile max, P = 2^(s - max) and P . w (the weight column, reduced
//           over the row's TPR threads into the running denominator);
//   P . V_S: thread (col = tid % D, rg = tid / D) owns value column col for ALL QR query rows over the
//           cache rows of row group rg (rows rg, rg + RS, ...; RS = 256 / D), so each X element is read
//           once from shared memory and P arrives as one vector load per cache row.
// QR = 4 serves one decode token of a 4-query-head group.
// part: [units][qz][splits][QR][D + 2] = (max, num[0..D-1], den) per CTA and row (log2 domain).
template <typename T, int D, int QR, bool COMPACT>
__global__ void __launch_bounds__(kDecT) attend_decode_kernel(
    const T *__restrict__ Q, const T *__restrict__ KS, const float *__restrict__ X, const T *__restrict__ VC,
    const float *__restrict__ WC, const int32_t *__restrict__ r_eff,
    const T *__restrict__ vmin, const T *__restrict__ vmax, int64_t m, int r, int group, int hq, int hkv, float sl2,
    int clip, T *__restrict__ O, float *__restrict__ part, unsigned *__restrict__ tickets) {
    extern __shared__ float sm[];
    using L = DecSmem<D, QR>;
    float *qs = sm + L::kQ, *xs = sm + L::kX, *ps = sm + L::kS, *fs = sm + L::kF, *dens = sm + L::kDen;
    float *red = sm + L::kRed;
    uint32_t *ks = reinterpret_cast<uint32_t *>(sm + L::kK);
    constexpr int KW = DecTile<T, D, COMPACT>::kW;
    constexpr int TPR = kDecT / QR, DC = D + 1, PW = D + 2, NS = kDecC / TPR;
    constexpr int WPR = TPR > 32 ? TPR / 32 : 1;  // warps per query row (score phase)
    constexpr int RS = kDecT / D;                 // row groups of the P . V_S phase
    const int split = blockIdx.x, u = blockIdx.y, z = blockIdx.z, splits = gridDim.x, qz = gridDim.z;
    const int tid = threadIdx.x, q = tid / TPR, g = tid % TPR, col = tid % D, rg = tid / D;
    const int b = u / hkv, h = u % hkv;
    const int64_t rows = (int64_t)group * m;  // the unit's query rows are contiguous
    const int64_t qoff = ((int64_t)b * hq + (int64_t)h * group) * m;
    const int64_t t0 = (int64_t)z * QR;
    const int nq = (int)(rows - t0 < QR ? rows - t0 : QR);
    const int re = r_eff[u];
    const int ntiles = (re + kDecC - 1) / kDecC;
    const T *KSu = KS + (int64_t)u * r * D;
    const float *Xu = X ? X + (int64_t)u * r * DC : nullptr;
    const T *VCu = VC ? VC + (int64_t)u * r * D : nullptr;
    const float *WCu = WC ? WC + (int64_t)u * r : nullptr;

    for (int e = tid; e < QR * D; e += kDecT) {
        const int qq = e / D, j = e % D;
        qs[e] = qq < nq ? to_f32(Q[(qoff + t0 + qq) * D + j]) * sl2 : 0.f;
    }
    if (tid < QR) dens[tid] = 0.f;
    float acc[QR];
#pragma unroll
    for (int k = 0; k < QR; ++k) acc[k] = 0.f;
    float mrun = -INFINITY;  // of query row q (score-phase mapping)
    // QR = 4, bf16: the scores run on the tensor cores (m16n8k16, the 4 query rows padded to 16): warp
    // w forms S[0:4, 8w:8w+8] of the 64-row tile over D/16 k-steps; A fragments (raw bf16 Q) stay in
    // registers for the whole CTA, B fragments are the raw key words in shared memory.  Products of
    // bf16 are exact in fp32; the beta*log2(e) scale is applied to the fp32 result.
    constexpr bool kMma = (QR == 4) && (sizeof(T) == 2);
    const int lane = tid & 31, wq = tid >> 5, gid = lane >> 2, tq = lane & 3;
    uint32_t aq[kMma ? D / 16 : 1][2];
    float *mrun_s = red + 64, *mnew_s = red + 68;
    if constexpr (kMma) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            const bool okq = gid < nq;
            const uint32_t *qr = reinterpret_cast<const uint32_t *>(Q + (qoff + t0 + (okq ? gid : 0)) * D);
            aq[kk][0] = okq ? __ldg(qr + kk * 8 + tq) : 0u;
            aq[kk][1] = okq ? __ldg(qr + kk * 8 + 4 + tq) : 0u;
        }
        if (tid < 4) mrun_s[tid] = -INFINITY;
    }
    DecTile<T, D, COMPACT> tile;
    int tcur = split;
    if (tcur < ntiles) tile.load(KSu, Xu, VCu, WCu, tcur * kDecC, min(kDecC, re - tcur * kDecC), tid);
    while (tcur < ntiles) {
        const int nc = min(kDecC, re - tcur * kDecC);
        __syncthreads();  // previous tile's readers are done with ks / xs / ps / red
        tile.store(ks, xs, tid);
        const int tnext = tcur + splits;
        if (tnext < ntiles) tile.load(KSu, Xu, VCu, WCu, tnext * kDecC, min(kDecC, re - tnext * kDecC), tid);
        __syncthreads();
        if constexpr (kMma) {
            float c4[4] = {0.f, 0.f, 0.f, 0.f};
            const uint32_t *kr = ks + (8 * wq + gid) * KW;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t a4[4] = {aq[kk][0], 0u, aq[kk][1], 0u};
                mma_bf16_16816(c4, a4, kr[kk * 8 + tq], kr[kk * 8 + 4 + tq]);
            }
            // lane (gid, tq): query gid, cache rows 8 wq + 2 tq + {0, 1}
            const int c0 = 8 * wq + 2 * tq;
            const float s0 = c0 < nc ? c4[0] * sl2 : -INFINITY, s1 = c0 + 1 < nc ? c4[1] * sl2 : -INFINITY;
            float tm = fmaxf(s0, s1);
            tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 1));
            tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 2));
            if (tq == 0 && gid < 4) red[wq * 4 + gid] = tm;
            __syncthreads();
            if (tid < 4) {  // per query: tile max over the 8 warps, running max, rescale factor
                float m8 = red[tid];
#pragma unroll
                for (int w8 = 1; w8 < 8; ++w8) m8 = fmaxf(m8, red[w8 * 4 + tid]);
                const float mo = mrun_s[tid], mn = fmaxf(mo, m8);  // nc >= 1, so finite
                fs[tid] = exp2f(mo - mn);  // 0 on the first tile
                mrun_s[tid] = mn;
                mnew_s[tid] = mn;
            }
            __syncthreads();
            float dp = 0.f;
            if (gid < 4) {
                const float mn = mnew_s[gid];
                const float p0 = exp2f(s0 - mn), p1 = exp2f(s1 - mn);  // 0 for rows past nc
                ps[c0 * QR + gid] = p0;
                ps[(c0 + 1) * QR + gid] = p1;
                if (c0 < nc) dp = fmaf(p0, xs[c0 * DC + D], dp);
                if (c0 + 1 < nc) dp = fmaf(p1, xs[(c0 + 1) * DC + D], dp);
            }
            dp += __shfl_xor_sync(0xffffffffu, dp, 1);
            dp += __shfl_xor_sync(0xffffffffu, dp, 2);
            if (tq == 0 && gid < 4) red[32 + wq * 4 + gid] = dp;
            __syncthreads();
            if (tid < 4) {
                float d8 = 0.f;
#pragma unroll
                for (int w8 = 0; w8 < 8; ++w8) d8 += red[32 + w8 * 4 + tid];
                dens[tid] = dens[tid] * fs[tid] + d8;
            }
            mrun = mrun_s[q];
            __syncthreads();
        } else {
        // ---- scores of query row q against cache rows g + TPR k
            float sc[NS], sc2[NS];
    #pragma unroll
            for (int k = 0; k < NS; ++k) sc[k] = sc2[k] = 0.f;
            if constexpr (sizeof(T) == 2) {
    #pragma unroll 8
                for (int j2 = 0; j2 < D / 2; ++j2) {
                    const float2 qv = *reinterpret_cast<const float2 *>(qs + q * D + 2 * j2);
    #pragma unroll
                    for (int k = 0; k < NS; ++k) {
                        const uint32_t w = ks[(g + TPR * k) * KW + j2];
                        sc[k] = fmaf(qv.x, __uint_as_float(w << 16), sc[k]);
                        sc2[k] = fmaf(qv.y, __uint_as_float(w & 0xffff0000u), sc2[k]);
                    }
                }
            } else {
    #pragma unroll 8
                for (int j = 0; j < D; j += 2) {
                    const float2 qv = *reinterpret_cast<const float2 *>(qs + q * D + j);
    #pragma unroll
                    for (int k = 0; k < NS; ++k) {
                        sc[k] = fmaf(qv.x, __uint_as_float(ks[(g + TPR * k) * KW + j]), sc[k]);
                        sc2[k] = fmaf(qv.y, __uint_as_float(ks[(g + TPR * k) * KW + j + 1]), sc2[k]);
                    }
                }
            }
            float tm = -INFINITY;
    #pragma unroll
            for (int k = 0; k < NS; ++k) {
                sc[k] = g + TPR * k < nc ? sc[k] + sc2[k] : -INFINITY;
                tm = fmaxf(tm, sc[k]);
            }
    #pragma unroll
            for (int o = (TPR < 32 ? TPR : 32) / 2; o; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
            if constexpr (WPR > 1) {
                if ((tid & 31) == 0) red[tid >> 5] = tm;
                __syncthreads();
    #pragma unroll
                for (int w = 0; w < WPR; ++w) tm = fmaxf(tm, red[q * WPR + w]);
            }
            const float mnew = fmaxf(mrun, tm);  // nc >= 1, so finite
            const float f = exp2f(mrun - mnew);  // 0 on the first tile
            mrun = mnew;
            float dp = 0.f;
    #pragma unroll
            for (int k = 0; k < NS; ++k) {
                const int c = g + TPR * k;
                const float pv = exp2f(sc[k] - mnew);  // 0 for rows past nc
                ps[c * QR + q] = pv;
                if (c < nc) dp = fmaf(pv, xs[c * DC + D], dp);
            }
    #pragma unroll
            for (int o = (TPR < 32 ? TPR : 32) / 2; o; o >>= 1) dp += __shfl_xor_sync(0xffffffffu, dp, o);
            if constexpr (WPR > 1) {
                if ((tid & 31) == 0) red[8 + (tid >> 5)] = dp;
                __syncthreads();
                if (g == 0) {
                    dp = 0.f;
    #pragma unroll
                    for (int w = 0; w < WPR; ++w) dp += red[8 + q * WPR + w];
                }
            }
            if (g == 0) {
                dens[q] = dens[q] * f + dp;
                fs[q] = f;
            }
            __syncthreads();
        }
        // ---- P . V_S: column col for all QR query rows over the row group's cache rows
#pragma unroll
        for (int k = 0; k < QR; ++k) acc[k] *= fs[k];
#pragma unroll 4
        for (int c = rg; c < nc; c += RS) {
            const float x = xs[c * DC + col];
#pragma unroll
            for (int k4 = 0; k4 < QR; k4 += 4) {
                const float4 p4 = *reinterpret_cast<const float4 *>(ps + c * QR + k4);
                acc[k4] = fmaf(p4.x, x, acc[k4]);
                acc[k4 + 1] = fmaf(p4.y, x, acc[k4 + 1]);
                acc[k4 + 2] = fmaf(p4.z, x, acc[k4 + 2]);
                acc[k4 + 3] = fmaf(p4.w, x, acc[k4 + 3]);
            }
        }
        tcur = tnext;
    }
    // ---- this CTA's partial (max, num, den) per query row; num summed over the RS row groups
    static_assert(RS > 1, "D <= 128");
    float *rsum = sm + L::kR;
#pragma unroll
    for (int k = 0; k < QR; ++k) rsum[(rg * QR + k) * D + col] = acc[k];
    __syncthreads();
    float *pbase = part + (((int64_t)u * qz + z) * splits + split) * QR * PW;
    if (g == 0) pbase[q * PW] = mrun;
    if (tid < QR) pbase[tid * PW + 1 + D] = dens[tid];
    for (int e = tid; e < QR * D; e += kDecT) {
        const int qq = e / D, cc = e % D;
        float v = 0.f;
#pragma unroll
        for (int k = 0; k < RS; ++k) v += rsum[(k * QR + qq) * D + cc];
        pbase[qq * PW + 1 + cc] = v;
    }
    // merge: the last CTA of (unit, query chunk) combines the partials (also when splits = 1)
    __shared__ unsigned s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned t = splits > 1 ? atomicAdd(tickets + (int64_t)u * qz + z, 1u) : 0u;
        s_last = (t == (unsigned)splits - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    constexpr int NCOL = (DC + TPR - 1) / TPR;
    const float *pu = part + (((int64_t)u * qz + z) * splits) * QR * PW;
    float M = -INFINITY;
    for (int s2 = g; s2 < splits; s2 += TPR) M = fmaxf(M, __ldcg(pu + ((int64_t)s2 * QR + q) * PW));
#pragma unroll
    for (int o = (TPR < 32 ? TPR : 32) / 2; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    if constexpr (WPR > 1) {
        if ((tid & 31) == 0) red[tid >> 5] = M;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < WPR; ++w) M = fmaxf(M, red[q * WPR + w]);
    }
    float o_[NCOL];
#pragma unroll
    for (int k = 0; k < NCOL; ++k) o_[k] = 0.f;
    if (M > -INFINITY) {
#pragma unroll 4
        for (int s2 = 0; s2 < splits; ++s2) {
            const float *pp = pu + ((int64_t)s2 * QR + q) * PW;
            const float ms = __ldcg(pp);
            const float f = ms > -INFINITY ? exp2f(ms - M) : 0.f;
#pragma unroll
            for (int k = 0; k < NCOL; ++k) {
                const int cc = g + TPR * k;
                if (cc < DC) o_[k] = fmaf(f, __ldcg(pp + 1 + cc), o_[k]);
            }
        }
    }
    if (splits > 1 && tid == 0) tickets[(int64_t)u * qz + z] = 0u;  // reusable without a reset launch
    // den = column D, owned by thread g = D % TPR as o_[D / TPR]
    __syncthreads();
    if (g == D % TPR) dens[q] = o_[D / TPR];
    __syncthreads();
    if (q >= nq) return;
    const float den = dens[q];
    T *orow = O + (qoff + t0 + q) * D;
#pragma unroll
    for (int k = 0; k < NCOL; ++k) {
        const int cc = g + TPR * k;
        if (cc < D) {
            float o = den > 0.f ? o_[k] / den : 0.f;
            if (clip) o = fminf(fmaxf(o, to_f32(vmin[(int64_t)u * D + cc])), to_f32(vmax[(int64_t)u * D + cc]));
            orow[cc] = from_f32<T>(o);
        }
    }
}

// Query rows per CTA: 4 when one CTA covers the unit's whole query group (a decode token of a
// 4-head GQA group), else 16.
inline int decode_qr(const Dims &D) { return (int64_t)D.group() * D.m <= 4 ? 4 : kDecQmax; }

// CTAs per (unit, query chunk): about two per SM over the whole grid, at most one per tile.
int decode_splits(const Dims &D) {
    const int64_t ntiles = std::max<int64_t>(1, (D.r + kDecC - 1) / kDecC);
    const int64_t qz = ((int64_t)D.group() * D.m + decode_qr(D) - 1) / decode_qr(D);
    const int64_t want = (2 * 148 + D.units() * qz - 1) / (D.units() * qz);
    return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, want));
}

template <typename T, int D, int QR>
int launch_decode_tdq(const Dims &Dm, const void *Q, const void *KS, const float *X, const void *VC, const float *WC,
                      const int32_t *r_eff, const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws,
                      cudaStream_t st) {
    using L = DecSmem<D, QR>;
    const int splits = decode_splits(Dm);
    const int qz = (int)(((int64_t)Dm.group() * Dm.m + QR - 1) / QR);
    float *part = static_cast<float *>(ws);
    unsigned *tickets = reinterpret_cast<unsigned *>(
        static_cast<char *>(ws) + (size_t)Dm.units() * qz * splits * QR * (D + 2) * sizeof(float));
    if (splits > 1 && cudaMemsetAsync(tickets, 0, (size_t)Dm.units() * qz * sizeof(unsigned), st) != cudaSuccess)
        return -1;
    auto kern = VC ? attend_decode_kernel<T, D, QR, true> : attend_decode_kernel<T, D, QR, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::kBytes);
    kern<<<dim3(splits, Dm.units(), qz), kDecT, L::kBytes, st>>>(
        static_cast<const T *>(Q), static_cast<const T *>(KS), X, static_cast<const T *>(VC), WC, r_eff,
        static_cast<const T *>(vmin),
        static_cast<const T *>(vmax), Dm.m, Dm.r, Dm.group(), Dm.hq, Dm.hkv, (float)(beta * 1.4426950408889634), clip,
        static_cast<T *>(O), part, tickets);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T, int D>
int launch_decode_td(const Dims &Dm, const void *Q, const void *KS, const float *X, const void *VC, const float *WC,
                     const int32_t *r_eff, const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws,
                     cudaStream_t st) {
    if (decode_qr(Dm) == 4)
        return launch_decode_tdq<T, D, 4>(Dm, Q, KS, X, VC, WC, r_eff, vmin, vmax, beta, clip, O, ws, st);
    return launch_decode_tdq<T, D, kDecQmax>(Dm, Q, KS, X, VC, WC, r_eff, vmin, vmax, beta, clip, O, ws, st);
}

template <typename T>
int launch_decode_t(const Dims &Dm, const void *Q, const void *KS, const float *X, const void *VC, const float *WC,
                    const int32_t *r_eff, const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws,
                    cudaStream_t st) {
    switch (Dm.d) {
        case 16: return launch_decode_td<T, 16>(Dm, Q, KS, X, VC, WC, r_eff, vmin, vmax, beta, clip, O, ws, st);
        case 32: return launch_decode_td<T, 32>(Dm, Q, KS, X, VC, WC, r_eff, vmin, vmax, beta, clip, O, ws, st);
        case 64: return launch_decode_td<T, 64>(Dm, Q, KS, X, VC, WC, r_eff, vmin, vmax, beta, clip, O, ws, st);
        case 128: return launch_decode_td<T, 128>(Dm, Q, KS, X, VC, WC, r_eff, vmin, vmax, beta, clip, O, ws, st);
    }
    return -1;
}

// (VC, WC) -> X = [V_S, w] fp32 rows (the general attend over a compact KV cache, m > 16)
template <typename T>
__global__ void vw_to_x_kernel(const T *__restrict__ VC, const float *__restrict__ WC, int64_t rows, int d,
                               float *__restrict__ X) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * (d + 1);
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / (d + 1);
        const int c = (int)(e - row * (d + 1));
        X[e] = c < d ? to_f32(VC[row * d + c]) : WC[row];
    }
}

}  // namespace

size_t attend_decode_ws_bytes(const Dims &D) {
    const int64_t splits = decode_splits(D), QR = decode_qr(D);
    const int64_t qz = ((int64_t)D.group() * D.m + QR - 1) / QR;
    return (size_t)D.units() * qz * splits * QR * (D.d + 2) * sizeof(float) + (size_t)D.units() * qz * 4 + 256;
}

int launch_attend_decode(const Dims &D, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                         const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws,
                         cudaStream_t st) {
    if (D.m == 0) return 0;
    if (!ws) return -1;
    if (D.dtype == 0) return launch_decode_t<float>(D, Q, KS, X, nullptr, nullptr, r_eff, vmin, vmax, beta, clip, O, ws, st);
    return launch_decode_t<__nv_bfloat16>(D, Q, KS, X, nullptr, nullptr, r_eff, vmin, vmax, beta, clip, O, ws, st);
}

int launch_attend_decode_vw(const Dims &D, const void *Q, const void *KC, const void *VC, const float *WC,
                            const int32_t *c_eff, const void *vmin, const void *vmax, double beta, int clip, void *O,
                            void *ws, cudaStream_t st) {
    if (D.m == 0) return 0;
    if (!ws) return -1;
    if (D.dtype == 0)
        return launch_decode_t<float>(D, Q, KC, nullptr, VC, WC, c_eff, vmin, vmax, beta, clip, O, ws, st);
    return launch_decode_t<__nv_bfloat16>(D, Q, KC, nullptr, VC, WC, c_eff, vmin, vmax, beta, clip, O, ws, st);
}

int launch_vw_to_x(const Dims &D, const void *VC, const float *WC, float *X, cudaStream_t st) {
    const int64_t rows = (int64_t)D.units() * D.r;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 148, ceil_div(rows * (D.d + 1), 256)));
    if (D.dtype == 0)
        vw_to_x_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float *>(VC), WC, rows, D.d, X);
    else
        vw_to_x_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16 *>(VC), WC, rows, D.d, X);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_kv_assemble(const Dims &D, const void *K, const void *V, int kf, int kl, int R, const void *KS,
                       const float *X, const int32_t *Smid, const int32_t *reff_mid, void *KC, void *VC, float *WC,
                       int32_t *c_eff, int32_t *S_out, cudaStream_t st) {
    const int C = kf + kl + R;
    dim3 g((unsigned)std::max(1, (C + 7) / 8), D.units());
    if (D.dtype == 0)
        kv_assemble_kernel<float><<<g, 256, 0, st>>>(static_cast<const float *>(K), static_cast<const float *>(V), D.n,
                                                     D.d, kf, kl, R, static_cast<const float *>(KS), X, Smid, reff_mid,
                                                     static_cast<float *>(KC), static_cast<float *>(VC), WC, c_eff,
                                                     S_out);
    else
        kv_assemble_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(
            static_cast<const __nv_bfloat16 *>(K), static_cast<const __nv_bfloat16 *>(V), D.n, D.d, kf, kl, R,
            static_cast<const __nv_bfloat16 *>(KS), X, Smid, reff_mid, static_cast<__nv_bfloat16 *>(KC),
            static_cast<__nv_bfloat16 *>(VC), WC, c_eff, S_out);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace wc
