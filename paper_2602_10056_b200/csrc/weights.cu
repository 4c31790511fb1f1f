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

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace wc {

namespace {

constexpr int kWT = 256;  // threads
constexpr int kTA = 32;   // coreset rows per CTA
constexpr int kTL = 32;   // keys per smem tile

template <typename T, int D>
__global__ void __launch_bounds__(kWT) weights_partial_kernel(const T *__restrict__ K, const T *__restrict__ V,
                                                              const int32_t *__restrict__ S,
                                                              const T *__restrict__ KSin,
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
    const double *st = stats + (int64_t)u * (kStatsHead + D);
    const float g = (float)st[1], mstar = (float)st[2];
    for (int j = tid; j < D; j += kWT) kb[j] = st[kStatsHead + j];
    __syncthreads();
    const T *Ku = K + (int64_t)u * n * D;
    const T *Vu = V + (int64_t)u * n * D;
    for (int e = tid; e < kTA * D; e += kWT) {
        const int a = e / D, j = e % D;
        float v = 0.f;
        if (a0 + a < re) {
            const T *ksrow = KSin ? KSin + ((int64_t)u * r + a0 + a) * D : Ku + (int64_t)S[(int64_t)u * r + a0 + a] * D;
            v = (float)(to_f64(ksrow[j]) - kb[j]);
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

// Reduce split partials (fixed order, fp64) and solve L L^T X = Y~ for 8 RHS columns per CTA
// (256 threads: thread t owns panel row t/8 and column t%8).  Blocked in 32-row panels so the
// sequential part only touches a 32 x 32 diagonal block held in shared memory:
//   forward  (L Z = Y):   z_P -= L[P, 0:p0] z_{0:p0}  (parallel), then solve the panel's block
//   backward (L^T X = Z): x_P -= L[pe:q, P]^T x_{pe:q} (parallel, reads rows of L), then the block
// Y~ = sum over n-splits of the fp32 partials, in fixed split order, in fp64.
template <int D>
__global__ void __launch_bounds__(256) weights_reduce_kernel(const float *__restrict__ Ypart,
                                                             const int32_t *__restrict__ r_eff, int r, int splits,
                                                             double *__restrict__ Y) {
    constexpr int DC = D + 1;
    const int u = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (a, c) flattened
    if (e >= (int64_t)r * DC) return;
    const int a = (int)(e / DC);
    double y = 0.0;
    if (a < r_eff[u]) {
        const float *src = Ypart + (int64_t)u * splits * r * DC + e;
#pragma unroll 8
        for (int sp = 0; sp < splits; ++sp) y += (double)__ldg(src + (int64_t)sp * r * DC);
    }
    Y[(int64_t)u * r * DC + e] = y;
}

template <int D>
__global__ void __launch_bounds__(256) weights_solve_kernel(const double *__restrict__ Y,
                                                            const double *__restrict__ L,
                                                            const int32_t *__restrict__ r_eff, int r,
                                                            float *__restrict__ X) {
    constexpr int DC = D + 1;
    constexpr int PB = 32;
    constexpr int CB = 64;          // L columns (forward) / rows (backward) staged per block
    extern __shared__ double zs[];  // z[r][8]
    __shared__ double Ld[PB][PB + 1];
    __shared__ double Lb[PB][CB + 1];  // staged block of L
    const int u = blockIdx.y, tid = threadIdx.x;
    const int w = warp_index(), lane = tid & 31;
    const int cbase = blockIdx.x * 8;
    const int q = r_eff[u];
    const double *Lu = L + (int64_t)u * r * r;
    float *Xu = X + (int64_t)u * r * DC;
    for (int e = tid; e < q * 8; e += 256) {
        const int a = e / 8, cc = e % 8, col = cbase + cc;
        zs[a * 8 + cc] = col < DC ? Y[((int64_t)u * r + a) * DC + col] : 0.0;
    }
    __syncthreads();
    const int pr = tid / 8, pc = tid % 8;  // panel row, column
    // ---- forward substitution
    for (int p0 = 0; p0 < q; p0 += PB) {
        const int nb = min(PB, q - p0);
        double acc = (pr < nb) ? zs[(p0 + pr) * 8 + pc] : 0.0;
        for (int b0 = 0; b0 < p0; b0 += CB) {  // z_P -= L[P, b0:b0+CB] z[b0:b0+CB], block staged in smem
            const int nbk = min(CB, p0 - b0);
            __syncthreads();
            for (int e = tid; e < nb * CB; e += 256) {
                const int rr = e / CB, cc2 = e % CB;
                Lb[rr][cc2] = cc2 < nbk ? Lu[(int64_t)(p0 + rr) * r + b0 + cc2] : 0.0;
            }
            __syncthreads();
            if (pr < nb)
#pragma unroll 8
                for (int b = 0; b < nbk; ++b) acc = fma(-Lb[pr][b], zs[(b0 + b) * 8 + pc], acc);
        }
        if (pr < nb) zs[(p0 + pr) * 8 + pc] = acc;
        for (int e = tid; e < nb * nb; e += 256) Ld[e / nb][e % nb] = Lu[(int64_t)(p0 + e / nb) * r + p0 + e % nb];
        __syncthreads();
        if (w < 8) {  // warp w solves column w of the panel block; lane i owns row p0 + i
            double zi = lane < nb ? zs[(p0 + lane) * 8 + w] : 0.0;
            double lrow[PB];  // this lane's row of the diagonal block, in registers
#pragma unroll
            for (int j = 0; j < PB; ++j) lrow[j] = (lane < nb && j < nb) ? Ld[lane][j] : 0.0;
            const double inv = lane < nb ? 1.0 / Ld[lane][lane] : 0.0;
#pragma unroll
            for (int j = 0; j < PB; ++j) {
                if (j < nb) {
                    const double zj = __shfl_sync(0xffffffffu, zi * inv, j);
                    if (lane == j) zi = zj;
                    else if (lane > j) zi = fma(-lrow[j], zj, zi);
                }
            }
            if (lane < nb) zs[(p0 + lane) * 8 + w] = zi;
        }
        __syncthreads();
    }
    // ---- backward substitution (upper-triangular L^T)
    const int npan = (q + PB - 1) / PB;
    for (int pi = npan - 1; pi >= 0; --pi) {
        const int p0 = pi * PB, nb = min(PB, q - p0), pe = p0 + nb;
        double acc = (pr < nb) ? zs[(p0 + pr) * 8 + pc] : 0.0;
        for (int b0 = pe; b0 < q; b0 += CB) {  // x_P -= L[b0:b0+CB, P]^T x[b0:b0+CB], staged transposed
            const int nbk = min(CB, q - b0);
            __syncthreads();
            for (int e = tid; e < CB * PB; e += 256) {
                const int bb = e / PB, cc2 = e % PB;  // row b0 + bb, column p0 + cc2 (coalesced)
                Lb[cc2][bb] = (bb < nbk && cc2 < nb) ? Lu[(int64_t)(b0 + bb) * r + p0 + cc2] : 0.0;
            }
            __syncthreads();
            if (pr < nb)
#pragma unroll 8
                for (int b = 0; b < nbk; ++b) acc = fma(-Lb[pr][b], zs[(b0 + b) * 8 + pc], acc);
        }
        if (pr < nb) zs[(p0 + pr) * 8 + pc] = acc;
        for (int e = tid; e < nb * nb; e += 256) Ld[e / nb][e % nb] = Lu[(int64_t)(p0 + e / nb) * r + p0 + e % nb];
        __syncthreads();
        if (w < 8) {
            double zi = lane < nb ? zs[(p0 + lane) * 8 + w] : 0.0;
            double lcol[PB];  // column `lane` of the diagonal block (row j, col lane), in registers
#pragma unroll
            for (int j = 0; j < PB; ++j) lcol[j] = (lane < nb && j < nb) ? Ld[j][lane] : 0.0;
            const double inv = lane < nb ? 1.0 / Ld[lane][lane] : 0.0;
#pragma unroll
            for (int j = PB - 1; j >= 0; --j) {
                if (j < nb) {
                    const double xj = __shfl_sync(0xffffffffu, zi * inv, j);
                    if (lane == j) zi = xj;
                    else if (lane < j) zi = fma(-lcol[j], xj, zi);
                }
            }
            if (lane < nb) zs[(p0 + lane) * 8 + w] = zi;
        }
        __syncthreads();
    }
    for (int e = tid; e < r * 8; e += 256) {
        const int a = e / 8, cc = e % 8, col = cbase + cc;
        if (col < DC) Xu[(int64_t)a * DC + col] = a < q ? (float)zs[a * 8 + cc] : 0.f;
    }
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

// =====================================================================================
// tcgen05 path for A3 (bf16, d in {64, 128}).  CTA = (n-split, 128 coreset rows, unit), 128
// threads; thread a owns coreset row a0 + a (= TMEM lane a).  Per slice of 128 keys:
//   GEMM1  S[128 x 128] = K_S . K_slice^T  (raw bf16 keys, exact products, fp32 accumulation)
//   P = exp(g S + alpha_a + gamma_l)  with alpha_a = g(|kbar|^2 - <k_a,kbar>) - mstar and
//       gamma_l = -g <k_l, kbar>  (= exp(g <k_a - kbar, k_l - kbar> - mstar), no rounding of
//       centred keys to bf16);  rowsum_a += P;  P -> bf16 smem
//   GEMM2  O[128 x d] += P . V_slice       (accumulated in TMEM across the CTA's slices)
// and the partial Y~[a][0:d] = O, Y~[a][d] = rowsum go to Ypart (summed in fp64 by the solve).
// =====================================================================================
constexpr int kWTc = 256;  // 8 warps: warps w and w+4 share TMEM lane quadrant w%4 (column halves)

__device__ __forceinline__ float ex2_approx_w(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int D> struct WtSmem {
    static constexpr int kA = 128 * D * 2, kB = 128 * D * 2, kP = 128 * 128 * 2, kV = D * 128 * 2;
    static constexpr int kOffA = 0, kOffB = kA, kOffP = kOffB + kB, kOffV = kOffP + kP;
    static constexpr int kOffG = kOffV + kV, kOffKb = kOffG + 128 * 4, kOffX = kOffKb + D * 4;
    static constexpr int kOffBar = kOffX + 2 * 128 * 4, kOffTb = kOffBar + 8;
    static constexpr int kTotal = kOffTb + 8;
};

template <int D>
__global__ void __launch_bounds__(kWTc, 1)
    weights_tc_kernel(const __nv_bfloat16 *__restrict__ K, const __nv_bfloat16 *__restrict__ V,
                      const int32_t *__restrict__ S, const __nv_bfloat16 *__restrict__ KSin,
                      const int32_t *__restrict__ r_eff,
                      const double *__restrict__ stats, int64_t n, int r, int splits, float *__restrict__ Ypart) {
    using L = WtSmem<D>;
    constexpr int DC = D + 1;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;  // offset 0 of the CTA's shared window (no static smem): 1024-aligned
    if (smem_u32(sm) & 1023u) __trap();
    unsigned char *sA = sm + L::kOffA, *sB = sm + L::kOffB, *sP = sm + L::kOffP, *sV = sm + L::kOffV;
    float *sG = reinterpret_cast<float *>(sm + L::kOffG);    // log2e * gamma_l of the slice [128]
    float *sKb = reinterpret_cast<float *>(sm + L::kOffKb);  // kbar (fp32) [D]
    float *xch = reinterpret_cast<float *>(sm + L::kOffX);   // [2][128] row-sum exchange
    uint64_t &bar = *reinterpret_cast<uint64_t *>(sm + L::kOffBar);
    uint32_t &tbase = *reinterpret_cast<uint32_t *>(sm + L::kOffTb);
    const int tid = threadIdx.x, w = tid >> 5, row = tid & 127, half = tid >> 7;
    const int split = blockIdx.x, a0 = blockIdx.y * 128, u = blockIdx.z;
    const int re = r_eff[u];
    if (a0 >= re) return;  // uniform per CTA
    const __nv_bfloat16 *Ku = K + (int64_t)u * n * D;
    const __nv_bfloat16 *Vu = V + (int64_t)u * n * D;
    const double *st = stats + (int64_t)u * (kStatsHead + D);
    const double g = st[1], mstar = st[2];
    constexpr int CPR = D / 8;
    constexpr float kLog2e = 1.4426950408889634f;

    if (w == 0) umma::tmem_alloc(&tbase, 256);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    for (int j = tid; j < D; j += kWTc) sKb[j] = (float)st[kStatsHead + j];
    // coreset rows (raw keys) -> A operand
    for (int e = tid; e < 128 * CPR; e += kWTc) {
        const int rw = e / CPR, cc = e % CPR;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (a0 + rw < re) {
            const __nv_bfloat16 *ksrow = KSin ? KSin + ((int64_t)u * r + a0 + rw) * D
                                              : Ku + (int64_t)S[(int64_t)u * r + a0 + rw] * D;
            v = __ldg(reinterpret_cast<const uint4 *>(ksrow) + cc);
        }
        *reinterpret_cast<uint4 *>(sA + umma::sw128_offset(rw, cc * 8, 128)) = v;
    }
    // alpha_a = g(|kbar|^2 - <k_a, kbar>) - mstar in fp64, scaled by log2(e) for ex2
    float alpha2 = 0.f;
    const bool row_ok = a0 + row < re;
    if (row_ok) {
        const __nv_bfloat16 *ksrow = KSin ? KSin + ((int64_t)u * r + a0 + row) * D
                                          : Ku + (int64_t)S[(int64_t)u * r + a0 + row] * D;
        double kk = 0.0, bb = 0.0;
        for (int j = 0; j < D; ++j) {
            const double kbj = st[kStatsHead + j];
            kk = fma(to_f64(ksrow[j]), kbj, kk);
            bb = fma(kbj, kbj, bb);
        }
        alpha2 = (float)((g * (bb - kk) - mstar) * 1.4426950408889634);
    }
    const float g2 = (float)(g * 1.4426950408889634);
    const int64_t rows = ceil_div(n, splits);
    const int64_t lo = (int64_t)split * rows, hi = std::min<int64_t>(n, lo + rows);
    const uint32_t tS = tbase, tO = tbase + 128, lane_off = (uint32_t)((w & 3) * 32) << 16;
    uint32_t phase = 0;
    float rowsum = 0.f;
    bool first = true;
    for (int64_t l0 = lo; l0 < hi; l0 += 128) {
        // keys of the slice -> B operand of GEMM1 (K-major, swizzled); V^T -> B operand of GEMM2
        for (int e = tid; e < 128 * CPR; e += kWTc) {
            const int rw = e / CPR, cc = e % CPR;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (l0 + rw < hi) v = __ldg(reinterpret_cast<const uint4 *>(Ku + (l0 + rw) * D) + cc);
            *reinterpret_cast<uint4 *>(sB + umma::sw128_offset(rw, cc * 8, 128)) = v;
        }
        for (int e = tid; e < 128 * CPR; e += kWTc) {
            const int rw = e / CPR, cc = e % CPR;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (l0 + rw < hi) v = __ldg(reinterpret_cast<const uint4 *>(Vu + (l0 + rw) * D) + cc);
            const __nv_bfloat16 *pv = reinterpret_cast<const __nv_bfloat16 *>(&v);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                *reinterpret_cast<__nv_bfloat16 *>(sV + umma::sw128_offset(cc * 8 + q, rw, D)) = pv[q];
        }
        if (tid < 128) {  // log2e * gamma_l = -log2e g <k_l, kbar> for key l0 + tid
            const int64_t l = l0 + tid;
            float gm = 0.f;
            if (l < hi) {
                const uint4 *kr = reinterpret_cast<const uint4 *>(Ku + l * D);
#pragma unroll 4
                for (int cc = 0; cc < CPR; ++cc) {
                    const uint4 v = __ldg(kr + cc);
                    const __nv_bfloat16 *pv = reinterpret_cast<const __nv_bfloat16 *>(&v);
#pragma unroll
                    for (int q = 0; q < 8; ++q) gm = fmaf(__bfloat162float(pv[q]), sKb[cc * 8 + q], gm);
                }
            }
            sG[tid] = -g2 * gm;
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        umma::fence_after_sync();
        if (tid == 0) {
            umma::gemm_128xNxK(tS, smem_u32(sA), smem_u32(sB), 128, D, false);
            umma::commit(&bar);
        }
        mbar_wait(&bar, phase);
        phase ^= 1u;
        umma::fence_after_sync();
        // P = exp2(g2 S + alpha2 + gamma2) for 64 columns per thread (its half), bf16 -> smem
        const int nl = (int)std::min<int64_t>(128, hi - l0);
        {
            const int cbase = half * 64;
            float v[64];
            umma::ld32(tS + lane_off + cbase, v);
            umma::ld32(tS + lane_off + cbase + 32, v + 32);
            float rs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int g8 = 0; g8 < 8; ++g8) {
                uint32_t pk[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int cl = g8 * 8 + 2 * i, l = cbase + cl;
                    const float p0 = (row_ok && l < nl) ? ex2_approx_w(fmaf(g2, v[cl], alpha2 + sG[l])) : 0.f;
                    const float p1 = (row_ok && l + 1 < nl) ? ex2_approx_w(fmaf(g2, v[cl + 1], alpha2 + sG[l + 1])) : 0.f;
                    const __nv_bfloat162 pb = __floats2bfloat162_rn(p0, p1);
                    rs[i] += __bfloat162float(pb.x) + __bfloat162float(pb.y);
                    pk[i] = *reinterpret_cast<const uint32_t *>(&pb);
                }
                *reinterpret_cast<uint4 *>(sP + umma::sw128_offset(row, cbase + g8 * 8, 128)) =
                    make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
            rowsum += (rs[0] + rs[1]) + (rs[2] + rs[3]);
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        umma::fence_after_sync();
        if (tid == 0) {
            umma::gemm_128xNxK(tO, smem_u32(sP), smem_u32(sV), D, 128, !first);
            umma::commit(&bar);
        }
        mbar_wait(&bar, phase);  // smem (sB, sV, sP) reusable and O updated
        phase ^= 1u;
        umma::fence_after_sync();
        first = false;
    }
    xch[half * 128 + row] = rowsum;
    __syncthreads();
    float *out = Ypart + (((int64_t)u * splits + split) * r + a0 + row) * DC;
    if (first) {  // empty key range: zero partial
        if (row_ok && half == 0)
            for (int c = 0; c < DC; ++c) out[c] = 0.f;
    } else {
        constexpr int HD = D / 2;
#pragma unroll
        for (int c0 = 0; c0 < HD; c0 += 32) {
            float v[32];
            umma::ld32(tO + lane_off + half * HD + c0, v);
            if (row_ok) {
#pragma unroll
                for (int i = 0; i < 32; ++i) out[half * HD + c0 + i] = v[i];
            }
        }
        if (row_ok && half == 0) out[D] = xch[row] + xch[128 + row];
    }
    umma::fence_before_sync();
    __syncthreads();
    if (w == 0) umma::tmem_dealloc(tbase, 256);
}

// A3: fp32 split partials of Y~ (tensor-core kernel for bf16 and d in {64, 128}), then their
// fixed-order fp64 sum into Yfull.  Coreset rows come from K[S] or, if KSin != nullptr, densely.
template <typename T, int D>
int launch_partial_td(const Dims &Dm, const void *K, const void *V, const int32_t *S, const void *KSin,
                      const int32_t *r_eff, const double *stats, float *Ypart, double **Yfull_out, cudaStream_t st) {
    const int units = Dm.units();
    const int splits = weights_num_splits(Dm);
    static const char *mode = std::getenv("WC_WEIGHTS");  // "cuda": CUDA-core kernel (A/B tests)
    bool done = false;
    if constexpr (sizeof(T) == 2 && (D == 64 || D == 128)) {
        if (!(mode && std::strcmp(mode, "cuda") == 0)) {
            const int smem_tc = WtSmem<D>::kTotal;  // A, B, V^T, P, gamma, kbar, exchange, barrier
            auto kt = weights_tc_kernel<D>;
            cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc);
            dim3 gt(splits, (Dm.r + 127) / 128, units);
            kt<<<gt, kWTc, smem_tc, st>>>(static_cast<const __nv_bfloat16 *>(K), static_cast<const __nv_bfloat16 *>(V),
                                          S, static_cast<const __nv_bfloat16 *>(KSin), r_eff, stats, Dm.n, Dm.r,
                                          splits, Ypart);
            done = true;
        }
    }
    if (!done) {
        dim3 g1(splits, (Dm.r + kTA - 1) / kTA, units);
        const size_t smem1 = D * sizeof(double) + (size_t)(kTA + 2 * kTL) * (D + 1) * sizeof(float) +
                             (size_t)kTA * (kTL + 1) * sizeof(float);
        auto pk = weights_partial_kernel<T, D>;
        cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
        pk<<<g1, kWT, smem1, st>>>(static_cast<const T *>(K), static_cast<const T *>(V), S,
                                   static_cast<const T *>(KSin), r_eff, stats, Dm.n, Dm.r, splits, Ypart);
    }
    const size_t parts = (size_t)units * splits * Dm.r * (D + 1);
    double *Yfull = *Yfull_out ? *Yfull_out : reinterpret_cast<double *>(Ypart + ((parts + 1) & ~size_t(1)));
    const int64_t cnt = (int64_t)Dm.r * (D + 1);
    dim3 gr((unsigned)ceil_div(cnt, 256), units);
    weights_reduce_kernel<D><<<gr, 256, 0, st>>>(Ypart, r_eff, Dm.r, splits, Yfull);
    *Yfull_out = Yfull;
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

template <int D>
int launch_solve_d(const Dims &Dm, const double *Yfull, const double *L, const int32_t *r_eff, float *X,
                   cudaStream_t st) {
    const size_t smem = (size_t)8 * Dm.r * sizeof(double);
    auto sk = weights_solve_kernel<D>;
    // the kernel also holds ~25 KB of static smem: always raise the dynamic limit
    cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 g2((D + 1 + 7) / 8, Dm.units());
    sk<<<g2, 256, smem, st>>>(Yfull, L, r_eff, Dm.r, X);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T, int D>
int launch_weights_td(const Dims &Dm, const void *K, const void *V, const int32_t *S, const int32_t *r_eff,
                      const double *L, const double *stats, float *Ypart, void *KS, float *X, cudaStream_t st) {
    double *Yfull = nullptr;
    const int k1 = launch_partial_td<T, D>(Dm, K, V, S, nullptr, r_eff, stats, Ypart, &Yfull, st);
    if (k1 < 0) return -1;
    const int k2 = launch_solve_d<D>(Dm, Yfull, L, r_eff, X, st);
    if (k2 < 0) return -1;
    dim3 g3(Dm.r, Dm.units());
    gather_ks_kernel<T, D><<<g3, 128, 0, st>>>(static_cast<const T *>(K), S, r_eff, Dm.n, Dm.r,
                                               static_cast<T *>(KS));
    return cudaPeekAtLastError() == cudaSuccess ? k1 + k2 + 1 : -1;
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

int launch_weights_partial_ks(const Dims &D, const void *K, const void *V, const void *KSin, const int32_t *r_eff,
                              const double *stats, float *Ypart, double *Yfull, cudaStream_t st) {
    double *Y = Yfull;
#define WC_PKS(TT, DD) return launch_partial_td<TT, DD>(D, K, V, nullptr, KSin, r_eff, stats, Ypart, &Y, st)
    if (D.dtype == 0) {
        switch (D.d) { case 16: WC_PKS(float, 16); case 32: WC_PKS(float, 32); case 64: WC_PKS(float, 64); case 128: WC_PKS(float, 128); }
    } else {
        switch (D.d) { case 16: WC_PKS(__nv_bfloat16, 16); case 32: WC_PKS(__nv_bfloat16, 32); case 64: WC_PKS(__nv_bfloat16, 64); case 128: WC_PKS(__nv_bfloat16, 128); }
    }
#undef WC_PKS
    return -1;
}

int launch_weights_solve(const Dims &D, const double *Yfull, const double *L, const int32_t *r_eff, float *X,
                         cudaStream_t st) {
    switch (D.d) {
        case 16: return launch_solve_d<16>(D, Yfull, L, r_eff, X, st);
        case 32: return launch_solve_d<32>(D, Yfull, L, r_eff, X, st);
        case 64: return launch_solve_d<64>(D, Yfull, L, r_eff, X, st);
        case 128: return launch_solve_d<128>(D, Yfull, L, r_eff, X, st);
    }
    return -1;
}

int weights_num_splits(const Dims &D) {
    const bool tc = D.dtype == 1 && (D.d == 64 || D.d == 128);
    const int rt = tc ? 128 : kTA;  // coreset rows per CTA (tensor-core / CUDA-core kernel)
    const int64_t tiles = (int64_t)D.units() * ((D.r + rt - 1) / rt);
    const int64_t want = std::max<int64_t>(1, ((tc ? 148 : 148 * 4) + tiles - 1) / tiles);
    const int64_t by_n = std::max<int64_t>(1, ceil_div(D.n, 256));
    return (int)std::min<int64_t>(std::min<int64_t>(want, by_n), 512);
}

int launch_weights(const Dims &D, const void *K, const void *V, const int32_t *S, const int32_t *r_eff,
                   const double *L, const double *stats, float *Ypart, void *KS, float *X, cudaStream_t st) {
    if (D.dtype == 0) return launch_weights_t<float>(D, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
    return launch_weights_t<__nv_bfloat16>(D, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
}

}  // namespace wc
