// prologue.cu -- A0 of the hot path: per-unit recentring statistics and temperature.
//   kbar = row mean of K (Alg 2 "Recenter keys")
//   R_K  = max_l ||k_l - kbar||,  R_Q = max_i ||q_i|| over the unit's query group (Alg 4)
//   tau  = Eq. 7, g = beta/tau^2, mstar = g R_K^2 (reading Z10)
//   (vmin, vmax) = columnwise range of V (Alg 4)
// HBM-bound streaming passes (one over K, Q, V; one over K), fp64 accumulation.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace wc {

namespace {

constexpr int kPT = 256;  // threads per prologue block

// Pass 1: per (split p, unit u): column sums of K (fp64), column min/max of V, max ||q||^2.
// Each thread owns 8 consecutive columns (16/32-byte vector loads); CPR = d/8 threads per row.
template <typename T>
__global__ void __launch_bounds__(kPT) prologue_pass1(const T *__restrict__ Q, const T *__restrict__ K,
                                                      const T *__restrict__ V, int64_t n, int64_t mq, int d,
                                                      int P, int want_q, int want_v, double *colsum,
                                                      float *vmin, float *vmax, double *rq2,
                                                      int64_t q_unit_stride_rows, int32_t *fill_S, int64_t nS,
                                                      double *zero_L, int64_t nL) {
    pdl_wait();
    if (nS > 0 || nL > 0) {  // the selection's outputs: S <- -1, L <- 0 (grid-stride, all blocks)
        const int64_t nth = (int64_t)gridDim.x * gridDim.y * blockDim.x;
        const int64_t g0 = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
        for (int64_t e = g0; e < nS; e += nth) fill_S[e] = -1;
        for (int64_t e = g0; e < nL; e += nth) zero_L[e] = 0.0;
    }
    extern __shared__ double sm1[];
    const int p = blockIdx.x, u = blockIdx.y;
    const int CPR = d / 8, RG = kPT / CPR;
    const int rg = threadIdx.x / CPR, cj = threadIdx.x % CPR;
    const int64_t rows = ceil_div(n, P);
    const int64_t lo = (int64_t)p * rows, hi = min(n, lo + rows);
    const T *Ku = K + (int64_t)u * n * d;
    const T *Vu = V + (int64_t)u * n * d;
    double cs[8];
    float mn[8], mx[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { cs[k] = 0.0; mn[k] = 3.0e38f; mx[k] = -3.0e38f; }
    constexpr int U4 = 8;  // rows per thread in flight
    for (int64_t l0 = lo + rg; l0 < hi; l0 += (int64_t)U4 * RG) {
        Raw8<T> xk[U4], xv[U4];
#pragma unroll
        for (int q = 0; q < U4; ++q) {
            const int64_t l = l0 + (int64_t)q * RG;
            if (l < hi) {
                xk[q].load(Ku + l * d + 8 * cj);
                if (want_v) xv[q].load(Vu + l * d + 8 * cj);
            }
        }
#pragma unroll
        for (int q = 0; q < U4; ++q) {
            if (l0 + (int64_t)q * RG < hi) {  // rows in ascending order: fixed summation order
#pragma unroll
                for (int k = 0; k < 8; ++k) cs[k] += xk[q].at(k);
                if (want_v) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        mn[k] = fminf(mn[k], (float)xv[q].at(k));
                        mx[k] = fmaxf(mx[k], (float)xv[q].at(k));
                    }
                }
            }
        }
    }
    double *s_cs = sm1;                                    // [RG][d]
    float *s_lo = reinterpret_cast<float *>(sm1 + RG * d);  // [RG][d]
    float *s_hi = s_lo + RG * d;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        s_cs[rg * d + 8 * cj + k] = cs[k];
        s_lo[rg * d + 8 * cj + k] = mn[k];
        s_hi[rg * d + 8 * cj + k] = mx[k];
    }
    __syncthreads();
    if (threadIdx.x < d) {
        double t = 0.0;
        float a = 3.0e38f, b = -3.0e38f;
        for (int g2 = 0; g2 < RG; ++g2) {
            t += s_cs[g2 * d + threadIdx.x];
            a = fminf(a, s_lo[g2 * d + threadIdx.x]);
            b = fmaxf(b, s_hi[g2 * d + threadIdx.x]);
        }
        const int64_t o = ((int64_t)u * P + p) * d + threadIdx.x;
        colsum[o] = t;
        vmin[o] = a;
        vmax[o] = b;
    }
    if (want_q) {
        const int64_t qrows = ceil_div(mq, P);
        const int64_t qlo = (int64_t)p * qrows, qhi = min(mq, qlo + qrows);
        const T *Qu = Q + (int64_t)u * q_unit_stride_rows * d;
        double best = 0.0;
        for (int64_t i0 = qlo; i0 < qhi; i0 += (int64_t)U4 * RG) {
            Raw8<T> xq[U4];
#pragma unroll
            for (int q = 0; q < U4; ++q) {
                const int64_t i = i0 + (int64_t)q * RG + rg;
                if (i < qhi) xq[q].load(Qu + i * d + 8 * cj);
            }
#pragma unroll
            for (int q = 0; q < U4; ++q) {
                const int64_t i = i0 + (int64_t)q * RG + rg;
                double sq = 0.0;
                if (i < qhi) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) sq += xq[q].at(k) * xq[q].at(k);
                }
                for (int o = 1; o < CPR; o <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
                best = fmax(best, sq);
            }
        }
        __shared__ double scr[40];
        best = block_max(best, scr);
        if (threadIdx.x == 0) rq2[(int64_t)u * P + p] = best;
    }
}

// Finalise kbar (fixed-order sum over splits) and the value range.  One block per (unit, column j):
// thread t sums splits t, t + 256, ... (in order), then a fixed-shape shared-memory tree combines
// the 256 partials -- every column is reduced by its own block, with all its loads in flight.
template <typename T>
__global__ void __launch_bounds__(kPT) prologue_kbar(int64_t n, int d, int P, const double *colsum,
                                                     const float *vmin_p, const float *vmax_p, double *stats,
                                                     T *vmin, T *vmax, int no_recenter) {
    pdl_wait();
    __shared__ double s_t[kPT];
    __shared__ float s_a[kPT], s_b[kPT];
    const int u = blockIdx.x, j = blockIdx.y, tid = threadIdx.x, nt = blockDim.x;
    double t = 0.0;
    float a = 3.0e38f, b = -3.0e38f;
    for (int p = tid; p < P; p += nt) {
        const int64_t o = ((int64_t)u * P + p) * d + j;
        t += colsum[o];
        a = fminf(a, vmin_p[o]);
        b = fmaxf(b, vmax_p[o]);
    }
    s_t[tid] = t;
    s_a[tid] = a;
    s_b[tid] = b;
    __syncthreads();
    for (int h = nt / 2; h > 0; h >>= 1) {  // nt is a power of two
        if (tid < h) {
            s_t[tid] += s_t[tid + h];
            s_a[tid] = fminf(s_a[tid], s_a[tid + h]);
            s_b[tid] = fmaxf(s_b[tid], s_b[tid + h]);
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (stats) stats[(int64_t)u * (kStatsHead + d) + kStatsHead + j] = no_recenter ? 0.0 : s_t[0] / (double)n;
        if (vmin) {
            vmin[(int64_t)u * d + j] = from_f32<T>(s_a[0]);
            vmax[(int64_t)u * d + j] = from_f32<T>(s_b[0]);
        }
    }
}

// Few splits (many units): finalise kbar and the value range for 32 columns per block.  Block (u, column chunk of 32):
// 8 groups of 32 threads; group g sums splits p = g, g + 8, ... (unrolled), combined in group order.
template <typename T>
__global__ void __launch_bounds__(kPT) prologue_kbar_small(int64_t n, int d, int P, const double *colsum,
                                                     const float *vmin_p, const float *vmax_p, double *stats,
                                                     T *vmin, T *vmax, int no_recenter) {
    pdl_wait();
    __shared__ double s_t[kPT];
    __shared__ float s_a[kPT], s_b[kPT];
    const int u = blockIdx.x, g = threadIdx.x >> 5, j = blockIdx.y * 32 + (threadIdx.x & 31);
    double t = 0.0;
    float a = 3.0e38f, b = -3.0e38f;
    if (j < d) {
#pragma unroll 8
        for (int p = g; p < P; p += 8) {
            const int64_t o = ((int64_t)u * P + p) * d + j;
            t += colsum[o];
            a = fminf(a, vmin_p[o]);
            b = fmaxf(b, vmax_p[o]);
        }
    }
    s_t[threadIdx.x] = t;
    s_a[threadIdx.x] = a;
    s_b[threadIdx.x] = b;
    __syncthreads();
    if (threadIdx.x < 32 && j < d) {
        double tt = 0.0;
        float aa = 3.0e38f, bb = -3.0e38f;
        for (int gg = 0; gg < 8; ++gg) {
            tt += s_t[gg * 32 + threadIdx.x];
            aa = fminf(aa, s_a[gg * 32 + threadIdx.x]);
            bb = fmaxf(bb, s_b[gg * 32 + threadIdx.x]);
        }
        if (stats) stats[(int64_t)u * (kStatsHead + d) + kStatsHead + j] = no_recenter ? 0.0 : tt / (double)n;
        if (vmin) {
            vmin[(int64_t)u * d + j] = from_f32<T>(aa);
            vmax[(int64_t)u * d + j] = from_f32<T>(bb);
        }
    }
}

// threads of a kbar block: a power of two in [32, kPT] covering the split count
inline int kbar_threads(int P) {
    int t = 32;
    while (t < P && t < kPT) t <<= 1;
    return t;
}

// kbar / value-range finalisation: one block per column for many splits, 32 columns per block else
template <typename T>
void launch_kbar(const Dims &D, int P, const ProloguePartials &pp, double *stats, void *vmin, void *vmax,
                 cudaStream_t st, int no_recenter = 0) {
    if (P >= 64)
        launch_pdl(prologue_kbar<T>, dim3(D.units(), D.d), dim3(kbar_threads(P)), 0, st, D.n, D.d, P,
                   (const double *)pp.colsum, (const float *)pp.vmin, (const float *)pp.vmax, stats,
                   static_cast<T *>(vmin), static_cast<T *>(vmax), no_recenter);
    else
        prologue_kbar_small<T><<<dim3(D.units(), (D.d + 31) / 32), kPT, 0, st>>>(
            D.n, D.d, P, pp.colsum, pp.vmin, pp.vmax, stats, static_cast<T *>(vmin), static_cast<T *>(vmax),
            no_recenter);
}

// Pass 2: nrm2_l = ||k_l - kbar||^2 (fp64) and the split max.  CPR threads per key.
template <typename T>
__global__ void __launch_bounds__(kPT) prologue_pass2(const T *__restrict__ K, int64_t n, int d, int P,
                                                      const double *stats, double *nrm2, double *rk2) {
    pdl_wait();
    __shared__ double kb[128];
    __shared__ double scr[40];
    const int p = blockIdx.x, u = blockIdx.y;
    const int CPR = d / 8, RG = kPT / CPR;
    const int rg = threadIdx.x / CPR, cj = threadIdx.x % CPR;
    const double *st = stats + (int64_t)u * (kStatsHead + d);
    for (int j = threadIdx.x; j < d; j += kPT) kb[j] = st[kStatsHead + j];
    __syncthreads();
    const int64_t rows = ceil_div(n, P);
    const int64_t lo = (int64_t)p * rows, hi = min(n, lo + rows);
    const T *Ku = K + (int64_t)u * n * d;
    double kbr[8];  // this thread's 8 columns of kbar, kept in registers across its rows
#pragma unroll
    for (int k = 0; k < 8; ++k) kbr[k] = kb[8 * cj + k];
    double best = 0.0;
    constexpr int U4 = 8;  // rows per thread in flight
    for (int64_t l0 = lo; l0 < hi; l0 += (int64_t)U4 * RG) {
        Raw8<T> xk[U4];
#pragma unroll
        for (int q = 0; q < U4; ++q) {
            const int64_t l = l0 + (int64_t)q * RG + rg;
            if (l < hi) xk[q].load(Ku + l * d + 8 * cj);
        }
#pragma unroll
        for (int q = 0; q < U4; ++q) {
            const int64_t l = l0 + (int64_t)q * RG + rg;
            double sq = 0.0;
            if (l < hi) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double c = __dadd_rn(xk[q].at(k), -kbr[k]);
                    sq = __dadd_rn(sq, __dmul_rn(c, c));
                }
            }
            for (int o = 1; o < CPR; o <<= 1) sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
            if (l < hi && cj == 0) nrm2[(int64_t)u * n + l] = sq;
            best = fmax(best, sq);
        }
    }
    best = block_max(best, scr);
    if (threadIdx.x == 0) rk2[(int64_t)u * P + p] = best;
}

// tau (Eq. 7), g, mstar.  One thread per unit.
// One warp per unit: maxima over the P splits, then lane 0 evaluates Eq. 7.
__global__ void prologue_tau(int units, int64_t n, int d, int P, const double *rk2, const double *rq2,
                             double rq_given, double beta, double *stats, int tau_one) {
    pdl_wait();
    const int u = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (u >= units) return;
    double mk = 0.0, mq = 0.0;
    for (int p = lane; p < P; p += 32) {
        mk = fmax(mk, rk2[(int64_t)u * P + p]);
        if (rq_given < 0.0) mq = fmax(mq, rq2[(int64_t)u * P + p]);
    }
    mk = warp_max(mk);
    mq = warp_max(mq);
    if (lane != 0) return;
    const double rk = sqrt(mk);
    const double rq = rq_given >= 0.0 ? rq_given : sqrt(mq);
    double tau = 1.0;  // WC_TAU_ONE, or the R_Q R_K = 0 fallback (reading Z20)
    if (!tau_one && rq * rk > 0.0) {
        const double rho0 = sqrt(1.0 + exp(lambert_w0_dev(2.0 / (2.718281828459045 * 2.718281828459045)) + 2.0));
        const double b0 = log((double)n) / (beta * rq * rk) + 2.0;
        const double w = lambert_w0_dev(b0 / (2.0 * rho0));
        tau = sqrt((rk / rq) * b0 / (2.0 * w));
    }
    const double g = beta / (tau * tau);
    double *st = stats + (int64_t)u * (kStatsHead + d);
    st[0] = tau;
    st[1] = g;
    st[2] = g * rk * rk;
    st[3] = rk;
    st[4] = rq;
    for (int k = 5; k < kStatsHead; ++k) st[k] = 0.0;
}

template <typename T>
int launch_prologue_t(const Dims &D, const void *Q, const void *K, const void *V, double rq, double beta,
                      ProloguePartials pp, double *stats, double *nrm2, void *vmin, void *vmax, int pflags,
                      cudaStream_t st) {
    const int units = D.units();
    const int P = pp.P;
    const int RG = kPT / (D.d / 8);
    const size_t smem = (size_t)RG * D.d * (sizeof(double) + 2 * sizeof(float));
    const int want_q = (rq < 0.0 && Q != nullptr && D.m > 0) ? 1 : 0;
    const int want_v = (V != nullptr) ? 1 : 0;
    const int64_t mq = want_q ? (int64_t)D.group() * D.m : 0;
    dim3 grid(P, units);
    prologue_pass1<T><<<grid, kPT, smem, st>>>(static_cast<const T *>(Q), static_cast<const T *>(K),
                                               static_cast<const T *>(V ? V : K), D.n, mq, D.d, P, want_q,
                                               want_v, pp.colsum, pp.vmin, pp.vmax, pp.rq2,
                                               (int64_t)D.group() * D.m, pp.fill_S, pp.nS, pp.zero_L, pp.nL);
    launch_kbar<T>(D, P, pp, stats, want_v ? vmin : nullptr, want_v ? vmax : nullptr, st,
                   (pflags & kPfNoRecenter) ? 1 : 0);
    launch_pdl(prologue_pass2<T>, grid, dim3(kPT), 0, st, static_cast<const T *>(K), D.n, D.d, P,
               (const double *)stats, nrm2, pp.rk2);
    launch_pdl(prologue_tau, dim3((unsigned)ceil_div(units, 4)), dim3(128), 0, st, units, D.n, D.d, P,
               (const double *)pp.rk2, (const double *)pp.rq2,
               want_q ? -1.0 : (rq < 0.0 ? 0.0 : rq), beta, stats, (pflags & kPfTauOne) ? 1 : 0);
    return cudaPeekAtLastError() == cudaSuccess ? 4 : -1;
}

template <typename T>
int launch_vrange_t(const Dims &D, const void *V, ProloguePartials pp, void *vmin, void *vmax, cudaStream_t st) {
    const int units = D.units();
    const int RG = kPT / (D.d / 8);
    const size_t smem = (size_t)RG * D.d * (sizeof(double) + 2 * sizeof(float));
    dim3 grid(pp.P, units);
    prologue_pass1<T><<<grid, kPT, smem, st>>>(nullptr, static_cast<const T *>(V), static_cast<const T *>(V), D.n,
                                               0, D.d, pp.P, 0, 1, pp.colsum, pp.vmin, pp.vmax, pp.rq2, 0, nullptr, 0,
                                               nullptr, 0);
    launch_kbar<T>(D, pp.P, pp, nullptr, vmin, vmax, st);
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

}  // namespace

template <typename T>
int launch_pass1_t(const Dims &D, const void *Q, const void *K, const void *V, bool want_q, ProloguePartials pp,
                   cudaStream_t st) {
    const int RG = kPT / (D.d / 8);
    const size_t smem = (size_t)RG * D.d * (sizeof(double) + 2 * sizeof(float));
    const int64_t mq = want_q ? (int64_t)D.group() * D.m : 0;
    dim3 grid(pp.P, D.units());
    prologue_pass1<T><<<grid, kPT, smem, st>>>(static_cast<const T *>(Q), static_cast<const T *>(K),
                                               static_cast<const T *>(V), D.n, mq, D.d, pp.P, want_q ? 1 : 0, 1,
                                               pp.colsum, pp.vmin, pp.vmax, pp.rq2, (int64_t)D.group() * D.m, nullptr, 0,
                                               nullptr, 0);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}
template <typename T>
int launch_pass2_t(const Dims &D, const void *K, ProloguePartials pp, const double *stats, double *nrm2,
                   cudaStream_t st) {
    dim3 grid(pp.P, D.units());
    prologue_pass2<T><<<grid, kPT, 0, st>>>(static_cast<const T *>(K), D.n, D.d, pp.P, stats, nrm2, pp.rk2);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_prologue_pass1(const Dims &D, const void *Q, const void *K, const void *V, bool want_q,
                          ProloguePartials pp, cudaStream_t st) {
    if (D.dtype == 0) return launch_pass1_t<float>(D, Q, K, V, want_q, pp, st);
    return launch_pass1_t<__nv_bfloat16>(D, Q, K, V, want_q, pp, st);
}
int launch_prologue_pass2(const Dims &D, const void *K, ProloguePartials pp, const double *stats, double *nrm2,
                          cudaStream_t st) {
    if (D.dtype == 0) return launch_pass2_t<float>(D, K, pp, stats, nrm2, st);
    return launch_pass2_t<__nv_bfloat16>(D, K, pp, stats, nrm2, st);
}

int launch_vrange(const Dims &D, const void *V, ProloguePartials pp, void *vmin, void *vmax, cudaStream_t st) {
    if (D.dtype == 0) return launch_vrange_t<float>(D, V, pp, vmin, vmax, st);
    return launch_vrange_t<__nv_bfloat16>(D, V, pp, vmin, vmax, st);
}

// WC_CHECK_FINITE: flag |= 1 if any element of x[0, count) is NaN or +-Inf (exponent field all ones).
// bf16 and fp32 are tested on their bit patterns, 16 bytes per thread per step.
__global__ void __launch_bounds__(256) check_finite_kernel(const uint4 *x, int64_t nvec, const unsigned char *tail,
                                                            int64_t ntail, int esz, int *flag) {
    const uint32_t m32 = 0x7f800000u;
    bool bad = false;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
        const uint4 q = __ldg(x + v);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (esz == 4) bad |= (w[k] & m32) == m32;
            else bad |= ((w[k] & 0x7f80u) == 0x7f80u) || (((w[k] >> 16) & 0x7f80u) == 0x7f80u);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < ntail) {  // the < 16 trailing bytes, one element per thread
        if (esz == 4) bad |= (reinterpret_cast<const uint32_t *>(tail)[threadIdx.x] & m32) == m32;
        else bad |= (reinterpret_cast<const uint16_t *>(tail)[threadIdx.x] & 0x7f80u) == 0x7f80u;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

int launch_check_finite(const void *x, int64_t count, int dtype, int *flag, cudaStream_t st) {
    if (!x || count <= 0) return 0;
    const int esz = dtype == 0 ? 4 : 2;
    const int64_t bytes = count * esz, nvec = bytes / 16;
    const int64_t ntail = (bytes - nvec * 16) / esz;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 148, ceil_div(nvec, 256)));
    check_finite_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint4 *>(x), nvec,
                                                static_cast<const unsigned char *>(x) + nvec * 16, ntail, esz, flag);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int prologue_num_splits(const Dims &D) {
    const int64_t by_rows = ceil_div(std::max<int64_t>(D.n, (int64_t)D.group() * D.m), 256);
    const int64_t cap = std::max<int64_t>(1, 1184 / D.units());
    return (int)std::max<int64_t>(1, std::min<int64_t>(by_rows, cap));
}

int launch_prologue(const Dims &D, const void *Q, const void *K, const void *V, double rq, double beta,
                    ProloguePartials pp, double *stats, double *nrm2, void *vmin, void *vmax, int pflags,
                    cudaStream_t st) {
    if (D.dtype == 0) return launch_prologue_t<float>(D, Q, K, V, rq, beta, pp, stats, nrm2, vmin, vmax, pflags, st);
    return launch_prologue_t<__nv_bfloat16>(D, Q, K, V, rq, beta, pp, stats, nrm2, vmin, vmax, pflags, st);
}

}  // namespace wc
