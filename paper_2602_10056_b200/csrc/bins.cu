// bins.cu -- Alg 2 binning on top of the per-unit kernels: every (unit u,
// bin b) pair is a sub-unit su = u*B + b of the selection and weights kernels (contiguous bins of
// nb = floor(n/B) keys, the last one also holding the n - B nb remainder: the kernels address a
// sub-unit's keys through Dims::sub_unit()).  Readings Z12 (tau_b uses n_b), Z13 (r_b =
// min(ceil(r/B), nb), remainder in the last bin), Z23 (Philox stream of sub-unit u*B + b).
//   bins_stats_kernel: per sub-unit R_K^b = max ||k_l - kbar|| over the bin (global kbar, from
//     the unit prologue's nrm2), tau_b (Eq. 7 with n_b), g_b, mstar_b; R_Q and kbar of the unit.
//   bins_pack_kernel:  concatenate the bins' valid coreset rows into the unit layout (S with
//     unit-level key indices, KS, X, r_eff = sum of the bins' r_eff), rows past r_eff zero / -1.
//   bins_unpack_kernel: the inverse for S (split API: wildcat_weights after wildcat_select).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace wc {

namespace {

constexpr int kBT = 256;

__global__ void __launch_bounds__(kBT) bins_stats_kernel(const double *__restrict__ stats_u, const double *__restrict__ nrm2,
                                                         int64_t nb, int64_t unit_n, int d, int bins, double beta,
                                                         double *__restrict__ stats_b, int tau_one) {
    pdl_wait();
    __shared__ double scr[40];
    const int su = blockIdx.x, u = su / bins;
    const SubUnit sub = sub_unit(su, nb, bins, nb, unit_n);  // the last bin also holds the remainder (Z13)
    const double *nr = nrm2 + sub.base;  // nrm2 [units][unit_n]
    double mx = 0.0;
    for (int64_t l = threadIdx.x; l < sub.count; l += kBT) mx = fmax(mx, __ldg(nr + l));
    mx = block_max(mx, scr);
    const double *su_u = stats_u + (int64_t)u * (kStatsHead + d);
    double *sb = stats_b + (int64_t)su * (kStatsHead + d);
    for (int j = threadIdx.x; j < d; j += kBT) sb[kStatsHead + j] = su_u[kStatsHead + j];  // global kbar
    if (threadIdx.x == 0) {
        const double rk = sqrt(mx), rq = su_u[4];
        double tau = 1.0;
        if (!tau_one && rq * rk > 0.0) {  // Eq. 7 with n_b (Z12); WC_TAU_ONE: tau = 1
            const double rho0 = sqrt(1.0 + exp(lambert_w0_dev(2.0 / (2.718281828459045 * 2.718281828459045)) + 2.0));
            const double b0 = log((double)sub.count) / (beta * rq * rk) + 2.0;
            const double w = lambert_w0_dev(b0 / (2.0 * rho0));
            tau = sqrt((rk / rq) * b0 / (2.0 * w));
        }
        const double g = beta / (tau * tau);
        sb[0] = tau;
        sb[1] = g;
        sb[2] = g * rk * rk;
        sb[3] = rk;
        sb[4] = rq;
        for (int k = 5; k < kStatsHead; ++k) sb[k] = 0.0;
    }
}

// Packed layout: row a of unit u comes from bin b, local row a - off_b, off_b = sum_{b' < b} r_eff_b'.
// Block (row tile of kPackRows, unit u): the block first forms off_b for all bins of the unit (a
// 128-thread exclusive scan in shared memory), then each warp places its rows by a binary search over
// the offsets and copies them with its lanes.  Ssub holds bin-local key indices.
constexpr int kPackRows = 8, kPackT = 128;
template <typename T>
__global__ void __launch_bounds__(kPackT) bins_pack_kernel(const int32_t *__restrict__ Ssub, const int32_t *__restrict__ reff_sub, int bins,
                                 int rb, int64_t nb, int d, const T *__restrict__ KSsub, const float *__restrict__ Xsub,
                                 int32_t *__restrict__ S, int32_t *__restrict__ reff, T *__restrict__ KS,
                                 float *__restrict__ X) {
    pdl_wait();
    extern __shared__ int offs[];  // [bins + 1]: exclusive prefix of the bins' r_eff, offs[bins] = total
    __shared__ int wsum[kPackT / 32];
    const int u = blockIdx.y, R = bins * rb, dc = d + 1, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int per = (bins + kPackT - 1) / kPackT, b0 = tid * per, b1 = min(bins, b0 + per);
    int v = 0;
    for (int bb = b0; bb < b1; ++bb) v += reff_sub[u * bins + bb];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    int base = 0;
    for (int k = 0; k < w; ++k) base += wsum[k];
    int run = base + incl - v;  // exclusive prefix at b0
    for (int bb = b0; bb < b1; ++bb) {
        offs[bb] = run;
        run += reff_sub[u * bins + bb];
    }
    if (tid == kPackT - 1) offs[bins] = base + incl;
    __syncthreads();
    const int total = offs[bins];
    if (blockIdx.x == 0 && tid == 0 && reff) reff[u] = total;
    for (int rr = w; rr < kPackRows; rr += kPackT / 32) {
        const int a = blockIdx.x * kPackRows + rr;
        if (a >= R) break;
        int b = -1, loc = 0;
        if (a < total) {  // last bin with offs[bin] <= a (bins with r_eff = 0 share offsets: take the last)
            int lo = 0, hi = bins - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (offs[mid] <= a) lo = mid; else hi = mid - 1;
            }
            b = lo;
            loc = a - offs[b];
        }
        const int64_t src = ((int64_t)u * bins + (b < 0 ? 0 : b)) * rb + loc;
        if (lane == 0 && S) S[(int64_t)u * R + a] = b < 0 ? -1 : (int32_t)(b * nb + Ssub[src]);
        if (KS)
            for (int j = lane; j < d; j += 32)
                KS[((int64_t)u * R + a) * d + j] = b < 0 ? from_f32<T>(0.f) : KSsub[src * d + j];
        if (X)
            for (int j = lane; j < dc; j += 32) X[((int64_t)u * R + a) * dc + j] = b < 0 ? 0.f : Xsub[src * dc + j];
    }
}

// One warp per unit: split the packed S (bin order) back into bin-local indices per sub-unit.
__global__ void bins_unpack_kernel(const int32_t *__restrict__ S, int units, int bins, int rb, int64_t nb,
                                   int32_t *__restrict__ Ssub, int32_t *__restrict__ reff_sub) {
    const int u = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (u >= units) return;
    const int R = bins * rb;
    for (int b = lane; b < bins; b += 32) reff_sub[u * bins + b] = 0;
    __syncwarp();
    if (lane == 0) {
        int cnt = 0, cur = -1;
        for (int a = 0; a < R; ++a) {
            const int s = S[(int64_t)u * R + a];
            if (s < 0) break;
            const int b = (int)(s / nb < bins - 1 ? s / nb : bins - 1);  // remainder keys belong to the last bin
            if (b != cur) { cur = b; cnt = 0; }
            Ssub[((int64_t)u * bins + b) * rb + cnt] = (int32_t)(s - b * nb);
            reff_sub[u * bins + b] = ++cnt;
        }
    }
}

}  // namespace

int launch_bins_stats(const Dims &D, int bins, double beta, const double *stats_u, const double *nrm2, double *stats_b,
                      int pflags, cudaStream_t st) {
    launch_pdl(bins_stats_kernel, dim3(D.units() * bins), dim3(kBT), 0, st, stats_u, nrm2, D.n / bins, D.n, D.d, bins,
               beta, stats_b, (pflags & kPfTauOne) ? 1 : 0);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_bins_pack(const Dims &D, int bins, int rb, const int32_t *Ssub, const int32_t *reff_sub, const void *KSsub,
                     const float *Xsub, int32_t *S, int32_t *reff, void *KS, float *X, cudaStream_t st) {
    dim3 g((bins * rb + kPackRows - 1) / kPackRows, D.units());
    const size_t smem = (size_t)(bins + 1) * sizeof(int);
    if (D.dtype == 0)
        launch_pdl(bins_pack_kernel<float>, g, dim3(kPackT), smem, st, Ssub, reff_sub, bins, rb, D.n / bins, D.d,
                   static_cast<const float *>(KSsub), Xsub, S, reff, static_cast<float *>(KS), X);
    else
        launch_pdl(bins_pack_kernel<__nv_bfloat16>, g, dim3(kPackT), smem, st, Ssub, reff_sub, bins, rb, D.n / bins,
                   D.d, static_cast<const __nv_bfloat16 *>(KSsub), Xsub, S, reff, static_cast<__nv_bfloat16 *>(KS), X);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_bins_unpack(const Dims &D, int bins, int rb, const int32_t *S, int32_t *Ssub, int32_t *reff_sub,
                       cudaStream_t st) {
    bins_unpack_kernel<<<(D.units() + 3) / 4, 128, 0, st>>>(S, D.units(), bins, rb, D.n / bins, Ssub, reff_sub);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace wc
