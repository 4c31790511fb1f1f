// select.cu -- A1+A2 of the hot path: randomly pivoted Cholesky / RPNys selection.
//
// Alg 1 in the equivalent partial-Cholesky form: round i, pivot s,
//   c_l    = h~(k_l, k_s) - sum_{j<i} F[j,l] F[j,s]         (kernel column + rank update)
//   F[i,l] = c_l / sqrt(p_s)                                (reading Z5)
//   p_l    = max(p_l - F[i,l]^2, 0);  p_s = 0               (diagonal downdate, Z4)
// with h~(a,b) = exp(g <a-kbar, b-kbar> - mstar) (P:306 on centred keys, Z10), the pivot
// drawn by Eq. 4 as an fp64 inverse CDF with strict '>' from a Philox4x32-10
// uniform (Z2), and the exhaustion stop T <= 1000 r 2^-52 T0 (Z3).
//
// Execution: a persistent kernel; each unit (batch, kv-head) is served by `cpu` co-resident
// CTAs that own contiguous key ranges.  One grid-group barrier per round: after it every CTA
// redundantly reads the per-CTA residual totals (fixed order), draws the same uniform, finds
// the owning CTA and scans that CTA's residual slice (L2-resident) to get s -- no second
// exchange.  Then every CTA streams its slice of F[0:i, :] (pivot-major fp64, coalesced), K
// and the residual diagonal.  State is fp64 throughout so the pivot sequence matches the fp64
// oracle (SURVEY.md key finding 2).  The residual diagonal is double-buffered across rounds
// so the scan of round i never races the downdate of round i.
//
// HBM traffic per unit: n r (d e + 24) + 4 n r (r-1) bytes.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace wc {

namespace {

constexpr int kSelThreads = 512;

struct SelArgs {
    const void *K;
    const double *stats;
    const double *nrm2;
    double *p;      // [2][units][n]
    double *F;      // [units][r][n]
    double *part;   // [units][2][kMaxCpu]
    unsigned *bar;  // [units]
    int32_t *S;
    int32_t *r_eff;
    double *L;
    int64_t n;
    int units, r, cpu;
    uint64_t seed;
};

constexpr int kST = 256;  // keys per super-tile (8 warp-tiles of 32 keys)
constexpr int kTK = kST / 32;

template <typename T, int D>
__global__ void __launch_bounds__(kSelThreads) rpc_select_kernel(SelArgs a) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, w = warp_index(), nw = nt >> 5;
    const int H = nt / kST;           // threads per key in the kernel-dot phase (1 or 2)
    double *kb = sm;                  // [D]    kbar
    double *kcs = kb + D;             // [D]    centred pivot key
    double *fs = kcs + D;             // [r]    F[0:i, s]
    double *red = fs + a.r;           // [nw][kST] per-warp partial F-dots
    double *kd = red + nw * kST;      // [H][kST] partial kernel dots
    double *scr = kd + 2 * kST;       // [40]   reduction scratch
    __shared__ int sh_s, sh_cstar, sh_done, sh_last;
    __shared__ double sh_t, sh_ps;

    const int u = blockIdx.x / a.cpu, c = blockIdx.x % a.cpu;
    const int64_t n = a.n;
    const int64_t chunk = ((ceil_div(n, a.cpu) + 31) / 32) * 32;
    const int64_t lo = std::min<int64_t>(n, (int64_t)c * chunk), hi = std::min<int64_t>(n, lo + chunk);

    const T *Ku = static_cast<const T *>(a.K) + (int64_t)u * n * D;
    const double *st = a.stats + (int64_t)u * (8 + D);
    const double g = st[1], mstar = st[2];
    double *p0 = a.p + (int64_t)u * n;
    double *p1 = a.p + ((int64_t)a.units + u) * n;
    double *Fu = a.F + (int64_t)u * a.r * n;
    double *partu = a.part + (int64_t)u * 2 * kMaxCpu;
    unsigned *bar = a.bar + u;
    for (int j = tid; j < D; j += nt) kb[j] = st[8 + j];

    // p <- kernel diagonal h~(k_l, k_l) = exp(g ||k_l - kbar||^2 - mstar)   (Alg 1)
    double loc = 0.0;
    for (int64_t l = lo + tid; l < hi; l += nt) {
        const double v = exp(__dadd_rn(__dmul_rn(g, a.nrm2[(int64_t)u * n + l]), -mstar));
        p0[l] = v;
        loc += v;
    }
    loc = block_sum(loc, scr);
    if (tid == 0) partu[c] = loc;
    unsigned epoch = 1;
    if (a.cpu > 1) group_barrier(bar, a.cpu, epoch++);
    else __syncthreads();

    double T0 = 0.0, theta = 0.0;  // meaningful in warp 0
    int i = 0;
    for (; i < a.r; ++i) {
        double *cur = (i & 1) ? p1 : p0;
        double *nxt = (i & 1) ? p0 : p1;
        const double *pc = partu + (i & 1) * kMaxCpu;
        double *pn = partu + ((i + 1) & 1) * kMaxCpu;

        // ---- A1a (warp 0): total T over the per-CTA residual sums, exhaustion test, uniform,
        // owning CTA c* = min{c : prefix_c > t}.  Fixed order => identical in every CTA.
        if (w == 0) {
            const int per = (a.cpu + 31) / 32;
            const int b0 = lane * per, b1 = min(a.cpu, b0 + per);
            double v = 0.0;
            for (int cc = b0; cc < b1; ++cc) v += __ldcg(pc + cc);
            double incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const double Ttot = __shfl_sync(0xffffffffu, incl, 31);
            if (i == 0) {
                T0 = Ttot;
                theta = 1000.0 * (double)a.r * 2.220446049250313e-16 * T0;
            }
            const bool done = Ttot <= theta;
            if (!done) {
                const double t = pivot_uniform(a.seed, (uint32_t)i, (uint64_t)u) * Ttot;
                const unsigned hit = __ballot_sync(0xffffffffu, b1 > b0 && incl > t);
                const unsigned pos = __ballot_sync(0xffffffffu, b1 > b0 && v > 0.0);
                const int L = hit ? __ffs(hit) - 1 : 31 - __clz(pos);
                if (lane == L) {
                    double acc = incl - v;
                    int cs = -1, last = -1;
                    double excl = 0.0, last_excl = 0.0;
                    for (int cc = b0; cc < b1; ++cc) {
                        const double pv = __ldcg(pc + cc);
                        if (pv > 0.0) { last = cc; last_excl = acc; }
                        const double nacc = acc + pv;
                        if (cs < 0 && hit && nacc > t) { cs = cc; excl = acc; }
                        acc = nacc;
                    }
                    if (cs < 0) { cs = last; excl = last_excl; }  // rounding fallback (reading Z2)
                    sh_cstar = cs;
                    sh_t = t - excl;
                }
            }
            if (lane == 0) {
                sh_done = done ? 1 : 0;
                sh_s = 0x7fffffff;
                sh_last = -1;
            }
        }
        __syncthreads();
        if (sh_done) break;
        const int cstar = sh_cstar;
        const double tp = sh_t;
        // ---- A1b: inverse CDF inside the owning CTA's slice (block scan, fixed order)
        {
            const int64_t slo = std::min<int64_t>(n, (int64_t)cstar * chunk);
            const int64_t shi = std::min<int64_t>(n, slo + chunk);
            const int64_t per = ceil_div(shi - slo, nt);
            const int64_t b0 = slo + (int64_t)tid * per, b1 = std::min<int64_t>(shi, b0 + per);
            double v = 0.0;
            for (int64_t l = b0; l < b1; ++l) v += __ldcg(cur + l);
            double tot;
            const double ex = block_exclusive_scan(v, scr, &tot);
            double run = ex;
            int found = -1, lastpos = -1;
            for (int64_t l = b0; l < b1; ++l) {
                const double pl = __ldcg(cur + l);
                if (pl > 0.0) lastpos = (int)l;
                run += pl;
                if (found < 0 && run > tp) found = (int)l;
            }
            if (found >= 0) atomicMin(&sh_s, found);
            if (lastpos >= 0) atomicMax(&sh_last, lastpos);
            __syncthreads();
            if (tid == 0 && sh_s == 0x7fffffff) sh_s = sh_last;  // rounding fallback (reading Z2)
            __syncthreads();
        }
        const int s = sh_s;
        // ---- pivot data: centred k_s (fp64) and F[0:i, s]
        for (int j = tid; j < D; j += nt) kcs[j] = __dadd_rn(to_f64(Ku[(int64_t)s * D + j]), -kb[j]);
        for (int j = tid; j < i; j += nt) fs[j] = __ldcg(Fu + (int64_t)j * n + s);
        if (tid == 0) sh_ps = __ldcg(cur + s);
        __syncthreads();
        const double rs = sqrt(sh_ps);
        if (c == cstar) {
            for (int j = tid; j < i; j += nt) a.L[((int64_t)u * a.r + i) * a.r + j] = fs[j];
            if (tid == 0) a.S[(int64_t)u * a.r + i] = s;
        }
        // ---- A2: kernel column, rank update and downdate of own keys, one super-tile of
        // kST keys at a time.  Phase A: warps split the rows j of F[0:i, tile] (coalesced
        // 256-byte row segments, kTK independent loads per row per lane); phase B: kernel dot
        // <k_l - kbar, k_s - kbar> (H threads per key); phase C: combine in fixed order.
        loc = 0.0;
        double *Fi = Fu + (int64_t)i * n;
        for (int64_t k0 = lo; k0 < hi; k0 += kST) {
            {
                double acc[kTK];
#pragma unroll
                for (int t = 0; t < kTK; ++t) acc[t] = 0.0;
                int j = w;
                for (; j + nw < i; j += 2 * nw) {
                    const double *F0 = Fu + (int64_t)j * n + k0 + lane;
                    const double *F1 = F0 + (int64_t)nw * n;
                    double x0[kTK], x1[kTK];
#pragma unroll
                    for (int t = 0; t < kTK; ++t) {
                        const bool ok = k0 + 32 * t + lane < hi;
                        x0[t] = ok ? __ldcg(F0 + 32 * t) : 0.0;
                        x1[t] = ok ? __ldcg(F1 + 32 * t) : 0.0;
                    }
                    const double f0 = fs[j], f1 = fs[j + nw];
#pragma unroll
                    for (int t = 0; t < kTK; ++t) {
                        acc[t] = __dadd_rn(acc[t], __dmul_rn(x0[t], f0));
                        acc[t] = __dadd_rn(acc[t], __dmul_rn(x1[t], f1));
                    }
                }
                if (j < i) {
                    const double *F0 = Fu + (int64_t)j * n + k0 + lane;
                    const double f0 = fs[j];
#pragma unroll
                    for (int t = 0; t < kTK; ++t) {
                        const bool ok = k0 + 32 * t + lane < hi;
                        const double x0 = ok ? __ldcg(F0 + 32 * t) : 0.0;
                        acc[t] = __dadd_rn(acc[t], __dmul_rn(x0, f0));
                    }
                }
#pragma unroll
                for (int t = 0; t < kTK; ++t) red[w * kST + 32 * t + lane] = acc[t];
            }
            {
                const int kk = tid % kST, half = tid / kST;
                const int64_t l = k0 + kk;
                double dot = 0.0;
                if (l < hi) {
                    constexpr int Dh = D;  // elements per thread when H == 1
                    const int len = Dh / H, j0 = half * len;
                    for (int jj = 0; jj < len; jj += 8) {
                        double kv[8];
                        Vec8<T>::load(Ku + l * D + j0 + jj, kv);
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            dot = __dadd_rn(dot, __dmul_rn(__dadd_rn(kv[q], -kb[j0 + jj + q]), kcs[j0 + jj + q]));
                    }
                }
                kd[half * kST + kk] = dot;
            }
            __syncthreads();
            if (tid < kST) {
                const int64_t l = k0 + tid;
                if (l < hi) {
                    double acc = 0.0;
                    for (int ww = 0; ww < nw; ++ww) acc = __dadd_rn(acc, red[ww * kST + tid]);
                    double dot = kd[tid];
                    for (int hh = 1; hh < H; ++hh) dot = __dadd_rn(dot, kd[hh * kST + tid]);
                    const double hval = exp(__dadd_rn(__dmul_rn(g, dot), -mstar));
                    const double f = (hval - acc) / rs;
                    Fi[l] = f;
                    double q = __dadd_rn(__ldcg(cur + l), -__dmul_rn(f, f));
                    q = q > 0.0 ? q : 0.0;
                    if (l == s) {
                        q = 0.0;
                        a.L[((int64_t)u * a.r + i) * a.r + i] = f;
                    }
                    nxt[l] = q;
                    loc += q;
                }
            }
            __syncthreads();
        }
        loc = block_sum(loc, scr);
        if (tid == 0) pn[c] = loc;
        if (a.cpu > 1) group_barrier(bar, a.cpu, epoch++);
        else __syncthreads();
    }
    if (c == 0 && tid == 0) {
        a.r_eff[u] = i;
        const_cast<double *>(st)[5] = T0;
    }
}

template <typename T, int D>
int launch_select_td(const Dims &Dm, const void *K, const double *stats, SelectBufs b, uint64_t seed,
                     int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    SelArgs a;
    a.K = K; a.stats = stats; a.nrm2 = b.nrm2; a.p = b.p; a.F = b.F; a.part = b.part; a.bar = b.bar;
    a.S = S; a.r_eff = r_eff; a.L = L; a.n = Dm.n; a.units = Dm.units(); a.r = Dm.r;
    a.cpu = select_ctas_per_unit(Dm); a.seed = seed;
    const int threads = (Dm.n / a.cpu >= 384) ? kSelThreads : 256;
    const size_t smem = (size_t)(2 * D + Dm.r + (threads / 32) * kST + 2 * kST + 40) * sizeof(double);
    auto kern = rpc_select_kernel<T, D>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaMemsetAsync(b.bar, 0, sizeof(unsigned) * a.units, st) != cudaSuccess) return -1;
    const dim3 grid(a.units * a.cpu);
    if (a.cpu > 1) {
        void *args[] = {&a};
        if (cudaLaunchCooperativeKernel((const void *)kern, grid, dim3(threads), args, smem, st) != cudaSuccess)
            return -1;
    } else {
        kern<<<grid, threads, smem, st>>>(a);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

template <typename T>
int launch_select_t(const Dims &Dm, const void *K, const double *stats, SelectBufs b, uint64_t seed,
                    int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    switch (Dm.d) {
        case 16: return launch_select_td<T, 16>(Dm, K, stats, b, seed, S, r_eff, L, st);
        case 32: return launch_select_td<T, 32>(Dm, K, stats, b, seed, S, r_eff, L, st);
        case 64: return launch_select_td<T, 64>(Dm, K, stats, b, seed, S, r_eff, L, st);
        case 128: return launch_select_td<T, 128>(Dm, K, stats, b, seed, S, r_eff, L, st);
    }
    return -1;
}

}  // namespace

int select_ctas_per_unit(const Dims &D) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int units = D.units();
    const int64_t per_unit = std::max<int64_t>(1, (int64_t)sms / units);
    const int64_t by_n = std::max<int64_t>(1, D.n / 256);
    return (int)std::min<int64_t>(std::min<int64_t>(per_unit, by_n), kMaxCpu);
}

int launch_select(const Dims &D, const void *K, const double *stats, SelectBufs b, uint64_t seed,
                  int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    if (D.dtype == 0) return launch_select_t<float>(D, K, stats, b, seed, S, r_eff, L, st);
    return launch_select_t<__nv_bfloat16>(D, K, stats, b, seed, S, r_eff, L, st);
}

}  // namespace wc
