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
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "select_common.cuh"

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
    int64_t n;    // keys per sub-unit buffer (the largest sub-unit)
    int bins;     // sub-unit geometry (Dims::bins, nb, unit_n; sub_unit())
    int64_t nb, unit_n;
    int64_t ldF;  // row stride of F (n rounded up to 32: every row segment is 256-byte aligned)
    int units, r, cpu;
    uint64_t seed;
    uint64_t unit0;  // Philox id of sub-unit 0 (wc_opts.unit_offset [x B]); unit u draws stream unit0 + u
    unsigned long long *trace;  // debug (WC_SELECT_TRACE): [r][16] globaltimer stamps of CTA 0
    int rkeep;                  // F rows [0, rkeep) are kept L2-resident (evict_last); later rows evict_first
    int nstm;                   // TMA kernel: super-tiles per CTA slice (tile-major F: [cpu][nstm][r][256])
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define WC_TR(k)                                                                              \
    do {                                                                                      \
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && i < a.r) a.trace[i * 16 + (k)] = gtimer(); \
    } while (0)


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
    const SubUnit sub = sub_unit(u, a.n, a.bins, a.nb, a.unit_n);
    const int64_t n = sub.count;  // this sub-unit's keys (a.n: the buffer stride)
    const int64_t chunk = ((ceil_div(n, a.cpu) + 31) / 32) * 32;
    const int64_t lo = std::min<int64_t>(n, (int64_t)c * chunk), hi = std::min<int64_t>(n, lo + chunk);

    const T *Ku = static_cast<const T *>(a.K) + sub.base * D;
    const double *st = a.stats + (int64_t)u * (kStatsHead + D);
    const double g = st[1], mstar = st[2];
    double *p0 = a.p + (int64_t)u * a.n;
    double *p1 = a.p + ((int64_t)a.units + u) * a.n;
    double *Fu = a.F + (int64_t)u * a.r * a.ldF;
    double *partu = a.part + (int64_t)u * 2 * kMaxCpu;
    unsigned *bar = a.bar + u;
    for (int j = tid; j < D; j += nt) kb[j] = st[kStatsHead + j];

    // p <- kernel diagonal h~(k_l, k_l) = exp(g ||k_l - kbar||^2 - mstar)   (Alg 1)
    double loc = 0.0;
    for (int64_t l = lo + tid; l < hi; l += nt) {
        const double v = exp(__dadd_rn(__dmul_rn(g, a.nrm2[sub.base + l]), -mstar));
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
                const double t = pivot_uniform(a.seed, (uint32_t)i, a.unit0 + (uint64_t)u) * Ttot;
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
        for (int j = tid; j < i; j += nt) fs[j] = __ldcg(Fu + (int64_t)j * a.ldF + s);
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
        double *Fi = Fu + (int64_t)i * a.ldF;
        for (int64_t k0 = lo; k0 < hi; k0 += kST) {
            {
                double acc[kTK];
#pragma unroll
                for (int t = 0; t < kTK; ++t) acc[t] = 0.0;
                int j = w;
                for (; j + nw < i; j += 2 * nw) {
                    const double *F0 = Fu + (int64_t)j * a.ldF + k0 + lane;
                    const double *F1 = F0 + (int64_t)nw * a.ldF;
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
                    const double *F0 = Fu + (int64_t)j * a.ldF + k0 + lane;
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
        double *stw = const_cast<double *>(st);
        stw[5] = T0;
        stw[6] = (double)i;                          // rounds run
        stw[7] = (double)i;                          // pivots drawn
        stw[8] = 0.5 * (double)i * (double)(i - 1);  // F rows re-read: sum over rounds q of q
        stw[9] = stw[8];                             // F-prefix dot work (one pivot per round)
    }
}

// =====================================================================================
// TMA-pipelined variant.  8 compute warps + 1 producer warp.  The producer streams the CTA's
// slice of F[0:i-1, :] (rows written >= 2 rounds ago) into a shared-memory ring of stages
// (kRPS rows x 256 keys fp64 = 16 KB each) with 1-D bulk async copies (cp.async.bulk, the TMA
// engine) completing on mbarriers.  It runs ahead of the compute warps by up to NS stages,
// across round boundaries: while the compute warps wait at the grid barrier and search the next
// pivot, the next round's F tiles are already landing in shared memory.  Row i-1 (written by
// this CTA in the previous round) is read directly.  Compute warps synchronise among themselves
// with named barrier 1 so the producer never joins a CTA-wide barrier.
// =====================================================================================
template <typename T, int D>
__global__ void __launch_bounds__(kTmaThreads, 1) rpc_select_tma_kernel(SelArgs a, int NS) {
    using KR = KRow<T, D>;
    extern __shared__ __align__(128) unsigned char smraw[];
    double *ring = reinterpret_cast<double *>(smraw);  // [NS][kRPS][kST]
    double *fs = ring + (size_t)NS * kRPS * kST;        // [r]
    double *red = fs + a.r;                             // [kCW][kST]
    double *kb = red + kCW * kST;                       // [D]
    double *kcs = kb + D;                               // [D]
    double *scr = kcs + D;                              // [40]
    uint64_t *full = reinterpret_cast<uint64_t *>(scr + 40);
    uint64_t *empty = full + NS;
    __shared__ int sh_s, sh_cstar, sh_done, sh_last;
    __shared__ volatile int sh_stop;
    __shared__ volatile int sh_rounds_done;  // rounds whose F row (this CTA) is complete and visible
    __shared__ double sh_ps, sh_c0, sh_t;

    const int tid = threadIdx.x, lane = tid & 31, w = warp_index();
    const int u = blockIdx.x / a.cpu, c = blockIdx.x % a.cpu;
    const SubUnit sub = sub_unit(u, a.n, a.bins, a.nb, a.unit_n);
    const int64_t n = sub.count;  // this sub-unit's keys (a.n: the buffer stride)
    const int64_t chunk = ((ceil_div(n, a.cpu) + 31) / 32) * 32;
    const int64_t chunk_max = ((ceil_div(a.n, a.cpu) + 31) / 32) * 32;
    const int64_t lo = std::min<int64_t>(n, (int64_t)c * chunk), hi = std::min<int64_t>(n, lo + chunk);
    const int nst = (int)ceil_div(hi - lo, kST);

    const T *Ku = static_cast<const T *>(a.K) + sub.base * D;
    const double *st = a.stats + (int64_t)u * (kStatsHead + D);
    // tile-major F: CTA c' owns [r x chunk]; its super-tile k' is the block [r][w_k'] at column
    // offset 256 k', w_k' = min(256, chunk - 256 k') (a multiple of 32): 8 rows = one contiguous copy
    double *Fu = a.F + (int64_t)u * a.cpu * chunk_max * a.r;
    double *Fc = Fu + (int64_t)c * chunk * a.r;  // this CTA's blocks
    auto tile_w = [&](int k) -> int { return (int)std::min<int64_t>(kST, chunk - (int64_t)k * kST); };

    if (tid == 0) {
        for (int q = 0; q < NS; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kCW);
        }
        flag_st(&sh_stop, 0);
        flag_st(&sh_rounds_done, 0);
        fence_mbar_init();
    }
    __syncthreads();  // the only CTA-wide barrier: everything after is role-specific

    if (w == kCW) {
        // ================= producer warp (one elected lane) =================
        if (lane == 0) {
            const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
            int stage = 0;
            uint32_t ph = 0, issued = 0, par = 0;
            for (int i = 2; i < a.r; ++i) {
                const int rows = i - 1;  // TMA rows 0..i-2; row i-1 is read directly
                while (flag_ld(&sh_rounds_done) < i - 1) {  // rows 0..i-2 of this CTA written and visible
                    if (flag_ld(&sh_stop)) goto drain;
                    __nanosleep(32);
                }
                for (int k = 0; k < nst; ++k) {
                    const double *blk = Fc + (int64_t)k * a.r * kST;
                    const int wk = tile_w(k);
                    for (int j0 = 0; j0 < rows; j0 += kRPS) {
                        const int nr = min(kRPS, rows - j0);
                        const uint32_t bytes = (uint32_t)(nr * wk * sizeof(double));
                        while (!mbar_try_wait(&empty[stage], ph ^ 1u)) {
                            if (flag_ld(&sh_stop)) goto drain;
                        }
                        if (flag_ld(&sh_stop)) goto drain;
                        mbar_arrive_expect_tx(&full[stage], bytes);
                        // one contiguous bulk copy of nr rows x 256 keys (tile-major layout)
                        bulk_g2s_hint(ring + (size_t)stage * kRPS * kST, blk + (int64_t)j0 * wk, bytes, &full[stage],
                                      j0 < a.rkeep ? keep : stream);
                        issued |= 1u << stage;
                        par = (par & ~(1u << stage)) | (ph << stage);
                        if (++stage == NS) { stage = 0; ph ^= 1u; }
                    }
                }
            }
        drain:
            // never leave the CTA with bulk copies in flight
            for (int q = 0; q < NS; ++q)
                if (issued & (1u << q)) mbar_wait(&full[q], (par >> q) & 1u);
        }
        return;
    }

    // ================= compute warps (256 threads) =================
    const double g = st[1], mstar = st[2];
    double *p0 = a.p + (int64_t)u * a.n;
    double *p1 = a.p + ((int64_t)a.units + u) * a.n;
    for (int j = tid; j < D; j += kCT) kb[j] = st[kStatsHead + j];

    double loc = 0.0;
    double p_first = 0.0;  // residual of this thread's key in super-tile 0 (kept in a register)
    for (int64_t l = lo + tid; l < hi; l += kCT) {
        const double v = exp(__dadd_rn(__dmul_rn(g, a.nrm2[sub.base + l]), -mstar));
        p0[l] = v;
        if (l == lo + tid) p_first = v;
        loc += v;
    }
    loc = cw_sum(loc, scr);
    if (tid == 0) a.part[(int64_t)u * 2 * kMaxCpu + c] = loc;
    unsigned epoch = 1;
    cw_group_barrier(a.bar + u, a.cpu, epoch++, &sh_rounds_done, 0);

    KR krow;  // K row of this thread's key for the next super-tile to process (prefetched)
    if (nst > 0 && lo + tid < hi) krow.load(Ku + (lo + tid) * D);
    else krow.zero();
    double pcur_next = p_first;
    double fkeep[2] = {0.0, 0.0};  // this thread's F[i-1, key] for super-tiles 0 and 1
    int rstage = 0;
    uint32_t rph = 0;

    double T0 = 0.0, theta = 0.0;
    int i = 0;
    for (; i < a.r; ++i) {
        double *cur = (i & 1) ? p1 : p0;
        double *nxt = (i & 1) ? p0 : p1;
        double p0_next = 0.0;

        // ---- A1a (warp 0): totals over the per-CTA residual sums (one L2 round trip, cached in
        // registers), exhaustion test, Philox uniform, owning CTA c*.  Fixed order.
        if (w == 0) {
            const double uni = pivot_uniform(a.seed, (uint32_t)i, a.unit0 + (uint64_t)u);
            const double *pc = a.part + (int64_t)u * 2 * kMaxCpu + (i & 1) * kMaxCpu;
            const int per = (a.cpu + 31) / 32;
            const int b0 = lane * per, b1 = min(a.cpu, b0 + per);
            constexpr int kPer = 8;  // fast path: cpu <= 256
            double pv[kPer];
            double v = 0.0;
            if (per <= kPer) {
#pragma unroll
                for (int q = 0; q < kPer; ++q) pv[q] = (b0 + q < b1) ? __ldcg(pc + b0 + q) : 0.0;
#pragma unroll
                for (int q = 0; q < kPer; ++q) v += pv[q];
            } else {
                for (int cc = b0; cc < b1; ++cc) v += __ldcg(pc + cc);
            }
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
                const double t = uni * Ttot;
                const unsigned hit = __ballot_sync(0xffffffffu, b1 > b0 && incl > t);
                const unsigned pos = __ballot_sync(0xffffffffu, b1 > b0 && v > 0.0);
                const int L = hit ? __ffs(hit) - 1 : 31 - __clz(pos);
                if (lane == L) {
                    double acc = incl - v;
                    int cs = -1, last = -1;
                    double excl = 0.0, last_excl = 0.0;
                    for (int cc = b0; cc < b1; ++cc) {
                        double pvv = 0.0;
                        if (per <= kPer) {
#pragma unroll
                            for (int q = 0; q < kPer; ++q) pvv = (q == cc - b0) ? pv[q] : pvv;
                        } else {
                            pvv = __ldcg(pc + cc);
                        }
                        if (pvv > 0.0) { last = cc; last_excl = acc; }
                        const double nacc = acc + pvv;
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
        cw_sync();
        if (sh_done) break;
        // ---- A1b: inverse CDF inside c*'s slice (all compute threads, block scan, fixed order).
        // The finder publishes p_s from its registers (no extra global round trip).
        int s;
        {
            const int64_t slo = std::min<int64_t>(n, (int64_t)sh_cstar * chunk);
            const int64_t shi = std::min<int64_t>(n, slo + chunk);
            const int64_t per = ceil_div(shi - slo, kCT);
            const int64_t b0 = slo + (int64_t)tid * per, b1 = std::min<int64_t>(shi, b0 + per);
            const double tp = sh_t;
            constexpr int kC = 4;  // fast path: slice <= 4 * 256 keys, values kept in registers
            double pr[kC];
            double v = 0.0;
            if (per <= kC) {
#pragma unroll
                for (int q = 0; q < kC; ++q) pr[q] = (b0 + q < b1) ? __ldcg(cur + b0 + q) : 0.0;
#pragma unroll
                for (int q = 0; q < kC; ++q) v += pr[q];
            } else {
                for (int64_t l = b0; l < b1; ++l) v += __ldcg(cur + l);
            }
            const double ex = cw_exclusive_scan(v, scr);
            double run = ex;
            int found = -1, lastpos = -1;
            double fval = 0.0, lval = 0.0;
            if (per <= kC) {
#pragma unroll
                for (int q = 0; q < kC; ++q) {
                    if (b0 + q < b1) {
                        const double pl = pr[q];
                        if (pl > 0.0) { lastpos = (int)(b0 + q); lval = pl; }
                        run += pl;
                        if (found < 0 && run > tp) { found = (int)(b0 + q); fval = pl; }
                    }
                }
            } else {
                for (int64_t l = b0; l < b1; ++l) {
                    const double pl = __ldcg(cur + l);
                    if (pl > 0.0) { lastpos = (int)l; lval = pl; }
                    run += pl;
                    if (found < 0 && run > tp) { found = (int)l; fval = pl; }
                }
            }
            if (found >= 0) atomicMin(&sh_s, found);
            if (lastpos >= 0) atomicMax(&sh_last, lastpos);
            cw_sync();
            const int smin = sh_s;
            s = (smin != 0x7fffffff) ? smin : sh_last;  // rounding fallback (reading Z2)
            if (smin != 0x7fffffff ? (found == s) : (lastpos == s)) sh_ps = (smin != 0x7fffffff) ? fval : lval;
        }
        WC_TR(0);
        cw_sync();
        WC_TR(2);
        const int cstar = sh_cstar;
        // ---- pivot data: centred k_s (fp64), c0 = <kbar, k_s - kbar>, F[0:i, s]
        if (w < (D + 31) / 32) {  // warp-uniform
            double pr = 0.0;
            if (tid < D) {
                const double kc = __dadd_rn(to_f64(Ku[(int64_t)s * D + tid]), -kb[tid]);
                kcs[tid] = kc;
                pr = kb[tid] * kc;
            }
            pr = warp_sum(pr);
            if (lane == 0) scr[32 + w] = pr;
        }
        {
            const int64_t cs_ = s / chunk, off = s - cs_ * chunk;
            const int kk_ = (int)(off / kST);
            const int64_t wk_ = std::min<int64_t>(kST, chunk - (int64_t)kk_ * kST);
            const double *fsrc = Fu + cs_ * chunk * a.r + (int64_t)kk_ * kST * a.r + (off % kST);
            for (int j = tid; j < i; j += kCT) fs[j] = __ldcg(fsrc + (int64_t)j * wk_);
        }
        cw_sync();
        WC_TR(3);
        const double rs = sqrt(sh_ps);
        double c0v = 0.0;  // <kbar, k_s - kbar> from the per-warp partials, fixed order
#pragma unroll
        for (int q = 0; q < (D + 31) / 32; ++q) c0v += scr[32 + q];
        if (c == cstar) {
            for (int j = tid; j < i; j += kCT) a.L[((int64_t)u * a.r + i) * a.r + j] = fs[j];
            if (tid == 0) a.S[(int64_t)u * a.r + i] = s;
        }
        // ---- A2 over super-tiles of 256 keys (one key per compute thread in phase C)
        loc = 0.0;
        const uint64_t fpol = i < a.rkeep ? policy_evict_last() : policy_evict_first();
        const int rows = i - 1;  // rows streamed through the ring
        const double flast = i > 0 ? fs[i - 1] : 0.0;
        for (int k = 0; k < nst; ++k) {
            const int64_t l = lo + (int64_t)k * kST + tid;
            const bool own = l < hi;
            const int wk = tile_w(k);
            double *Fk = Fc + (int64_t)k * a.r * kST + tid;  // this key's column in its block (row stride wk)
            const double pcur = pcur_next;
            const double fprev = k < 2 ? fkeep[k & 1] : ((own && i > 0) ? __ldcg(Fk + (int64_t)(i - 1) * wk) : 0.0);
            if (k < 2) WC_TR(4 + 3 * k);
            // phase B: kernel dot <k_l, k_s - kbar> from the prefetched K row (dot = . - c0);
            // phase A: F rows 0..i-2 from the ring, warp w takes row j0 + w of every stage
            double part[4] = {0.0, 0.0, 0.0, 0.0};
            double acc[kTK];
#pragma unroll
            for (int t = 0; t < kTK; ++t) acc[t] = 0.0;
            krow.dot(kcs, part);
            for (int j0 = 0; j0 < rows; j0 += kRPS) {
                const int nr = min(kRPS, rows - j0);
                mbar_wait(&full[rstage], rph);
                if (w < nr) {
                    const double *src = ring + (size_t)rstage * kRPS * kST + (size_t)w * wk + lane;
                    const double fj = fs[j0 + w];
#pragma unroll
                    for (int t = 0; t < kTK; ++t)
                        if (32 * t < wk) acc[t] = fma(src[32 * t], fj, acc[t]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[rstage]);
                if (++rstage == NS) {
                    rstage = 0;
                    rph ^= 1u;
                }
            }
            const double dot = ((part[0] + part[1]) + (part[2] + part[3])) - c0v;
            // prefetch the K row and residual of the next super-tile (wrapping to super-tile 0 of
            // the next round, whose residual this thread computes below)
            if (nst > 1) {
                const int kn = (k + 1 == nst) ? 0 : k + 1;
                const int64_t ln = lo + (int64_t)kn * kST + tid;
                if (ln < hi) {
                    krow.load(Ku + ln * D);
                    if (kn != 0) pcur_next = __ldcg(cur + ln);
                }
            }
#pragma unroll
            for (int t = 0; t < kTK; ++t) red[w * kST + 32 * t + lane] = acc[t];
            if (k < 2) WC_TR(5 + 3 * k);
            cw_sync();
            // phase C: combine (fixed order), new F column entry, residual downdate
            if (own) {
                double accv = 0.0;
#pragma unroll
                for (int ww = 0; ww < kCW; ++ww) accv += red[ww * kST + tid];
                accv = fma(fprev, flast, accv);
                const double hval = exp(__dadd_rn(__dmul_rn(g, dot), -mstar));
                const double f = (hval - accv) / rs;
                st_f64_hint(Fk + (int64_t)i * wk, f, fpol);
                fence_proxy_async_global();
                double q = __dadd_rn(pcur, -__dmul_rn(f, f));
                q = q > 0.0 ? q : 0.0;
                if (l == s) {
                    q = 0.0;
                    a.L[((int64_t)u * a.r + i) * a.r + i] = f;
                }
                nxt[l] = q;
                loc += q;
                if (k == 0) p0_next = q;  // next round's residual for super-tile 0
                if (k < 2) fkeep[k] = f;
            }
            cw_sync();
            if (k < 2) WC_TR(6 + 3 * k);
        }
        pcur_next = p0_next;
        loc = cw_sum(loc, scr);
        WC_TR(10);
        if (tid == 0) a.part[(int64_t)u * 2 * kMaxCpu + ((i + 1) & 1) * kMaxCpu + c] = loc;
        // rounds 0..i complete: this CTA's F row i is globally visible for the producer's TMA reads
        cw_group_barrier(a.bar + u, a.cpu, epoch++, &sh_rounds_done, i + 1);
        WC_TR(11);
    }
    if (tid == 0) flag_st(&sh_stop, 1);
    if (c == 0 && tid == 0) {
        a.r_eff[u] = i;
        double *stw = const_cast<double *>(st);
        stw[5] = T0;
        stw[6] = (double)i;                          // rounds run
        stw[7] = (double)i;                          // pivots drawn
        stw[8] = 0.5 * (double)i * (double)(i - 1);  // F rows re-read: sum over rounds q of q
        stw[9] = stw[8];                             // F-prefix dot work (one pivot per round)
    }
}

// Debug: print the per-round phase durations of CTA 0 (ns, averaged over round bins).
void dump_trace(unsigned long long *dtrace, int r, cudaStream_t st) {
    std::vector<unsigned long long> h((size_t)16 * r);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dtrace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(dtrace);
    const char *names[] = {"a1a", "a1a_sync", "a1b", "pivld", "st0_B", "st0_A", "st0_C",
                           "st1_B", "st1_A", "st1_C", "sum", "gbar"};
    for (int b0 = 0; b0 < r; b0 += r / 8 > 0 ? r / 8 : 1) {
        const int b1 = std::min(r, b0 + (r / 8 > 0 ? r / 8 : 1));
        double acc[12] = {0};
        int cnt = 0;
        for (int i = b0; i < b1; ++i) {
            const unsigned long long *t = &h[(size_t)i * 16];
            const unsigned long long prev = i > 0 ? h[(size_t)(i - 1) * 16 + 11] : t[0];
            if (!t[11]) continue;
            unsigned long long last = prev;
            for (int k = 0; k < 12; ++k) {
                if (!t[k]) continue;
                acc[k] += (double)(t[k] - last);
                last = t[k];
            }
            ++cnt;
        }
        if (!cnt) continue;
        std::fprintf(stderr, "[trace] rounds %4d-%4d:", b0, b1 - 1);
        for (int k = 0; k < 12; ++k) std::fprintf(stderr, " %s=%.0f", names[k], acc[k] / cnt);
        std::fprintf(stderr, "\n");
    }
}

template <typename T, int D>
int launch_select_td(const Dims &Dm, const void *K, const double *stats, SelectBufs b, uint64_t seed, uint64_t unit0,
                     int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    SelArgs a;
    a.K = K; a.stats = stats; a.nrm2 = b.nrm2; a.p = b.p; a.F = b.F; a.part = b.part; a.bar = b.bar;
    a.S = S; a.r_eff = r_eff; a.L = L; a.n = Dm.n; a.ldF = f_ld(Dm.n); a.units = Dm.units(); a.r = Dm.r;
    a.bins = Dm.bins; a.nb = Dm.nb; a.unit_n = Dm.unit_n;
    a.nstm = f_tile_nst(Dm.n, select_ctas_per_unit(Dm));
    a.cpu = select_ctas_per_unit(Dm); a.seed = seed; a.unit0 = unit0; a.trace = nullptr;
    {
        // keep the first F rows L2-resident: ~3/4 of L2 for F (the rest holds K, p and streams)
        int dev = 0, l2 = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        const char *env = std::getenv("WC_L2_KEEP_FRAC");
        const double frac = env ? std::atof(env) : 0.0;  // measured best: F streamed evict-first
        const double row_bytes = (double)a.units * (double)a.ldF * sizeof(double);
        a.rkeep = (int)std::min<double>(Dm.r, std::max(0.0, frac * l2 / row_bytes));
    }
    static const bool tracing = std::getenv("WC_SELECT_TRACE") != nullptr;
    if (tracing) cudaMalloc(&a.trace, sizeof(unsigned long long) * 16 * Dm.r);
    if (a.trace) cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long) * 16 * Dm.r, st);
    if (cudaMemsetAsync(b.bar, 0, sizeof(unsigned) * a.units, st) != cudaSuccess) return -1;
    if (cudaMemsetAsync(b.part, 0, sizeof(double) * 2 * kMaxCpu * a.units, st) != cudaSuccess) return -1;
    const dim3 grid(a.units * a.cpu);
    static const char *mode = std::getenv("WC_SELECT");  // "simple": the non-TMA kernel (A/B tests)
    if (!(mode && std::strcmp(mode, "simple") == 0)) {
        const size_t fixed = (size_t)(Dm.r + kCW * kST + 2 * D + 40) * sizeof(double) + 64 * sizeof(uint64_t);
        const size_t stage_bytes = (size_t)kRPS * kST * sizeof(double);
        const int NS = (int)std::min<size_t>(16, (220 * 1024 - fixed) / stage_bytes);
        const size_t smem = fixed + (size_t)NS * stage_bytes;
        auto kt = rpc_select_tma_kernel<T, D>;
        cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (a.cpu > 1) {
            void *args[] = {&a, (void *)&NS};
            if (cudaLaunchCooperativeKernel((const void *)kt, grid, dim3(kTmaThreads), args, smem, st) != cudaSuccess)
                return -1;
        } else {
            kt<<<grid, kTmaThreads, smem, st>>>(a, NS);
        }
        if (a.trace) dump_trace(a.trace, Dm.r, st);
        return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
    }
    const int threads = (Dm.n / a.cpu >= 384) ? kSelThreads : 256;
    const size_t smem = (size_t)(2 * D + Dm.r + (threads / 32) * kST + 2 * kST + 40) * sizeof(double);
    auto kern = rpc_select_kernel<T, D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
int launch_select_t(const Dims &Dm, const void *K, const double *stats, SelectBufs b, uint64_t seed, uint64_t unit0,
                    int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    switch (Dm.d) {
        case 16: return launch_select_td<T, 16>(Dm, K, stats, b, seed, unit0, S, r_eff, L, st);
        case 32: return launch_select_td<T, 32>(Dm, K, stats, b, seed, unit0, S, r_eff, L, st);
        case 64: return launch_select_td<T, 64>(Dm, K, stats, b, seed, unit0, S, r_eff, L, st);
        case 128: return launch_select_td<T, 128>(Dm, K, stats, b, seed, unit0, S, r_eff, L, st);
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

int launch_select(const Dims &D, const void *K, const double *stats, SelectBufs b, uint64_t seed, uint64_t unit0,
                  int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    if (D.dtype == 0) return launch_select_t<float>(D, K, stats, b, seed, unit0, S, r_eff, L, st);
    return launch_select_t<__nv_bfloat16>(D, K, stats, b, seed, unit0, S, r_eff, L, st);
}

}  // namespace wc
