// select_blocked.cu -- blocked ("accelerated") RPCholesky selection: SURVEY.md 8(f)-1, the
// oversampling route out of the sequential pivot loop the paper names as future work (P:678,
// citing accelerated RPCholesky), reading Z22 of DESIGN.md.
//
// Per block, with i pivots accepted and block-start residual diagonal p (T = sum p):
//   1. draw b candidates s_0..s_{b-1} i.i.d. from p / T by the Eq. 4 inverse CDF;
//      candidate c (global count) uses the pivot uniform of Philox counter c (reading Z2);
//   2. H[a][e] = h~(k_sa, k_se) - sum_{q<i} F[q,s_a] F[q,s_e],  H[a][a] = p[s_a];
//   3. in candidate order: accept s_j iff it is new and v_j p[s_j] < H[j][j] (v_j = the accept
//      uniform of counter c, Philox tag 'ACPT'); on acceptance eliminate j from H (Schur step);
//   4. the na accepted pivots run na F-form rounds (Alg 1 P:221-231 in the F form of P:844):
//        F[i+a, l] = (h~(k_l, k_sa) - sum_{q<i+a} F[q,l] F[q,s_a]) / sqrt(p_{s_a})
//        p_l <- max(p_l - F[i+a,l]^2, 0),  p_{s_a} <- 0.
// The accepted sequence has the law of sequential RPC; for a given seed it differs from the
// sequential kernel unless b = 1.  The tests compare it with the fp64 CPU oracle of this exact
// procedure (test infrastructure under oracle/, which shares nothing with this file).
//
// Why it is faster: step 4 reads the F prefix F[0:i, :] ONCE per block instead of once per
// round -- the na rounds become one fp64 GEMM  G = h~(K, K_A) - F[0:i,:]^T F[0:i, A]  (n x i x na)
// plus an na x na triangular correction per key.  The F traffic, which dominates the sequential
// kernel (4 n r (r-1) bytes), drops by the mean accepted block size.
//
// Execution (one persistent kernel, `cpu` co-resident CTAs per unit, 8 compute warps + 1 TMA
// producer warp, one grid-group barrier per BLOCK):
//   - steps 1-3 run redundantly and identically in every CTA (fixed-order fp64), so all CTAs
//     agree on the accepted pivots without a second exchange: warp w draws candidates w, w+8 (a
//     warp inverse-CDF over the owning CTA's residual slice), the H entries are fixed-order dots
//     over gathered F columns (L2), the rejection is one warp (lane = column of H);
//   - the pre-phase (warp 0) runs the triangular recursion on the accepted pivots themselves to
//     get Fx[x][a] = F[i+a, s_x] and sqrt(p_{s_a}) -- the coefficients every key needs;
//   - step 4 streams the CTA's slice of F[0:i, :] through a TMA bulk-copy ring (as the
//     sequential kernel), one key per compute thread: na fp64 accumulators fed by broadcast
//     reads of the accepted columns, the kernel dots against the accepted centred keys from the
//     raw K row in registers, then the per-key triangle, the F row writes and the downdate.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "select_common.cuh"

namespace wc {

namespace {

constexpr int kBMax = 16;  // largest supported block size b

__device__ __forceinline__ double accept_uniform(uint64_t seed, uint32_t cand, uint64_t unit) {
    uint32_t c[4] = {cand, (uint32_t)unit, (uint32_t)(unit >> 32), 0x41435054u};  // 'ACPT'
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double x = (double)(c[0] >> 5), y = (double)(c[1] >> 6);
    return (x * 67108864.0 + y) * (1.0 / 9007199254740992.0);
}

struct BlkArgs {
    const void *K;
    double *stats;
    const double *nrm2;
    double *p;      // [2][units][n]
    double *F;      // per unit tile-major [cpu][nst][r][256]
    double *part;   // [units][2][kMaxCpu]
    unsigned *bar;  // [units]
    int32_t *S;
    int32_t *r_eff;
    double *L;
    int64_t n;
    int units, r, cpu, b;
    uint64_t seed;
    unsigned long long *trace;  // debug (WC_SELECT_TRACE): [r][16] globaltimer stamps of CTA 0 per block
};

__device__ __forceinline__ unsigned long long btimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define WC_BTR(k)                                                                                   \
    do {                                                                                            \
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && blk < a.r) a.trace[blk * 16 + (k)] = btimer(); \
    } while (0)

template <typename T, int D>
__global__ void __launch_bounds__(kTmaThreads, 1) rpc_select_blocked_kernel(BlkArgs a, int NS) {
    using KR = KRow<T, D>;
    extern __shared__ __align__(128) unsigned char smraw[];
    double *ring = reinterpret_cast<double *>(smraw);  // [NS][kRPS][kST]
    double *FsT = ring + (size_t)NS * kRPS * kST;       // [r][kBMax]   F[q, s] of the candidates / accepted
    double *kcT = FsT + (size_t)a.r * kBMax;            // [D][kBMax]   centred candidate keys (fp64)
    double *Hw = kcT + D * kBMax;                        // [kBMax][kBMax] working H (Schur updates)
    double *H0 = Hw + kBMax * kBMax;                     // [kBMax][kBMax] block-start H
    double *Fx = H0 + kBMax * kBMax;                     // [kBMax][kBMax] Fx[x][a] = F[i+a, s_x]
    double *cp = Fx + kBMax * kBMax;                     // [kBMax] block-start p[s_j]
    double *c0r = cp + kBMax;                            // [kBMax] <kbar, k_sj - kbar> per candidate
    double *c0 = c0r + kBMax;                            // [kBMax] ... per accepted pivot (0-padded)
    double *rsp = c0 + kBMax;                            // [kBMax] sqrt(p_{s_a}) at round i+a
    double *vac = rsp + kBMax;                           // [kBMax] accept uniforms
    double *kb = vac + kBMax;                            // [D]
    double *scr = kb + D;                                // [40]
    int *cs = reinterpret_cast<int *>(scr + 40);         // [kBMax] candidates
    int *sA = cs + kBMax;                                // [kBMax] accepted pivots (in order)
    int *jA = sA + kBMax;                                // [kBMax] their candidate slots
    uint64_t *full = reinterpret_cast<uint64_t *>(jA + kBMax);
    uint64_t *empty = full + NS;
    __shared__ volatile int sh_stop;
    __shared__ volatile long long sh_req;  // (block + 1) << 32 | rows to stream
    __shared__ volatile int sh_dummy;
    __shared__ int sh_na;

    const int tid = threadIdx.x, lane = tid & 31, w = warp_index();
    const int u = blockIdx.x / a.cpu, c = blockIdx.x % a.cpu;
    const int64_t n = a.n;
    const int64_t chunk = ((ceil_div(n, a.cpu) + 31) / 32) * 32;
    const int64_t lo = std::min<int64_t>(n, (int64_t)c * chunk), hi = std::min<int64_t>(n, lo + chunk);
    const int nst = (int)ceil_div(hi - lo, kST);
    const int bsz = a.b;

    const T *Ku = static_cast<const T *>(a.K) + (int64_t)u * n * D;
    double *st = a.stats + (int64_t)u * (kStatsHead + D);
    double *Fu = a.F + (int64_t)u * a.cpu * chunk * a.r;
    double *Fc = Fu + (int64_t)c * chunk * a.r;
    auto tile_w = [&](int k) -> int { return (int)std::min<int64_t>(kST, chunk - (int64_t)k * kST); };
    // address of F[q, key] in the tile-major layout
    auto fptr = [&](int q, int64_t key) -> const double * {
        const int64_t cc = key / chunk, off = key - cc * chunk;
        const int kk = (int)(off / kST);
        const int64_t wk = std::min<int64_t>(kST, chunk - (int64_t)kk * kST);
        return Fu + cc * chunk * a.r + (int64_t)kk * kST * a.r + (int64_t)q * wk + (off % kST);
    };

    if (tid == 0) {
        for (int q = 0; q < NS; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kCW);
        }
        sh_stop = 0;
        sh_req = 0;
        fence_mbar_init();
    }
    __syncthreads();  // the only CTA-wide barrier: everything after is role-specific

    if (w == kCW) {
        // ================= producer warp: streams F[0:i, own slice] once per block =================
        if (lane == 0) {
            int stage = 0;
            uint32_t ph = 0, issued = 0, par = 0;
            long long seen = 0;
            while (true) {
                long long req;
                while (((req = sh_req) >> 32) == seen) {
                    if (sh_stop) goto drain;
                    __nanosleep(32);
                }
                seen = req >> 32;
                const int rows = (int)(req & 0xffffffffLL);
                for (int k = 0; k < nst; ++k) {
                    const double *blk = Fc + (int64_t)k * a.r * kST;
                    const int wk = tile_w(k);
                    for (int j0 = 0; j0 < rows; j0 += kRPS) {
                        const int nr = min(kRPS, rows - j0);
                        const uint32_t bytes = (uint32_t)(nr * wk * sizeof(double));
                        while (!mbar_try_wait(&empty[stage], ph ^ 1u)) {
                            if (sh_stop) goto drain;
                        }
                        mbar_arrive_expect_tx(&full[stage], bytes);
                        bulk_g2s(ring + (size_t)stage * kRPS * kST, blk + (int64_t)j0 * wk, bytes, &full[stage]);
                        issued |= 1u << stage;
                        par = (par & ~(1u << stage)) | (ph << stage);
                        if (++stage == NS) { stage = 0; ph ^= 1u; }
                    }
                }
            }
        drain:
            for (int q = 0; q < NS; ++q)
                if (issued & (1u << q)) mbar_wait(&full[q], (par >> q) & 1u);
        }
        return;
    }

    // ================= compute warps (256 threads) =================
    const double g = st[1], mstar = st[2];
    double *p0 = a.p + (int64_t)u * n;
    double *p1 = a.p + ((int64_t)a.units + u) * n;
    double *partu = a.part + (int64_t)u * 2 * kMaxCpu;
    for (int j = tid; j < D; j += kCT) kb[j] = st[kStatsHead + j];

    // p <- kernel diagonal h~(k_l, k_l) (Alg 1)
    double loc = 0.0;
    for (int64_t l = lo + tid; l < hi; l += kCT) {
        const double v = exp(__dadd_rn(__dmul_rn(g, a.nrm2[(int64_t)u * n + l]), -mstar));
        p0[l] = v;
        loc += v;
    }
    loc = cw_sum(loc, scr);
    if (tid == 0) partu[c] = loc;
    unsigned epoch = 1;
    cw_group_barrier(a.bar + u, a.cpu, epoch++, &sh_dummy, 0);

    int rstage = 0;
    uint32_t rph = 0;
    double T0 = 0.0, theta = 0.0;
    int i = 0, blk = 0;
    uint32_t cbase = 0;
    double fread = 0.0;
    while (i < a.r) {
        double *cur = (blk & 1) ? p1 : p0;
        double *nxt = (blk & 1) ? p0 : p1;
        const double *pc = partu + (blk & 1) * kMaxCpu;
        double *pn = partu + ((blk + 1) & 1) * kMaxCpu;
        WC_BTR(0);

        // ---- 1a: total residual T over the per-CTA sums (every warp, identical fixed order)
        const int per = (a.cpu + 31) / 32;
        const int b0 = lane * per, b1 = min(a.cpu, b0 + per);
        constexpr int kPer = 8;  // fast path (cpu <= 256): the lane's CTA sums kept in registers
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
        if (blk == 0) {
            T0 = Ttot;
            theta = 1000.0 * (double)a.r * 2.220446049250313e-16 * T0;
        }
        if (Ttot <= theta) break;  // exhausted (reading Z3), tested at block starts
        if (tid == 0) sh_req = ((long long)(blk + 1) << 32) | (long long)i;  // producer: stream F[0:i]

        // ---- 1b: candidates, warp w draws j = w, w + 8 (Eq. 4 inverse CDF, strict '>')
        for (int j = w; j < bsz; j += kCW) {
            const double t = pivot_uniform(a.seed, cbase + (uint32_t)j, (uint64_t)u) * Ttot;
            const unsigned hit = __ballot_sync(0xffffffffu, b1 > b0 && incl > t);
            const unsigned pos = __ballot_sync(0xffffffffu, b1 > b0 && v > 0.0);
            const int Ln = hit ? __ffs(hit) - 1 : 31 - __clz(pos);
            int cstar = 0;
            double tp = 0.0;
            if (lane == Ln) {
                double acc = incl - v;
                int csel = -1, last = -1;
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
                    if (csel < 0 && hit && nacc > t) { csel = cc; excl = acc; }
                    acc = nacc;
                }
                if (csel < 0) { csel = last; excl = last_excl; }  // rounding fallback (reading Z2)
                cstar = csel;
                tp = t - excl;
            }
            cstar = __shfl_sync(0xffffffffu, cstar, Ln);
            tp = __shfl_sync(0xffffffffu, tp, Ln);
            // warp inverse CDF over c*'s slice of the block-start residual
            const int64_t slo = std::min<int64_t>(n, (int64_t)cstar * chunk);
            const int64_t shi = std::min<int64_t>(n, slo + chunk);
            const int64_t per2 = ceil_div(shi - slo, 32);
            const int64_t q0 = slo + (int64_t)lane * per2, q1 = std::min<int64_t>(shi, q0 + per2);
            constexpr int kSl = 16;  // fast path (slice <= 512 keys): the lane's residuals in registers
            double pr[kSl];
            double v2 = 0.0;
            if (per2 <= kSl) {
#pragma unroll
                for (int q = 0; q < kSl; ++q) pr[q] = (q0 + q < q1) ? __ldcg(cur + q0 + q) : 0.0;
#pragma unroll
                for (int q = 0; q < kSl; ++q) v2 += pr[q];
            } else {
                for (int64_t l = q0; l < q1; ++l) v2 += __ldcg(cur + l);
            }
            double inc2 = v2;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, inc2, o);
                if (lane >= o) inc2 += y;
            }
            double run = inc2 - v2;
            int found = INT_MAX, lastpos = -1;
            double fval = 0.0, lval = 0.0;
            if (per2 <= kSl) {
#pragma unroll
                for (int q = 0; q < kSl; ++q) {
                    if (q0 + q < q1) {
                        const double pl = pr[q];
                        if (pl > 0.0) { lastpos = (int)(q0 + q); lval = pl; }
                        run += pl;
                        if (found == INT_MAX && run > tp) { found = (int)(q0 + q); fval = pl; }
                    }
                }
            } else {
                for (int64_t l = q0; l < q1; ++l) {
                    const double pl = __ldcg(cur + l);
                    if (pl > 0.0) { lastpos = (int)l; lval = pl; }
                    run += pl;
                    if (found == INT_MAX && run > tp) { found = (int)l; fval = pl; }
                }
            }
            const int smin = __reduce_min_sync(0xffffffffu, found);
            int s;
            double psv;
            if (smin != INT_MAX) {
                s = smin;
                const int src = __ffs(__ballot_sync(0xffffffffu, found == smin)) - 1;
                psv = __shfl_sync(0xffffffffu, fval, src);
            } else {  // rounding fallback (reading Z2): last key with positive residual
                s = __reduce_max_sync(0xffffffffu, lastpos);
                const int src = __ffs(__ballot_sync(0xffffffffu, lastpos == s)) - 1;
                psv = __shfl_sync(0xffffffffu, lval, src);
            }
            if (lane == 0) {
                cs[j] = s;
                cp[j] = psv;
                vac[j] = accept_uniform(a.seed, cbase + (uint32_t)j, (uint64_t)u);
            }
        }
        cw_sync();
        WC_BTR(1);

        // ---- 2: candidate data: centred keys (fp64), F[0:i, s_j] (gathered from L2)
        for (int idx = tid; idx < bsz * D; idx += kCT) {
            const int j = idx / D, e = idx - j * D;
            kcT[e * kBMax + j] = __dadd_rn(to_f64(Ku[(int64_t)cs[j] * D + e]), -kb[e]);
        }
#pragma unroll 4
        for (int idx = tid; idx < bsz * i; idx += kCT) {
            const int q = idx / bsz, j = idx - q * bsz;
            FsT[q * kBMax + j] = __ldcg(fptr(q, cs[j]));
        }
        cw_sync();
        WC_BTR(2);
        // H off-diagonal: two threads per pair (a < e), halves combined in fixed order
        {
            const int npairs = bsz * (bsz - 1) / 2;
            const int pidx = tid >> 1, half = tid & 1;
            double kd = 0.0, fd = 0.0;
            int pa = 0, pe = 0;
            if (pidx < npairs) {
                int rem = pidx;
                while (rem >= bsz - 1 - pa) { rem -= bsz - 1 - pa; ++pa; }
                pe = pa + 1 + rem;
                double kd2 = 0.0, fd2 = 0.0;  // two chains per half (fixed order)
#pragma unroll 4
                for (int e = 2 * half; e < D; e += 4) {
                    kd = fma(kcT[e * kBMax + pa], kcT[e * kBMax + pe], kd);
                    kd2 = fma(kcT[(e + 1) * kBMax + pa], kcT[(e + 1) * kBMax + pe], kd2);
                }
                int q = 2 * half;
#pragma unroll 4
                for (; q + 1 < i; q += 4) {
                    fd = fma(FsT[q * kBMax + pa], FsT[q * kBMax + pe], fd);
                    fd2 = fma(FsT[(q + 1) * kBMax + pa], FsT[(q + 1) * kBMax + pe], fd2);
                }
                if (q < i) fd = fma(FsT[q * kBMax + pa], FsT[q * kBMax + pe], fd);
                kd += kd2;
                fd += fd2;
            }
            const double kd1 = __shfl_xor_sync(0xffffffffu, kd, 1);
            const double fd1 = __shfl_xor_sync(0xffffffffu, fd, 1);
            if (pidx < npairs && half == 0) {
                const double h = exp(__dadd_rn(__dmul_rn(g, kd + kd1), -mstar)) - (fd + fd1);
                H0[pa * kBMax + pe] = h;
                H0[pe * kBMax + pa] = h;
                Hw[pa * kBMax + pe] = h;
                Hw[pe * kBMax + pa] = h;
            }
            if (tid < bsz) {
                H0[tid * kBMax + tid] = cp[tid];
                Hw[tid * kBMax + tid] = cp[tid];
                double s0 = 0.0;
                for (int e = 0; e < D; ++e) s0 = fma(kb[e], kcT[e * kBMax + tid], s0);
                c0r[tid] = s0;
            }
        }
        cw_sync();
        WC_BTR(3);

        // ---- 3: rejection in candidate order (warp 0; lane e owns column e of H)
        if (w == 0) {
            int na = 0;
            for (int j = 0; j < bsz; ++j) {
                if (i + na >= a.r) break;
                const int sj = cs[j];
                bool dup = false;
                for (int x = 0; x < na; ++x) dup |= (sA[x] == sj);
                const double hjj = Hw[j * kBMax + j];
                const bool acc = !dup && (__dmul_rn(vac[j], cp[j]) < hjj);
                if (acc) {
                    if (lane > j && lane < bsz) {
                        const double hje = Hw[j * kBMax + lane];
                        for (int x = j + 1; x < bsz; ++x)
                            Hw[x * kBMax + lane] =
                                __dsub_rn(Hw[x * kBMax + lane], __ddiv_rn(__dmul_rn(Hw[x * kBMax + j], hje), hjj));
                    }
                    if (lane == 0) {
                        sA[na] = sj;
                        jA[na] = j;
                    }
                    ++na;
                }
                __syncwarp();
            }
            // pre-phase: the triangular recursion on the accepted pivots themselves (lane x = pivot
            // s_x) gives Fx[x][a] = F[i+a, s_x] and sqrt(p_{s_a}) just before round i+a
            const int x = lane;
            double px = (x < na) ? cp[jA[x]] : 0.0;
            for (int aa = 0; aa < na; ++aa) {
                const double rs = sqrt(__shfl_sync(0xffffffffu, px, aa));
                if (x < na) {
                    double cv = H0[jA[x] * kBMax + jA[aa]];
                    for (int a2 = 0; a2 < aa; ++a2) cv = fma(-Fx[x * kBMax + a2], Fx[aa * kBMax + a2], cv);
                    const double f = cv / rs;
                    Fx[x * kBMax + aa] = f;
                    const double q = __dadd_rn(px, -__dmul_rn(f, f));
                    px = (x == aa || !(q > 0.0)) ? 0.0 : q;
                }
                if (lane == 0) rsp[aa] = rs;
                __syncwarp();
            }
            if (lane < kBMax) c0[lane] = lane < na ? c0r[jA[lane]] : 0.0;
            if (lane == 0) sh_na = na;
        }
        cw_sync();
        WC_BTR(4);
        const int na = sh_na;
        // compact the candidate columns of FsT / kcT to accepted order, zero padding
        for (int row = tid; row < i + D; row += kCT) {
            double *R = row < i ? FsT + (size_t)row * kBMax : kcT + (size_t)(row - i) * kBMax;
            double tmp[kBMax];
#pragma unroll
            for (int x = 0; x < kBMax; ++x) tmp[x] = x < na ? R[jA[x]] : 0.0;
#pragma unroll
            for (int x = 0; x < kBMax; ++x) R[x] = tmp[x];
        }
        cw_sync();
        // owner CTA of each accepted pivot: S and L[i+x][0:i] = F[0:i, s_x]
        for (int x = 0; x < na; ++x) {
            const int s = sA[x];
            if (s >= lo && s < hi) {
                for (int q = tid; q < i; q += kCT) a.L[((int64_t)u * a.r + i + x) * a.r + q] = FsT[(size_t)q * kBMax + x];
                if (tid == 0) a.S[(int64_t)u * a.r + i + x] = s;
            }
        }

        WC_BTR(5);
        // ---- 4: na F-form rounds over this CTA's keys, one key per thread per super-tile
        loc = 0.0;
        for (int k = 0; k < nst; ++k) {
            const int64_t l = lo + (int64_t)k * kST + tid;
            const bool own = l < hi;
            const int wk = tile_w(k);
            double *Fk = Fc + (int64_t)k * a.r * kST + tid;
            const double pcur = own ? __ldcg(cur + l) : 0.0;
            // kernel dots <k_l, k_sa - kbar> against the accepted centred keys; the raw K row is
            // read in chunks of <= 16 16-byte vectors (register budget: 9 warps => <= 168 regs)
            double hv[kBMax];
#pragma unroll
            for (int x = 0; x < kBMax; ++x) hv[x] = 0.0;
            constexpr int kVec = KR::kVec, kEl = KR::kEl, kChunk = kVec < 16 ? kVec : 16;
#pragma unroll
            for (int q0 = 0; q0 < kVec; q0 += kChunk) {
                uint4 kv[kChunk];
                const uint4 *kp = reinterpret_cast<const uint4 *>(Ku + (own ? l : lo) * D) + q0;
#pragma unroll
                for (int q = 0; q < kChunk; ++q) kv[q] = own ? __ldg(kp + q) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int q = 0; q < kChunk; ++q) {
                    const uint32_t wd[4] = {kv[q].x, kv[q].y, kv[q].z, kv[q].w};
#pragma unroll
                    for (int e = 0; e < kEl; ++e) {
                        double xe;
                        if constexpr (sizeof(T) == 2) {
                            const uint32_t bits = (e & 1) ? (wd[e >> 1] & 0xffff0000u) : (wd[e >> 1] << 16);
                            xe = (double)__uint_as_float(bits);
                        } else {
                            xe = (double)__uint_as_float(wd[e]);
                        }
                        const double2 *kr = reinterpret_cast<const double2 *>(kcT + ((q0 + q) * kEl + e) * kBMax);
#pragma unroll
                        for (int x2 = 0; x2 < kBMax / 2; ++x2) {
                            const double2 kk = kr[x2];
                            hv[2 * x2] = fma(xe, kk.x, hv[2 * x2]);
                            hv[2 * x2 + 1] = fma(xe, kk.y, hv[2 * x2 + 1]);
                        }
                    }
                }
            }
#pragma unroll
            for (int x = 0; x < kBMax; ++x)
                if (x < na) hv[x] = exp(__dadd_rn(__dmul_rn(g, hv[x] - c0[x]), -mstar));
            if (k == 0) WC_BTR(6);
            // F-prefix dots: rows 0..i-1 of this super-tile from the ring
            double acc[kBMax];
#pragma unroll
            for (int x = 0; x < kBMax; ++x) acc[x] = 0.0;
            for (int j0 = 0; j0 < i; j0 += kRPS) {
                const int nr = min(kRPS, i - j0);
                mbar_wait(&full[rstage], rph);
                const double *src = ring + (size_t)rstage * kRPS * kST + tid;
                for (int rr = 0; rr < nr; ++rr) {
                    const double xv = tid < wk ? src[rr * wk] : 0.0;
                    const double2 *fr = reinterpret_cast<const double2 *>(FsT + (size_t)(j0 + rr) * kBMax);
#pragma unroll
                    for (int x2 = 0; x2 < kBMax / 2; ++x2) {
                        const double2 ff = fr[x2];
                        acc[2 * x2] = fma(xv, ff.x, acc[2 * x2]);
                        acc[2 * x2 + 1] = fma(xv, ff.y, acc[2 * x2 + 1]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[rstage]);
                if (++rstage == NS) {
                    rstage = 0;
                    rph ^= 1u;
                }
            }
            if (k == 0) WC_BTR(7);
            // per-key triangle over the block's rounds, F row writes, downdate
            if (own) {
                double f[kBMax];
                double pl = pcur;
#pragma unroll
                for (int aa = 0; aa < kBMax; ++aa) {
                    f[aa] = 0.0;
                    if (aa < na) {
                        double cv = hv[aa] - acc[aa];
#pragma unroll
                        for (int a2 = 0; a2 < aa; ++a2) cv = fma(-f[a2], Fx[aa * kBMax + a2], cv);
                        const double fv = cv / rsp[aa];
                        f[aa] = fv;
                        Fk[(int64_t)(i + aa) * wk] = fv;
                        const double q = __dadd_rn(pl, -__dmul_rn(fv, fv));
                        pl = q > 0.0 ? q : 0.0;
                        if (l == sA[aa]) pl = 0.0;
                    }
                }
                nxt[l] = pl;
                loc += pl;
                for (int aa = 0; aa < na; ++aa) {
                    if (l == sA[aa]) {
                        double *Lrow = a.L + ((int64_t)u * a.r + i + aa) * a.r + i;
#pragma unroll
                        for (int a2 = 0; a2 < kBMax; ++a2)
                            if (a2 <= aa) Lrow[a2] = f[a2];
                    }
                }
            }
        }
        WC_BTR(8);
        fence_proxy_async_global();  // this block's F rows are read by later TMA copies
        loc = cw_sum(loc, scr);
        if (tid == 0) pn[c] = loc;
        WC_BTR(9);
        fread += (double)i;
        i += na;
        cbase += (uint32_t)bsz;
        ++blk;
        cw_group_barrier(a.bar + u, a.cpu, epoch++, &sh_dummy, 0);
    }
    if (tid == 0) sh_stop = 1;
    if (c == 0 && tid == 0) {
        a.r_eff[u] = i;
        st[5] = T0;
        st[6] = (double)blk;    // blocks run
        st[7] = (double)cbase;  // candidates drawn
        st[8] = fread;          // F rows re-read: sum over blocks of the block-start i
    }
}

// Debug: per-block phase durations of CTA 0 (ns), printed per block.
void dump_block_trace(unsigned long long *dtrace, int r, cudaStream_t st) {
    std::vector<unsigned long long> h((size_t)16 * r);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dtrace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(dtrace);
    const char *names[] = {"cand", "gather", "H", "accept", "compact", "t0_kdot", "t0_fdot", "tiles", "sum",
                           "gbar"};
    for (int b = 0; b < r; ++b) {
        const unsigned long long *t = &h[(size_t)b * 16];
        if (!t[0] || !t[9]) break;
        std::fprintf(stderr, "[btrace] block %3d:", b);
        unsigned long long last = t[0];
        for (int k = 1; k <= 10; ++k) {
            const unsigned long long v = (k == 10) ? (b + 1 < r ? h[(size_t)(b + 1) * 16] : 0) : t[k];
            if (!v) continue;
            std::fprintf(stderr, " %s=%llu", names[k - 1], v - last);
            last = v;
        }
        std::fprintf(stderr, "\n");
    }
}

template <typename T, int D>
int launch_blocked_td(const Dims &Dm, const void *K, double *stats, SelectBufs b, uint64_t seed, int block,
                      int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    BlkArgs a;
    a.K = K; a.stats = stats; a.nrm2 = b.nrm2; a.p = b.p; a.F = b.F; a.part = b.part; a.bar = b.bar;
    a.S = S; a.r_eff = r_eff; a.L = L; a.n = Dm.n; a.units = Dm.units(); a.r = Dm.r;
    a.cpu = select_ctas_per_unit(Dm); a.b = block; a.seed = seed; a.trace = nullptr;
    static const bool tracing = std::getenv("WC_SELECT_TRACE") != nullptr;
    if (tracing && cudaMalloc(&a.trace, sizeof(unsigned long long) * 16 * Dm.r) == cudaSuccess)
        cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long) * 16 * Dm.r, st);
    const size_t fixed = ((size_t)Dm.r * kBMax + (size_t)D * kBMax + 3 * kBMax * kBMax + 5 * kBMax + D + 40) *
                             sizeof(double) + 3 * kBMax * sizeof(int) + 64;
    const size_t stage_bytes = (size_t)kRPS * kST * sizeof(double);
    if (fixed + 2 * stage_bytes + 2 * 16 > 220 * 1024) return -2;  // r too large for the shared-memory plan
    int NS = (int)std::min<size_t>(12, (220 * 1024 - fixed) / (stage_bytes + 16));
    const size_t smem = fixed + (size_t)NS * (stage_bytes + 16);
    auto kt = rpc_select_blocked_kernel<T, D>;
    cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaMemsetAsync(b.bar, 0, sizeof(unsigned) * a.units, st) != cudaSuccess) return -1;
    if (cudaMemsetAsync(b.part, 0, sizeof(double) * 2 * kMaxCpu * a.units, st) != cudaSuccess) return -1;
    const dim3 grid(a.units * a.cpu);
    if (a.cpu > 1) {
        void *args[] = {&a, (void *)&NS};
        if (cudaLaunchCooperativeKernel((const void *)kt, grid, dim3(kTmaThreads), args, smem, st) != cudaSuccess)
            return -1;
    } else {
        kt<<<grid, kTmaThreads, smem, st>>>(a, NS);
    }
    if (a.trace) dump_block_trace(a.trace, Dm.r, st);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T>
int launch_blocked_t(const Dims &Dm, const void *K, double *stats, SelectBufs b, uint64_t seed, int block,
                     int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    switch (Dm.d) {
        case 16: return launch_blocked_td<T, 16>(Dm, K, stats, b, seed, block, S, r_eff, L, st);
        case 32: return launch_blocked_td<T, 32>(Dm, K, stats, b, seed, block, S, r_eff, L, st);
        case 64: return launch_blocked_td<T, 64>(Dm, K, stats, b, seed, block, S, r_eff, L, st);
        case 128: return launch_blocked_td<T, 128>(Dm, K, stats, b, seed, block, S, r_eff, L, st);
    }
    return -1;
}

}  // namespace

int select_blocked_max_block() { return kBMax; }

int launch_select_blocked(const Dims &D, const void *K, double *stats, SelectBufs b, uint64_t seed, int block,
                          int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    if (block < 2 || block > kBMax) return -1;
    if (D.dtype == 0) return launch_blocked_t<float>(D, K, stats, b, seed, block, S, r_eff, L, st);
    return launch_blocked_t<__nv_bfloat16>(D, K, stats, b, seed, block, S, r_eff, L, st);
}

}  // namespace wc
