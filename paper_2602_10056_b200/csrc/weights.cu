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
                                                              const double *__restrict__ stats, int64_t n_buf,
                                                              int r, int splits, float *__restrict__ Ypart, int bins,
                                                              int64_t nb, int64_t unit_n) {
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
    const SubUnit sub = sub_unit(u, n_buf, bins, nb, unit_n);  // keys of this (sub-)unit (Z13)
    const int64_t n = sub.count;
    const T *Ku = K + sub.base * D;
    const T *Vu = V + sub.base * D;
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

// Y~ = sum over n-splits of the fp32 partials, in fixed split order, in fp64.
template <int D>
__global__ void __launch_bounds__(256) weights_reduce_kernel(const float *__restrict__ Ypart,
                                                             const int32_t *__restrict__ r_eff, int r, int splits,
                                                             double *__restrict__ Y) {
    pdl_wait();
    constexpr int DC = D + 1;
    const int u = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (a, c) flattened
    if (e >= (int64_t)r * DC) return;
    const int a = (int)(e / DC);
    double y = 0.0;
    if (a < r_eff[u]) {
        const float *src = Ypart + (int64_t)u * splits * r * DC + e;
        int sp = 0;
        for (; sp + 32 <= splits; sp += 32) {  // 32 independent loads in flight, summed in split order
            float t[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) t[k] = __ldg(src + (int64_t)(sp + k) * r * DC);
#pragma unroll
            for (int k = 0; k < 32; ++k) y += (double)t[k];
        }
        if (sp < splits) {  // the remaining < 32 splits, all loads in flight
            float t[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) t[k] = sp + k < splits ? __ldg(src + (int64_t)(sp + k) * r * DC) : 0.f;
#pragma unroll
            for (int k = 0; k < 32; ++k)
                if (sp + k < splits) y += (double)t[k];
        }
    }
    Y[(int64_t)u * r * DC + e] = y;
}

// A4: X = L^{-T} (L^{-1} Y~), blocked in 32-row panels.  weights_dinv_kernel inverts the 32 x 32
// diagonal blocks of L once per unit (one warp per block; lane c owns column c of the inverse, a
// sequential substitution with broadcast reads of the block), so that the panel solves are plain
// 32 x 32 products; the sequential part of the solve is only the panel order.
constexpr int kPB = 32;   // panel size
constexpr int kCBs = 128; // L columns (forward) / rows (backward) fetched per round trip

// Inverse of the 32 x 32 diagonal block blk of unit u's L (one warp; lane c owns column c of the
// inverse, a sequential substitution with broadcast reads of the block).
__device__ __forceinline__ void dinv_block(const double *__restrict__ L, const int32_t *__restrict__ r_eff, int r,
                                           double *__restrict__ Dinv, int blk, int u, int lane,
                                           double (*Lb)[kPB + 1]) {
    const int q = r_eff[u], p0 = blk * kPB;
    if (p0 >= q) return;
    const int nb = min(kPB, q - p0);
    const double *Lu = L + (int64_t)u * r * r;
#pragma unroll 8
    for (int i = 0; i < kPB; ++i) Lb[i][lane] = (i < nb && lane <= i) ? __ldg(Lu + (int64_t)(p0 + i) * r + p0 + lane) : 0.0;
    __syncwarp();
    // 1 / L_ii computed by lane i up front, so that no division sits on the substitution's dependent chain
    const double rdi = lane < nb ? 1.0 / Lb[lane][lane] : 0.0;
    // column c = lane of inv(Lb): x_i = (delta_ic - sum_{j<i} L_ij x_j) / L_ii, i = c .. nb-1
    double x[kPB];
#pragma unroll
    for (int i = 0; i < kPB; ++i) {
        double acc = (i == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int j = 0; j < i; ++j) acc = fma(-Lb[i][j], x[j], acc);
        const double ri = __shfl_sync(0xffffffffu, rdi, i);
        x[i] = (i < nb && i >= lane) ? acc * ri : 0.0;
    }
    double *Du = Dinv + ((int64_t)u * ((r + kPB - 1) / kPB) + blk) * kPB * kPB;
#pragma unroll
    for (int i = 0; i < kPB; ++i) Du[i * kPB + lane] = x[i];  // row-major inverse, lower triangular
}

__global__ void __launch_bounds__(32) weights_dinv_kernel(const double *__restrict__ L, const int32_t *__restrict__ r_eff,
                                                          int r, double *__restrict__ Dinv) {
    pdl_wait();
    __shared__ double Lb[kPB][kPB + 1];
    dinv_block(L, r_eff, r, Dinv, blockIdx.x, blockIdx.y, threadIdx.x, Lb);
}

// Coreset key row a of unit u for the attend: KS[u][a] = K[S[u][a]] (zeros past r_eff).
template <typename T, int D>
__device__ __forceinline__ void gather_ks_row(const T *__restrict__ K, const int32_t *__restrict__ S,
                                              const int32_t *__restrict__ r_eff, int64_t n, int r, T *__restrict__ KS,
                                              int bins, int64_t nb, int64_t unit_n, int u, int a) {
    const int q = r_eff[u];
    const int s = a < q ? S[(int64_t)u * r + a] : -1;
    for (int j = threadIdx.x; j < D; j += blockDim.x)
        KS[((int64_t)u * r + a) * D + j] = s >= 0 ? K[(sub_unit(u, n, bins, nb, unit_n).base + s) * D + j] : from_f32<T>(0.f);
}

// weights_reduce_kernel + the diagonal-block inverses + the K_S gather in one launch (single-GPU
// path): blocks [0, nred) reduce the split partials, blocks [nred, nred + nbl) invert one diagonal
// block each, blocks [nred + nbl, nred + nbl + r) gather one coreset key row each (all depend only on
// earlier kernels, so they run side by side).
template <typename T, int D>
__global__ void __launch_bounds__(256) weights_reduce_dinv_kernel(const float *__restrict__ Ypart,
                                                                  const int32_t *__restrict__ r_eff, int r, int splits,
                                                                  double *__restrict__ Y, const double *__restrict__ L,
                                                                  double *__restrict__ Dinv, int nred, int nbl,
                                                                  const T *__restrict__ K, const int32_t *__restrict__ S,
                                                                  T *__restrict__ KS, int64_t n, int bins, int64_t nb,
                                                                  int64_t unit_n) {
    pdl_wait();
    __shared__ double Lb[kPB][kPB + 1];
    constexpr int DC = D + 1;
    const int u = blockIdx.y;
    if ((int)blockIdx.x >= nred + nbl) {
        gather_ks_row<T, D>(K, S, r_eff, n, r, KS, bins, nb, unit_n, u, (int)blockIdx.x - nred - nbl);
        return;
    }
    if ((int)blockIdx.x >= nred) {
        if (threadIdx.x < 32) dinv_block(L, r_eff, r, Dinv, blockIdx.x - nred, u, threadIdx.x, Lb);
        return;
    }
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (a, c) flattened
    if (e >= (int64_t)r * DC) return;
    const int a = (int)(e / DC);
    double y = 0.0;
    if (a < r_eff[u]) {
        const float *src = Ypart + (int64_t)u * splits * r * DC + e;
        int sp = 0;
        for (; sp + 32 <= splits; sp += 32) {  // 32 independent loads in flight, summed in split order
            float t[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) t[k] = __ldg(src + (int64_t)(sp + k) * r * DC);
#pragma unroll
            for (int k = 0; k < 32; ++k) y += (double)t[k];
        }
        if (sp < splits) {  // the remaining < 32 splits, all loads in flight
            float t[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) t[k] = sp + k < splits ? __ldg(src + (int64_t)(sp + k) * r * DC) : 0.f;
#pragma unroll
            for (int k = 0; k < 32; ++k)
                if (sp + k < splits) y += (double)t[k];
        }
    }
    Y[(int64_t)u * r * DC + e] = y;
}

// The solve is a chain of steps: per panel P (kPB rows), CHUNK steps (acc -= L-block . z over kCBs
// already-solved rows) and one DIAG step (z_P = Dinv_PP . acc); forward over P = 0.., then backward
// (L^T) over P = npan-1..0.  No L or Dinv load depends on z, so the operands of the next kSolveNS-1
// steps are in flight (cp.async, zero-filled out of range, transposes done by the copy placement)
// while the current step computes: the chain carries shared-memory latency only.
constexpr int kSolveNS = 4;                              // operand ring stages
constexpr int kSolveMaxSteps = 2 * (kMaxR / kPB) * (kMaxR / kCBs + 1);  // r <= kMaxR is checked at the ABI

// 8-byte async copy, zero-filled (no global read) when !ok; `safe` is any valid global address
__device__ __forceinline__ void cp_async8_zfill(double *dst, const double *src, bool ok, const double *safe) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(ok ? src : safe),
                 "r"(ok ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// C RHS columns per CTA, 256 threads: thread t owns panel row t / 8, column (t / PARTS) % C and the
// part t % PARTS of every dot (PARTS = 8 / C, combined by shuffles).  C = 2 (65 CTAs per unit at
// d = 128) when there are few units, C = 8 when there are many (binned sub-units).  The operand ring
// stage holds kPB rows of lb = min(kCBs, r) + 1 doubles (>= kPB + 1 for the Dinv blocks).
template <int D, int C>
__global__ void __launch_bounds__(256) weights_solve_kernel(const double *__restrict__ Y,
                                                            const double *__restrict__ L,
                                                            const double *__restrict__ Dinv,
                                                            const int32_t *__restrict__ r_eff, int r,
                                                            float *__restrict__ X) {
    pdl_wait();
    constexpr int DC = D + 1, PARTS = 8 / C;
    const int lb = min(kCBs, r) + 1, sbuf = kPB * max(lb, kPB + 1);
    extern __shared__ double zs[];  // z[r][C], then the operand ring [kSolveNS][sbuf]
    __shared__ double tP[kPB][C];
    __shared__ int steps[kSolveMaxSteps];
    __shared__ int nsteps;
    const int u = blockIdx.y, tid = threadIdx.x;
    const int cbase = blockIdx.x * C;
    const int q = r_eff[u];
    const int nbl = (r + kPB - 1) / kPB;
    const double *Lu = L + (int64_t)u * r * r;
    const double *Du = Dinv + (int64_t)u * nbl * kPB * kPB;
    float *Xu = X + (int64_t)u * r * DC;
    double *ring = zs + (size_t)r * C;
    const int npan = (q + kPB - 1) / kPB;
    auto nch = [&](int dir, int P) {
        const int p0 = P * kPB, pe = min(p0 + kPB, q);
        return dir == 0 ? (p0 + kCBs - 1) / kCBs : (q - pe + kCBs - 1) / kCBs;
    };
    if (tid == 0) {  // step list: dir << 24 | P << 12 | (chunk + 1), chunk -1 = DIAG
        int k = 0;
        for (int P = 0; P < npan; ++P) {
            for (int c = 0; c < nch(0, P); ++c) steps[k++] = (P << 12) | (c + 1);
            steps[k++] = P << 12;
        }
        for (int P = npan - 1; P >= 0; --P) {
            for (int c = 0; c < nch(1, P); ++c) steps[k++] = (1 << 24) | (P << 12) | (c + 1);
            steps[k++] = (1 << 24) | (P << 12);
        }
        nsteps = k;
    }
    for (int e = tid; e < q * C; e += 256) {
        const int a = e / C, cc = e % C, col = cbase + cc;
        zs[a * C + cc] = col < DC ? __ldg(Y + ((int64_t)u * r + a) * DC + col) : 0.0;
    }
    __syncthreads();
    const int ns = nsteps;
    // issue the operand copies of step k into ring stage k % kSolveNS (one commit group per step)
    auto issue = [&](int k) {
        if (k < ns) {
            const int code = steps[k], dir = code >> 24, P = (code >> 12) & 0xfff, c = (code & 0xfff) - 1;
            const int p0 = P * kPB, nb = min(kPB, q - p0), pe = p0 + nb;
            double *buf = ring + (size_t)(k % kSolveNS) * sbuf;
            if (c < 0) {  // Di (forward: row-major lower; backward: transposed)
                const double *src = Du + (int64_t)P * kPB * kPB;
#pragma unroll
                for (int kk = 0; kk < kPB * kPB / 256; ++kk) {
                    const int e = tid + 256 * kk;
                    double *dst = dir ? buf + (e % kPB) * (kPB + 1) + e / kPB : buf + (e / kPB) * (kPB + 1) + e % kPB;
                    cp_async8_zfill(dst, src + e, true, Lu);
                }
            } else if (dir == 0) {  // Lb[rr][c2] = L[p0 + rr][b0 + c2]
                const int b0 = c * kCBs, nbk = min(kCBs, p0 - b0);
#pragma unroll
                for (int kk = 0; kk < kPB * kCBs / 256; ++kk) {
                    const int e = tid + 256 * kk, rr = e / kCBs, c2 = e % kCBs;
                    if (c2 < lb - 1)
                        cp_async8_zfill(buf + rr * lb + c2, Lu + (int64_t)(p0 + rr) * r + b0 + c2, rr < nb && c2 < nbk, Lu);
                }
            } else {  // Lb[c2][bb] = L[b0 + bb][p0 + c2]  (coalesced rows of L, transposed placement)
                const int b0 = pe + c * kCBs, nbk = min(kCBs, q - b0);
#pragma unroll
                for (int kk = 0; kk < kPB * kCBs / 256; ++kk) {
                    const int e = tid + 256 * kk, bb = e / kPB, c2 = e % kPB;
                    if (bb < lb - 1)
                        cp_async8_zfill(buf + c2 * lb + bb, Lu + (int64_t)(b0 + bb) * r + p0 + c2, bb < nbk && c2 < nb, Lu);
                }
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < kSolveNS - 1; ++k) issue(k);
    const int pr = tid >> 3, pc = (tid / PARTS) % C, part = tid % PARTS;
    double acc = 0.0;  // this thread's quarter of the panel row's running right-hand side
    bool panel_start = true;
    for (int k = 0; k < ns; ++k) {
        const int code = steps[k], dir = code >> 24, P = (code >> 12) & 0xfff, c = (code & 0xfff) - 1;
        const int p0 = P * kPB, nb = min(kPB, q - p0), pe = p0 + nb;
        const double *buf = ring + (size_t)(k % kSolveNS) * sbuf;
        if (panel_start) acc = (pr < nb && part == 0) ? zs[(p0 + pr) * C + pc] : 0.0;
        cp_async_wait<kSolveNS - 2>();  // this thread's copies of step k landed
        if (c < 0) {                    // combine the four parts of the row's right-hand side
            double t = acc;
#pragma unroll
            for (int o = 1; o < PARTS; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (part == 0) tP[pr][pc] = t;
        }
        __syncthreads();  // everyone's copies (and tP) visible
        if (c < 0) {
            // Di is triangular with explicit zeros: full-length dot, split over the four parts
            double z0 = 0.0, z1 = 0.0;
#pragma unroll
            for (int j = part; j < kPB; j += 2 * PARTS) {
                z0 = fma(buf[pr * (kPB + 1) + j], tP[j][pc], z0);
                z1 = fma(buf[pr * (kPB + 1) + j + PARTS], tP[j + PARTS][pc], z1);
            }
            double z = z0 + z1;
#pragma unroll
            for (int o = 1; o < PARTS; o <<= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
            if (pr < nb && part == 0) zs[(p0 + pr) * C + pc] = z;
        } else if (pr < nb) {
            const int b0 = dir == 0 ? c * kCBs : pe + c * kCBs;
            const int nbk = dir == 0 ? min(kCBs, p0 - b0) : min(kCBs, q - b0);
            const double *lr = buf + pr * lb;
            double a0 = 0.0, a1 = 0.0;
            int bb = part;
#pragma unroll 4
            for (; bb + PARTS < nbk; bb += 2 * PARTS) {
                a0 = fma(-lr[bb], zs[(b0 + bb) * C + pc], a0);
                a1 = fma(-lr[bb + PARTS], zs[(b0 + bb + PARTS) * C + pc], a1);
            }
            if (bb < nbk) a0 = fma(-lr[bb], zs[(b0 + bb) * C + pc], a0);
            acc += a0 + a1;
        }
        __syncthreads();  // stage k % NS and tP free; z of a DIAG step visible
        issue(k + kSolveNS - 1);
        panel_start = (c < 0);
    }
    cp_async_wait<0>();
    for (int e = tid; e < r * C; e += 256) {
        const int a = e / C, cc = e % C, col = cbase + cc;
        if (col < DC) Xu[(int64_t)a * DC + col] = a < q ? (float)zs[a * C + cc] : 0.f;
    }
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
    static constexpr int kOffA = 0, kOffB = kA, kOffP = kOffB + 2 * kB, kOffV = kOffP + kP;  // B, V double-buffered
    static constexpr int kOffG = kOffV + 2 * kV, kOffKb = kOffG + 2 * 128 * 4, kOffX = kOffKb + D * 4;
    static constexpr int kOffBar = kOffX + 2 * 128 * 4, kOffTb = kOffBar + 16;
    static constexpr int kTotal = kOffTb + 8;
};

// Software pipeline over the CTA's 128-key slices: the next slice's K and V rows are loaded into
// registers while the tensor cores run GEMM1 / GEMM2 of the current one, then written (swizzled;
// V transposed) into the other B / V buffer; gamma_l = -g <k_l, kbar> comes from the same registers.
// tcgen05.commit on bar1 after GEMM1(s) also retires GEMM2(s-1), which frees P and the old buffers.
template <int D>
__global__ void __launch_bounds__(kWTc, 1)
    weights_tc_kernel(const __nv_bfloat16 *__restrict__ K, const __nv_bfloat16 *__restrict__ V,
                      const int32_t *__restrict__ S, const __nv_bfloat16 *__restrict__ KSin,
                      const int32_t *__restrict__ r_eff,
                      const double *__restrict__ stats, int64_t n_buf, int r, int splits, float *__restrict__ Ypart,
                      int bins, int64_t nb, int64_t unit_n) {
    pdl_wait();
    using L = WtSmem<D>;
    constexpr int DC = D + 1;
    constexpr int CPR = D / 8;          // 16-byte chunks per row
    constexpr int NCH = 128 * CPR / kWTc;  // chunks per thread per slice (K: same chunk column, rows tid/CPR + k*RPS;
                                           // V: row tid % 128, chunk columns tid/128 + 2k)
    constexpr int RPS = kWTc / CPR;     // rows per pass
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;  // offset 0 of the CTA's shared window (no static smem): 1024-aligned
    if (smem_u32(sm) & 1023u) __trap();
    unsigned char *sA = sm + L::kOffA, *sP = sm + L::kOffP;
    float *sG = reinterpret_cast<float *>(sm + L::kOffG);    // [2][128] log2e * gamma_l of the slice
    float *sKb = reinterpret_cast<float *>(sm + L::kOffKb);  // kbar (fp32) [D]
    float *xch = reinterpret_cast<float *>(sm + L::kOffX);   // [2][128] row-sum exchange
    uint64_t *bar1 = reinterpret_cast<uint64_t *>(sm + L::kOffBar), *bar2 = bar1 + 1;
    uint32_t &tbase = *reinterpret_cast<uint32_t *>(sm + L::kOffTb);
    const int tid = threadIdx.x, w = tid >> 5, row = tid & 127, half = tid >> 7;
    const int split = blockIdx.x, a0 = blockIdx.y * 128, u = blockIdx.z;
    const int re = r_eff[u];
    if (a0 >= re) return;  // uniform per CTA
    const SubUnit sub = sub_unit(u, n_buf, bins, nb, unit_n);  // keys of this (sub-)unit (Z13)
    const int64_t n = sub.count;
    const __nv_bfloat16 *Ku = K + sub.base * D;
    const __nv_bfloat16 *Vu = V + sub.base * D;
    const double *st = stats + (int64_t)u * (kStatsHead + D);
    const double g = st[1], mstar = st[2];

    if (w == 0) umma::tmem_alloc(&tbase, 256);
    if (tid == 0) {
        mbar_init(bar1, 1);
        mbar_init(bar2, 1);
        fence_mbar_init();
    }
    for (int j = tid; j < D; j += kWTc) sKb[j] = (float)st[kStatsHead + j];
    // coreset rows (raw keys) -> A operand (all of the thread's loads in flight)
    {
        uint4 av[NCH];
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const int e = tid + k * kWTc, rw = e / CPR, cc = e % CPR;
            av[k] = make_uint4(0, 0, 0, 0);
            if (a0 + rw < re) {
                const __nv_bfloat16 *ksrow = KSin ? KSin + ((int64_t)u * r + a0 + rw) * D
                                                  : Ku + (int64_t)S[(int64_t)u * r + a0 + rw] * D;
                av[k] = __ldg(reinterpret_cast<const uint4 *>(ksrow) + cc);
            }
        }
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const int e = tid + k * kWTc, rw = e / CPR, cc = e % CPR;
            *reinterpret_cast<uint4 *>(sA + umma::sw128_offset(rw, cc * 8, 128)) = av[k];
        }
    }
    // alpha_a = g(|kbar|^2 - <k_a, kbar>) - mstar in fp64, scaled by log2(e) for ex2: from shared
    // memory (the staged A rows and an fp64 copy of kbar), the two halves of a row on its two threads
    double *sKbd = reinterpret_cast<double *>(sP);  // sP is unused until the first exp epilogue
    for (int j = tid; j < D; j += kWTc) sKbd[j] = st[kStatsHead + j];
    __syncthreads();
    const bool row_ok = a0 + row < re;
    double kk = 0.0, bb = 0.0;
#pragma unroll 8
    for (int j = half * (D / 2); j < (half + 1) * (D / 2); ++j) {
        const double kbj = sKbd[j];
        const __nv_bfloat16 kv = *reinterpret_cast<const __nv_bfloat16 *>(sA + umma::sw128_offset(row, j, 128));
        kk = fma(to_f64(kv), kbj, kk);
        bb = fma(kbj, kbj, bb);
    }
    double *xd = reinterpret_cast<double *>(sP) + D;  // [2][128] half-row partials
    xd[half * 256 + row] = kk;
    xd[half * 256 + 128 + row] = bb;
    __syncthreads();
    float alpha2 = 0.f;
    if (row_ok) {
        const double kks = xd[row] + xd[256 + row], bbs = xd[128 + row] + xd[256 + 128 + row];
        alpha2 = (float)((g * (bbs - kks) - mstar) * 1.4426950408889634);
    }
    __syncthreads();  // sP is reused below
    const float g2 = (float)(g * 1.4426950408889634);
    const int64_t rows = ceil_div(n, splits);
    const int64_t lo = (int64_t)split * rows, hi = std::min<int64_t>(n, lo + rows);
    const int nsl = (int)ceil_div(std::max<int64_t>(0, hi - lo), 128);
    const uint32_t tS = tbase, tO = tbase + 128, lane_off = (uint32_t)((w & 3) * 32) << 16;
    const int cc_t = tid % CPR, r_t = tid / CPR;  // this thread's chunk column and first row

    uint4 kreg[NCH], vreg[NCH];
    auto prefetch = [&](int64_t l0) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const int64_t l = l0 + r_t + k * RPS;
            kreg[k] = l < hi ? __ldg(reinterpret_cast<const uint4 *>(Ku + l * D) + cc_t) : make_uint4(0, 0, 0, 0);
            // V: lane <-> key row, so that the transposed 2-byte stores below are bank-conflict free
            const int64_t lv = l0 + (tid & 127);
            const int ccv = (tid >> 7) + 2 * k;
            vreg[k] = lv < hi ? __ldg(reinterpret_cast<const uint4 *>(Vu + lv * D) + ccv) : make_uint4(0, 0, 0, 0);
        }
    };
    auto stage = [&](int buf) {
        unsigned char *sB = sm + L::kOffB + buf * L::kB, *sV = sm + L::kOffV + buf * L::kV;
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const int rw = r_t + k * RPS;
            *reinterpret_cast<uint4 *>(sB + umma::sw128_offset(rw, cc_t * 8, 128)) = kreg[k];
            const __nv_bfloat16 *pv = reinterpret_cast<const __nv_bfloat16 *>(&vreg[k]);
            const int lvr = tid & 127, ccv = (tid >> 7) + 2 * k;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                *reinterpret_cast<__nv_bfloat16 *>(sV + umma::sw128_offset(ccv * 8 + q, lvr, D)) = pv[q];
            // gamma: partial <k_l, kbar> over this chunk, reduced over the CPR lanes of the row
            const __nv_bfloat16 *pk = reinterpret_cast<const __nv_bfloat16 *>(&kreg[k]);
            float gm = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) gm = fmaf(__bfloat162float(pk[q]), sKb[cc_t * 8 + q], gm);
#pragma unroll
            for (int o = 1; o < CPR; o <<= 1) gm += __shfl_xor_sync(0xffffffffu, gm, o);
            if (cc_t == 0) sG[buf * 128 + rw] = -g2 * gm;
        }
    };

    float rowsum = 0.f;
    if (nsl > 0) {
        prefetch(lo);
        stage(0);
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    for (int s = 0; s < nsl; ++s) {
        const int buf = s & 1;
        const int64_t l0 = lo + (int64_t)s * 128;
        if (tid == 0) {
            umma::gemm_128xNxK(tS, smem_u32(sA), smem_u32(sm + L::kOffB + buf * L::kB), 128, D, false);
            umma::commit(bar1);  // also retires GEMM2(s-1)
        }
        if (s + 1 < nsl) prefetch(l0 + 128);  // global loads in flight during GEMM1 / exp
        mbar_wait(bar1, (uint32_t)(s & 1));
        umma::fence_after_sync();
        // P = exp2(g2 S + alpha2 + gamma2) for 64 columns per thread (its half), bf16 -> smem
        const int nl = (int)std::min<int64_t>(128, hi - l0);
        {
            const float *gmb = sG + buf * 128;
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
                    const float p0 = (row_ok && l < nl) ? ex2_approx_w(fmaf(g2, v[cl], alpha2 + gmb[l])) : 0.f;
                    const float p1 = (row_ok && l + 1 < nl) ? ex2_approx_w(fmaf(g2, v[cl + 1], alpha2 + gmb[l + 1])) : 0.f;
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
            umma::gemm_128xNxK(tO, smem_u32(sP), smem_u32(sm + L::kOffV + buf * L::kV), D, 128, s > 0);
            // GEMM2(s) of the earlier slices is retired by the next bar1 commit; only the last one is
            // waited on through bar2 (one phase: no mbarrier phase completes without a waiter)
            if (s + 1 == nsl) umma::commit(bar2);
        }
        if (s + 1 < nsl) {
            stage(buf ^ 1);  // B/V buffers of slice s-1: retired by the bar1 wait above
            umma::fence_async_smem();
            umma::fence_before_sync();
            __syncthreads();
            umma::fence_after_sync();
        }
    }
    if (nsl > 0) {
        mbar_wait(bar2, 0u);
        umma::fence_after_sync();
    }
    xch[half * 128 + row] = rowsum;
    __syncthreads();
    // the [128][d+1] partial tile is staged in the idle B / P / V buffers (all MMAs have retired) and
    // written as one contiguous run (its rows are consecutive rows of Ypart): coalesced stores
    float *ytile = reinterpret_cast<float *>(sm + L::kOffB);
    static_assert(128 * (D + 1) * 4 <= L::kOffG - L::kOffB, "partial tile fits the idle operand buffers");
    {
        constexpr int HD = D / 2;
        if (nsl == 0) {  // empty key range: zero partial
            for (int c = half * HD; c < half * HD + HD; ++c) ytile[row * DC + c] = 0.f;
        } else {
#pragma unroll
            for (int c0 = 0; c0 < HD; c0 += 32) {
                float v[32];
                umma::ld32(tO + lane_off + half * HD + c0, v);
#pragma unroll
                for (int i = 0; i < 32; ++i) ytile[row * DC + half * HD + c0 + i] = v[i];
            }
        }
        if (half == 0) ytile[row * DC + D] = nsl == 0 ? 0.f : xch[row] + xch[128 + row];
    }
    __syncthreads();
    {
        const int nrows = min(128, re - a0);  // rows past r_eff are not written
        float *dst = Ypart + (((int64_t)u * splits + split) * r + a0) * DC;
        for (int e = tid; e < nrows * DC; e += kWTc) dst[e] = ytile[e];
    }
    umma::fence_before_sync();
    __syncthreads();
    if (w == 0) umma::tmem_dealloc(tbase, 256);
}

// A3: fp32 split partials of Y~ (tensor-core kernel for bf16 and d in {64, 128}), then their
// fixed-order fp64 sum into Yfull.  Coreset rows come from K[S] or, if KSin != nullptr, densely.
template <typename T, int D>
int launch_partial_td(const Dims &Dm, const void *K, const void *V, const int32_t *S, const void *KSin,
                      const int32_t *r_eff, const double *stats, float *Ypart, double **Yfull_out, cudaStream_t st,
                      const double *L_dinv = nullptr, void *KSout = nullptr) {
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
            launch_pdl(kt, gt, dim3(kWTc), smem_tc, st, static_cast<const __nv_bfloat16 *>(K),
                       static_cast<const __nv_bfloat16 *>(V), S, static_cast<const __nv_bfloat16 *>(KSin), r_eff,
                       stats, Dm.n, Dm.r, splits, Ypart, Dm.bins, Dm.nb, Dm.unit_n);
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
                                   static_cast<const T *>(KSin), r_eff, stats, Dm.n, Dm.r, splits, Ypart, Dm.bins, Dm.nb,
                                   Dm.unit_n);
    }
    const size_t parts = (size_t)units * splits * Dm.r * (D + 1);
    double *Yfull = *Yfull_out ? *Yfull_out : reinterpret_cast<double *>(Ypart + ((parts + 1) & ~size_t(1)));
    const int64_t cnt = (int64_t)Dm.r * (D + 1);
    dim3 gr((unsigned)ceil_div(cnt, 256), units);
    if (L_dinv) {  // single-GPU path: the diagonal-block inverses of L ride along (Dinv follows Y~)
        const int nbl = (Dm.r + kPB - 1) / kPB;
        double *Dinv = Yfull + (size_t)units * Dm.r * (D + 1);
        // (with KSout: the K_S gather of the attend rides along, one block per coreset row)
        launch_pdl(weights_reduce_dinv_kernel<T, D>, dim3(gr.x + nbl + (KSout ? Dm.r : 0), units), dim3(256), 0, st,
                   (const float *)Ypart, r_eff, Dm.r, splits, Yfull, L_dinv, Dinv, (int)gr.x, nbl,
                   static_cast<const T *>(K), S, static_cast<T *>(KSout), Dm.n, Dm.bins, Dm.nb, Dm.unit_n);
    } else {
        launch_pdl(weights_reduce_kernel<D>, gr, dim3(256), 0, st, (const float *)Ypart, r_eff, Dm.r, splits, Yfull);
    }
    *Yfull_out = Yfull;
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

// r <= 32 (e.g. binned sub-units): the whole solve is one diagonal block, X = Dinv^T (Dinv Y); one
// CTA per unit does both 32 x 32 products for all d + 1 columns out of shared memory.
template <int D>
__global__ void __launch_bounds__(256) weights_solve_small_kernel(const double *__restrict__ Y,
                                                                  const double *__restrict__ Dinv,
                                                                  const int32_t *__restrict__ r_eff, int r,
                                                                  float *__restrict__ X) {
    pdl_wait();
    constexpr int DC = D + 1;
    __shared__ double Di[kPB][kPB + 1];
    __shared__ double Z[kPB][DC];
    const int u = blockIdx.x, tid = threadIdx.x;
    const int q = r_eff[u];
    const double *Du = Dinv + (int64_t)u * kPB * kPB;  // one block per unit (r <= 32)
    for (int e = tid; e < kPB * kPB; e += 256) Di[e / kPB][e % kPB] = q > 0 ? Du[e] : 0.0;
    for (int e = tid; e < kPB * DC; e += 256) {
        const int a = e / DC, c = e % DC;
        Z[a][c] = a < q ? Y[((int64_t)u * r + a) * DC + c] : 0.0;
    }
    __syncthreads();
    double t[(kPB * DC + 255) / 256];
#pragma unroll
    for (int k = 0; k < (kPB * DC + 255) / 256; ++k) {  // z = Dinv y (lower triangular)
        const int e = tid + 256 * k;
        double acc = 0.0;
        if (e < kPB * DC) {
            const int a = e / DC, c = e % DC;
            for (int j = 0; j <= a; ++j) acc = fma(Di[a][j], Z[j][c], acc);
        }
        t[k] = acc;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < (kPB * DC + 255) / 256; ++k) {
        const int e = tid + 256 * k;
        if (e < kPB * DC) Z[e / DC][e % DC] = t[k];
    }
    __syncthreads();
    float *Xu = X + (int64_t)u * r * DC;
    for (int e = tid; e < r * DC; e += 256) {  // x = Dinv^T z (upper triangular)
        const int a = e / DC, c = e % DC;
        double acc = 0.0;
        for (int j = a; j < kPB; ++j) acc = fma(Di[j][a], Z[j][c], acc);
        Xu[e] = a < q ? (float)acc : 0.f;
    }
}

// A4 for r <= 256 with few units: one thread per row of L, C right-hand-side columns per CTA.  Forward
// substitution L z = y right-looking over the 32-row panels P: the panel's rows finish (z_P = Dinv_PP
// acc_P), then every later row a subtracts L[a, P] z_P; the backward substitution L^T x = z likewise over
// the columns of L (row a < 32 P subtracts L[P, a]^T x_P).  Per panel two barriers and 32-term dots.  The
// panel's L block (forward: rows below it x its 32 columns; backward: its 32 rows x the columns before it)
// and its Dinv block are copied coalesced into shared memory (cp.async, double-buffered) one panel ahead --
// no copy depends on z -- so the panel chain carries shared-memory and FMA latency only
// (weights_solve_kernel streams L blocks through a cp.async ring per step instead).  Rows >= r_eff have
// zero Y~ rows and Dinv rows / columns and are never updated, so they stay 0.
constexpr int kSrLd = kPB + 2;                 // forward L / Dinv block: [row][j], row stride 34 doubles
constexpr int kSrLdB = 8 * kPB + 2;            // backward L block: [j][column a], row stride 258 doubles
constexpr int kSrLBuf = 8 * kPB * kSrLd;       // doubles per L buffer (>= kPB * kSrLdB)
constexpr int kSrDBuf = kPB * kSrLd;           // doubles per Dinv buffer
constexpr size_t kSrSmem = (size_t)2 * (kSrLBuf + kSrDBuf) * sizeof(double);
static_assert(kPB * kSrLdB <= kSrLBuf, "backward L block fits the buffer");

template <int D, int C>
__global__ void __launch_bounds__(256) weights_solve_rows_kernel(const double *__restrict__ Y,
                                                                 const double *__restrict__ L,
                                                                 const double *__restrict__ Dinv,
                                                                 const int32_t *__restrict__ r_eff, int r,
                                                                 float *__restrict__ X) {
    pdl_wait();
    constexpr int DC = D + 1, NCH = C >= 4 ? 1 : 4 / C;  // independent FMA chains per column
    extern __shared__ double srs[];                       // [2][L block], then [2][Dinv block]
    __shared__ double sacc[kPB][C];
    __shared__ double sz[8 * kPB][C];
    const int u = blockIdx.y, a = threadIdx.x, nth = blockDim.x, c0 = blockIdx.x * C;
    const int q = r_eff[u];
    const int npan = (q + kPB - 1) / kPB, nbl = (r + kPB - 1) / kPB;
    const int pa = a / kPB, ra = a % kPB;
    const double *Lu = L + (int64_t)u * r * r;
    const double *Du = Dinv + (int64_t)u * nbl * kPB * kPB;
    double acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = (a < q && c0 + c < DC) ? Y[((int64_t)u * r + a) * DC + c0 + c] : 0.0;
    // copies of panel P (buffer P & 1): the Dinv block, and the L block of the direction
    // 16-byte copies (two 8-byte ones when odd r leaves L rows 8-byte aligned only); pairs of doubles
    const bool al16 = (r & 1) == 0;
    auto cp2 = [&](double *dst, const double *src) {
        if (al16) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
        } else {
            cp_async8(dst, src);
            cp_async8(dst + 1, src + 1);
        }
    };
    auto issue = [&](int P, bool fwd) {
        double *Lb = srs + (size_t)(P & 1) * kSrLBuf;
        double *Db = srs + (size_t)2 * kSrLBuf + (size_t)(P & 1) * kSrDBuf;
        const double *Dp = Du + (int64_t)P * kPB * kPB;  // 16-byte aligned (blocks of 1024 doubles)
        for (int e = a; e < kPB * kPB / 2; e += nth) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(Db + (e >> 4) * kSrLd + 2 * (e & 15))),
                         "l"(Dp + 2 * e)
                         : "memory");
        }
        if (fwd) {  // L[a][32P + j] for rows a in [32(P+1), q): 16 pairs per row, nth / 16 rows at a time
            const int ch = a & 15;
            for (int rr = (P + 1) * kPB + (a >> 4); rr < q; rr += nth >> 4)
                cp2(Lb + rr * kSrLd + 2 * ch, Lu + (int64_t)rr * r + P * kPB + 2 * ch);
        } else if (2 * a < P * kPB) {  // L[32P + j][a] for columns a < 32P (rows 32P + j < q)
            const int nr = min(kPB, q - P * kPB);
            for (int j = 0; j < nr; ++j) cp2(Lb + j * kSrLdB + 2 * a, Lu + (int64_t)(P * kPB + j) * r + 2 * a);
        }
        cp_async_commit();
    };
    auto panel = [&](int P, bool fwd) {
        const double *Lb = srs + (size_t)(P & 1) * kSrLBuf;
        const double *Db = srs + (size_t)2 * kSrLBuf + (size_t)(P & 1) * kSrDBuf;
        cp_async_wait<0>();  // this thread's copies of panel P (the only group in flight)
        if (pa == P) {
#pragma unroll
            for (int c = 0; c < C; ++c) sacc[ra][c] = acc[c];
        }
        __syncthreads();  // panel P's blocks and sacc visible; every thread is past panel P - 1
        const int Pn = fwd ? P + 1 : P - 1;
        if (fwd ? Pn < npan : Pn >= 0) issue(Pn, fwd);  // into the buffer panel P - 1 used
        if (pa == P) {  // z_P = Dinv_PP acc_P (forward), x_P = Dinv_PP^T acc_P (backward)
            double t[C][NCH];
#pragma unroll
            for (int c = 0; c < C; ++c)
#pragma unroll
                for (int h = 0; h < NCH; ++h) t[c][h] = 0.0;
#pragma unroll
            for (int j = 0; j < kPB; j += 2) {
                double d0, d1;
                if (fwd) {  // row ra, 16-byte reads (conflict-free with the 34-double stride)
                    const double2 v = *reinterpret_cast<const double2 *>(Db + ra * kSrLd + j);
                    d0 = v.x;
                    d1 = v.y;
                } else {
                    d0 = Db[j * kSrLd + ra];
                    d1 = Db[(j + 1) * kSrLd + ra];
                }
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    t[c][j % NCH] = fma(d0, sacc[j][c], t[c][j % NCH]);
                    t[c][(j + 1) % NCH] = fma(d1, sacc[j + 1][c], t[c][(j + 1) % NCH]);
                }
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                double z = t[c][0];
#pragma unroll
                for (int h = 1; h < NCH; ++h) z += t[c][h];
                acc[c] = z;
                sz[a][c] = z;
            }
        }
        __syncthreads();
        if (a < q && (fwd ? pa > P : pa < P)) {
            double t[C][NCH];
#pragma unroll
            for (int c = 0; c < C; ++c)
#pragma unroll
                for (int h = 0; h < NCH; ++h) t[c][h] = 0.0;
            const int jn = fwd ? kPB : min(kPB, q - P * kPB);
            if (fwd) {
#pragma unroll
                for (int j = 0; j < kPB; j += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(Lb + a * kSrLd + j);
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        t[c][j % NCH] = fma(v.x, sz[P * kPB + j][c], t[c][j % NCH]);
                        t[c][(j + 1) % NCH] = fma(v.y, sz[P * kPB + j + 1][c], t[c][(j + 1) % NCH]);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < kPB; ++j) {
                    if (j < jn) {
                        const double lv = Lb[j * kSrLdB + a];
#pragma unroll
                        for (int c = 0; c < C; ++c) t[c][j % NCH] = fma(lv, sz[P * kPB + j][c], t[c][j % NCH]);
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                double z = t[c][0];
#pragma unroll
                for (int h = 1; h < NCH; ++h) z += t[c][h];
                acc[c] -= z;
            }
        }
    };
    if (npan > 0) issue(0, true);
    for (int P = 0; P < npan; ++P) panel(P, true);
    __syncthreads();  // every thread is past the forward panels (their buffers are reused)
    if (npan > 0) issue(npan - 1, false);
    for (int P = npan - 1; P >= 0; --P) panel(P, false);
    if (a < r) {
        float *Xr = X + ((int64_t)u * r + a) * DC + c0;
#pragma unroll
        for (int c = 0; c < C; ++c)
            if (c0 + c < DC) Xr[c] = a < q ? (float)acc[c] : 0.f;
    }
}

// Columns per CTA of weights_solve_rows_kernel (0: not used): r <= 256 and at most one wave of CTAs.
inline int solve_rows_cols(const Dims &Dm) {
    if (Dm.r <= kPB || Dm.r > 8 * kPB) return 0;
    static const char *force = std::getenv("WC_SOLVE_COLS");  // A/B: force C (1, 2, 4, 8)
    if (force) return std::atoi(force);
    for (int C = 1; C <= 8; C *= 2)
        if ((int64_t)Dm.units() * ceil_div(Dm.d + 1, C) <= 148) return C;
    return 0;
}

template <int D>
int launch_solve_d(const Dims &Dm, const double *Yfull, const double *L, const int32_t *r_eff, float *X,
                   double *Dinv, cudaStream_t st, bool dinv_done = false) {
    const int nbl = (Dm.r + kPB - 1) / kPB;
    if (!dinv_done) launch_pdl(weights_dinv_kernel, dim3(nbl, Dm.units()), dim3(32), 0, st, L, r_eff, Dm.r, Dinv);
    if (Dm.r <= kPB && Dm.units() >= 148) {  // many small units: both products in one CTA per unit
        launch_pdl(weights_solve_small_kernel<D>, dim3(Dm.units()), dim3(256), 0, st, Yfull, (const double *)Dinv,
                   r_eff, Dm.r, X);
        return cudaPeekAtLastError() == cudaSuccess ? (dinv_done ? 1 : 2) : -1;
    }
    static const char *rmode = std::getenv("WC_SOLVE");  // "panel": keep the streamed panel chain (A/B tests)
    const int Cr = (rmode && std::strcmp(rmode, "panel") == 0) ? 0 : solve_rows_cols(Dm);
    if (Cr > 0) {
        const dim3 grid((unsigned)ceil_div(D + 1, Cr), Dm.units()), block((unsigned)(nbl * kPB));
        const double *Dc = Dinv;
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSrSmem);
            launch_pdl(kern, grid, block, kSrSmem, st, Yfull, L, Dc, r_eff, Dm.r, X);
        };
        switch (Cr) {
            case 1: go(weights_solve_rows_kernel<D, 1>); break;
            case 2: go(weights_solve_rows_kernel<D, 2>); break;
            case 4: go(weights_solve_rows_kernel<D, 4>); break;
            default: go(weights_solve_rows_kernel<D, 8>); break;
        }
        return cudaPeekAtLastError() == cudaSuccess ? (dinv_done ? 1 : 2) : -1;
    }
    // few units: 2 columns per CTA (more CTAs on the panel chain); many units: 8 per CTA
    const bool wide = (int64_t)Dm.units() * ((D + 1 + 1) / 2) <= 4 * 148;
    const int lb = std::min(kCBs, Dm.r) + 1;
    const size_t ring = (size_t)kSolveNS * kPB * std::max(lb, kPB + 1);
    if (wide) {
        const size_t smem = ((size_t)2 * Dm.r + ring) * sizeof(double);
        auto sk = weights_solve_kernel<D, 2>;
        cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(sk, dim3((D + 1 + 1) / 2, Dm.units()), dim3(256), smem, st, Yfull, L, (const double *)Dinv, r_eff,
                   Dm.r, X);
    } else {
        const size_t smem = ((size_t)8 * Dm.r + ring) * sizeof(double);
        auto sk = weights_solve_kernel<D, 8>;
        cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(sk, dim3((D + 1 + 7) / 8, Dm.units()), dim3(256), smem, st, Yfull, L, (const double *)Dinv, r_eff,
                   Dm.r, X);
    }
    return cudaPeekAtLastError() == cudaSuccess ? (dinv_done ? 1 : 2) : -1;
}

// =====================================================================================
// A4 by an explicit inverse: W = L^{-1} by recursive doubling over the 32 x 32 diagonal-block
// inverses (Dinv), then X = W^T (W Y~) -- every step a batched fp64 GEMM on the DMMA pipe, so the
// dependent chain is log2(R / 32) + 2 GEMM launches instead of the panel-by-panel substitution.
// For lower-triangular L = [[A, 0], [B, C]]:  L^{-1} = [[A^{-1}, 0], [-C^{-1} B A^{-1}, C^{-1}]].
// R = 32 * 2^k >= r; L is read with its valid extent r_eff (zero beyond), W is R x R (zero padded),
// so W's valid block is exactly L[:q, :q]^{-1} and rows >= r_eff of X come out 0.
// =====================================================================================
constexpr int kGT = 64;   // output tile (rows and columns) of one CTA
constexpr int kGK = 32;   // K extent staged per step

inline int inv_pad(int r) {
    int R = kPB;
    while (R < r) R *= 2;
    return R;
}

// Batched GEMM  C (+)= alpha * op(A) B  on 64 x 64 output tiles (blockIdx.x: column tile, blockIdx.y:
// row tile, blockIdx.z: batch = unit * nper + j).  A(i, k) = TA ? Abuf[k * lda + i] : Abuf[i * lda + k].
// Element (i, k) of A exists only for i < a_rows, k < a_cols (zero otherwise); B(k, c) for k < b_rows,
// c < b_cols.  Pointers of batch z: base + unit * ustride + j * jstride (+ the per-mode block offsets
// folded in by the launcher through jrow / jcol multipliers below).
struct GemmArgs {
    const double *A;
    const double *B;
    void *C;
    int64_t a_ustride, a_jstride, b_ustride, b_jstride, c_ustride, c_jstride;
    int lda, ldb, ldc;
    int M, N, K;
    int nper;
    const int32_t *valid;  // r_eff per unit: A rows/cols and B rows limited to it when ka_valid / kb_valid
    int a_limit_rows, a_limit_cols, b_limit_rows;  // flags: 1 -> limit that extent by valid[unit] - offset
    int a_row0, a_col0, b_row0;                    // offsets (in the unit's matrix) of the first row / col
    int64_t a_row0_j, a_col0_j, b_row0_j;          // their per-j increments
    double alpha;
};

template <bool TA, bool OUTF32, bool ACC>
__global__ void __launch_bounds__(256) dgemm_batched_kernel(GemmArgs g) {
    pdl_wait();
    __shared__ double As[kGT][kGK + 1];  // As[i][k]
    __shared__ double Bs[kGK][kGT + 1];  // Bs[k][c]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, gid = lane >> 2, tq = lane & 3;
    const int z = blockIdx.z, u = z / g.nper, j = z % g.nper;
    const int i0 = blockIdx.y * kGT, c0 = blockIdx.x * kGT;
    if (i0 >= g.M || c0 >= g.N) return;
    const double *A = g.A + u * g.a_ustride + j * g.a_jstride;
    const double *B = g.B + u * g.b_ustride + j * g.b_jstride;
    const int q = g.valid ? g.valid[u] : INT32_MAX;
    const int64_t ar0 = g.a_row0 + j * g.a_row0_j, ac0 = g.a_col0 + j * g.a_col0_j, br0 = g.b_row0 + j * g.b_row0_j;
    const int64_t arows = g.a_limit_rows ? std::min<int64_t>(g.M, q - ar0) : g.M;
    const int64_t acols = g.a_limit_cols ? std::min<int64_t>(g.K, q - ac0) : g.K;
    const int64_t brows = g.b_limit_rows ? std::min<int64_t>(g.K, q - br0) : g.K;
    double acc[kGT / 8][2];
#pragma unroll
    for (int nt = 0; nt < kGT / 8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
    for (int k0 = 0; k0 < g.K; k0 += kGK) {
        for (int e = tid; e < kGT * kGK; e += 256) {
            int i, k;
            if (TA) { k = e / kGT; i = e % kGT; } else { i = e / kGK; k = e % kGK; }  // coalesced reads
            const int gi = i0 + i, gk = k0 + k;
            double v = 0.0;
            if (gi < arows && gk < acols) v = TA ? A[(int64_t)gk * g.lda + gi] : A[(int64_t)gi * g.lda + gk];
            As[i][k] = v;
        }
        for (int e = tid; e < kGK * kGT; e += 256) {
            const int k = e / kGT, c = e % kGT, gk = k0 + k, gc = c0 + c;
            Bs[k][c] = (gk < brows && gc < g.N) ? B[(int64_t)gk * g.ldb + gc] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGK; kk += 4) {
            const double a = As[8 * w + gid][kk + tq];
#pragma unroll
            for (int nt = 0; nt < kGT / 8; ++nt) {
                const double b = Bs[kk + tq][8 * nt + gid];
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(acc[nt][0]), "+d"(acc[nt][1])
                    : "d"(a), "d"(b));
            }
        }
        __syncthreads();
    }
    const int gi = i0 + 8 * w + gid;
    if (gi >= g.M) return;
#pragma unroll
    for (int nt = 0; nt < kGT / 8; ++nt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int gc = c0 + 8 * nt + 2 * tq + hh;
            if (gc >= g.N) continue;
            const int64_t o = u * g.c_ustride + j * g.c_jstride + (int64_t)gi * g.ldc + gc;
            if (OUTF32) {
                static_cast<float *>(g.C)[o] = (float)(g.alpha * acc[nt][hh]);
            } else {
                double *C = static_cast<double *>(g.C);
                C[o] = ACC ? C[o] + g.alpha * acc[nt][hh] : g.alpha * acc[nt][hh];
            }
        }
}

// W <- 0 with the 32 x 32 diagonal-block inverses of L on its diagonal (block b < ceil(q/32)).
__global__ void __launch_bounds__(256) winit_kernel(const double *__restrict__ Dinv, const int32_t *__restrict__ r_eff,
                                                    int r, int R, double *__restrict__ W) {
    pdl_wait();
    const int u = blockIdx.y;
    const int nbl = (r + kPB - 1) / kPB;
    double *Wu = W + (int64_t)u * R * R;
    const double *Du = Dinv + (int64_t)u * nbl * kPB * kPB;
    for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < (int64_t)R * R; e += (int64_t)gridDim.x * 256) {
        const int i = (int)(e / R), c = (int)(e % R);
        const int bi = i / kPB;
        // blocks at or past r_eff were never written by the inversion: zero
        Wu[e] = (bi == c / kPB && bi < nbl && bi * kPB < r_eff[u]) ? Du[(int64_t)bi * kPB * kPB + (i % kPB) * kPB + (c % kPB)]
                                                                   : 0.0;
    }
}

template <bool TA, bool OUTF32, bool ACC>
void launch_gemm(const GemmArgs &g, int batch, cudaStream_t st) {
    launch_pdl(dgemm_batched_kernel<TA, OUTF32, ACC>, dim3((unsigned)ceil_div(g.N, kGT), (unsigned)ceil_div(g.M, kGT),
                                                         (unsigned)batch),
               dim3(256), 0, st, g);
}

// X = W^T W Y~ with W = L^{-1}.  scratch: units * (R*R + R*R/4 + R*(d+1)) doubles.
int launch_solve_inverse(const Dims &Dm, const double *Y, const double *L, const int32_t *r_eff, float *X,
                         const double *Dinv, double *scratch, cudaStream_t st) {
    const int r = Dm.r, R = inv_pad(r), U = Dm.units(), DC = Dm.d + 1;
    double *W = scratch, *T = W + (size_t)U * R * R, *X1 = T + (size_t)U * R * R / 4;
    int launches = 0;
    launch_pdl(winit_kernel, dim3((unsigned)std::min<int64_t>(ceil_div((int64_t)R * R, 256), 64), U), dim3(256), 0, st,
               Dinv, r_eff, r, R, W);
    ++launches;
    for (int s2 = kPB; s2 < R; s2 *= 2) {
        const int np = R / (2 * s2);
        // T_j = L[(2j+1)s : (2j+2)s, 2js : 2js+s] . W[2js : 2js+s, 2js : 2js+s]
        // (batch j: L block rows [(2j+1)s, (2j+2)s), columns [2js, 2js + s), limited to r_eff)
        GemmArgs g{};
        g.A = L + (int64_t)s2 * r; g.a_ustride = (int64_t)r * r; g.a_jstride = (int64_t)(2 * s2) * r + 2 * s2;
        g.lda = r;
        g.a_row0 = s2; g.a_row0_j = 2 * s2; g.a_col0 = 0; g.a_col0_j = 2 * s2;
        g.a_limit_rows = 1; g.a_limit_cols = 1;
        g.B = W; g.b_ustride = (int64_t)R * R; g.b_jstride = (int64_t)(2 * s2) * R + 2 * s2; g.ldb = R;
        g.C = T; g.c_ustride = (int64_t)R * R / 4; g.c_jstride = (int64_t)s2 * s2; g.ldc = s2;
        g.M = s2; g.N = s2; g.K = s2; g.nper = np; g.valid = r_eff;
        g.alpha = 1.0;
        launch_gemm<false, false, false>(g, U * np, st);
        // W[(2j+1)s :, 2js :] = -W[(2j+1)s :, (2j+1)s :] . T_j
        GemmArgs h{};
        h.A = W + (int64_t)s2 * R + s2; h.a_ustride = (int64_t)R * R; h.a_jstride = (int64_t)(2 * s2) * R + 2 * s2;
        h.lda = R;
        h.B = T; h.b_ustride = (int64_t)R * R / 4; h.b_jstride = (int64_t)s2 * s2; h.ldb = s2;
        h.C = W + (int64_t)s2 * R; h.c_ustride = (int64_t)R * R; h.c_jstride = (int64_t)(2 * s2) * R + 2 * s2; h.ldc = R;
        h.M = s2; h.N = s2; h.K = s2; h.nper = np; h.valid = nullptr;
        h.alpha = -1.0;
        launch_gemm<false, false, false>(h, U * np, st);
        launches += 2;
    }
    // X1 = W Y~ (R x DC), then X = W^T X1 (rows >= r_eff of W are zero: X rows >= r_eff come out 0)
    GemmArgs g1{};
    g1.A = W; g1.a_ustride = (int64_t)R * R; g1.lda = R;
    g1.B = Y; g1.b_ustride = (int64_t)r * DC; g1.ldb = DC;
    g1.C = X1; g1.c_ustride = (int64_t)R * DC; g1.ldc = DC;
    g1.M = r; g1.N = DC; g1.K = r; g1.nper = 1; g1.alpha = 1.0;
    launch_gemm<false, false, false>(g1, U, st);
    GemmArgs g2{};
    g2.A = W; g2.a_ustride = (int64_t)R * R; g2.lda = R;
    g2.B = X1; g2.b_ustride = (int64_t)R * DC; g2.ldb = DC;
    g2.C = X; g2.c_ustride = (int64_t)r * DC; g2.ldc = DC;
    g2.M = r; g2.N = DC; g2.K = r; g2.nper = 1; g2.alpha = 1.0;
    launch_gemm<true, true, false>(g2, U, st);
    launches += 2;
    return cudaPeekAtLastError() == cudaSuccess ? launches : -1;
}

template <typename T, int D>
int launch_weights_td(const Dims &Dm, const void *K, const void *V, const int32_t *S, const int32_t *r_eff,
                      const double *L, const double *stats, float *Ypart, void *KS, float *X, cudaStream_t st) {
    double *Yfull = nullptr;
    // (the reduction launch also inverts L's diagonal blocks and gathers K_S for the attend)
    const int k1 = launch_partial_td<T, D>(Dm, K, V, S, nullptr, r_eff, stats, Ypart, &Yfull, st, L, KS);
    if (k1 < 0) return -1;
    // scratch for the diagonal-block inverses: after Y~ in the weights workspace (carve_weights),
    // then W = L^{-1}, the level products and W Y~ (solve_scratch_elems)
    double *Dinv = Yfull + (size_t)Dm.units() * Dm.r * (D + 1);
    // the explicit inverse wins for large r (LLM r = 1024: weights 2.58 -> 2.04 ms); for r <= 256 the
    // panel chain is shorter than its log2(R/32) + 2 GEMM launches (headline: 0.093 vs 0.235 ms)
    static const char *mode = std::getenv("WC_SOLVE");  // "panel" / "inverse": force one (A/B tests)
    const bool panel = mode ? std::strcmp(mode, "panel") == 0 : Dm.r < 512;
    const int k2 = panel ? launch_solve_d<D>(Dm, Yfull, L, r_eff, X, Dinv, st, true)
                         : launch_solve_inverse(Dm, Yfull, L, r_eff, X, Dinv, Dinv + (size_t)Dm.units() * dinv_elems(Dm.r), st);
    if (k2 < 0) return -1;
    return cudaPeekAtLastError() == cudaSuccess ? k1 + k2 : -1;
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
                         double *Dinv, cudaStream_t st) {
    switch (D.d) {
        case 16: return launch_solve_d<16>(D, Yfull, L, r_eff, X, Dinv, st);
        case 32: return launch_solve_d<32>(D, Yfull, L, r_eff, X, Dinv, st);
        case 64: return launch_solve_d<64>(D, Yfull, L, r_eff, X, Dinv, st);
        case 128: return launch_solve_d<128>(D, Yfull, L, r_eff, X, Dinv, st);
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
