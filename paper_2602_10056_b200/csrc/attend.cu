// attend.cu -- A5 of the hot path: weighted coreset attention, Alg 3 WtdAttn.
//   S = beta Q K_S^T (K_S uncentred);  P = exp(S - rowmax)
//   num = P X[:, :d],  den = P X[:, d]       (X = [V_S, w])
//   O = clip(num/den where den > 0 else 0, vmin, vmax)        (Z14, Z15)
// CUDA-core fp32 version: 64-query tiles, 32-row coreset tiles staged in shared memory,
// online max rescaling across coreset tiles (exact: the shift cancels in num/den).
#include <algorithm>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

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

// =====================================================================================
// tcgen05 path (bf16, d in {64, 128}, r <= 256).  One CTA of 128 threads per SM loops over
// 128-query tiles.  Per tile:
//   GEMM1 (tensor core)  S[128 x RP] = Q_tile . K_S^T          (fp32 in TMEM columns [0, RP))
//   softmax epilogue      P = exp(beta (S - rowmax)), den = P . w (fp32, CUDA cores), P -> bf16 smem
//   GEMM2 (tensor core)  O[128 x d]  = P . X_hi + P . X_lo       (fp32 in TMEM columns [256, 256+d))
//   output epilogue       O / den (den > 0, else 0), clip to [vmin, vmax], bf16 store
// X = [V_S, w] is split into bf16 hi + lo parts so the values keep ~16 bits.  Thread t owns
// TMEM lane t = query row t.  Operands are K-major, 128-byte swizzled (see umma.cuh).
// =====================================================================================
constexpr int kTcThreads = 256;  // 8 warps: warps w and w+4 share TMEM lane quadrant w%4 (column halves)

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ unsigned long long gtimer_a() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int D, int RP> struct TcSmem {
    // K-major SW128 rows are at least 128 bytes (64 bf16) wide
    static constexpr int kRK = RP < 64 ? 64 : RP;   // padded K extent of the [*, RP] operands
    static constexpr int kQ = 128 * D * 2;          // Q tile
    static constexpr int kK = RP * D * 2;           // K_S
    static constexpr int kX = D * kRK * 2;          // one of X_hi / X_lo (B operand [d][RP])
    static constexpr int kP = 128 * kRK * 2;        // P (A operand [128][RP])
    // Layout choice: keep K_S resident across tiles (P in its own region).  X is split into bf16
    // hi + lo parts when that still fits; otherwise (d = 128, r = 256) X_hi alone, so that nothing
    // has to be re-staged per tile.
    static constexpr int kBudget = 224 * 1024;
    static constexpr bool kSplitX = kQ + kK + 2 * kX + kP <= kBudget;
    static constexpr bool kAliasP = false;
    static constexpr int kOffQ = 0, kOffK = kQ, kOffXh = kQ + kK, kOffXl = kOffXh + (kSplitX ? kX : 0);
    static constexpr int kOffP = kOffXl + kX;
    static constexpr int kBytes = kOffP + kP;
    // + w (fp32), vmin/vmax (bf16), row exchange (2 x 128 fp32), mbarrier, TMEM base; no static smem,
    // so the dynamic segment starts at shared offset 0 (1024-aligned, checked at run time)
    static constexpr int kOffW = kBytes, kOffV = kOffW + RP * 4, kOffXch = kOffV + 2 * D * 2;
    static constexpr int kOffBar = kOffXch + 2 * 128 * 4, kOffTb = kOffBar + 8, kOffBarI = kOffTb + 8;
    static constexpr int kTotal = kOffBarI + 8;
    // per-unit staging image in global memory (attend_img_prep_kernel): [K_S | X_hi^T | X_lo^T] in
    // the shared-memory layout from kOffK on (one bulk copy), then w (fp32)
    static constexpr int kImgKX = kOffP - kOffK;
    static constexpr int kImgStride = (kImgKX + RP * 4 + 1023) & ~1023;
};

// Per unit: the swizzled K_S / X_hi^T / X_lo^T operand image and w, built once for all CTAs (each
// CTA then stages a unit with one bulk copy instead of re-converting X from fp32).
template <int D, int RP>
__global__ void __launch_bounds__(256) attend_img_prep_kernel(const __nv_bfloat16 *__restrict__ KS,
                                                              const float *__restrict__ X,
                                                              const int32_t *__restrict__ r_eff, int r,
                                                              unsigned char *__restrict__ img) {
    pdl_wait();
    using L = TcSmem<D, RP>;
    constexpr int DC = D + 1, CPR = D / 8;
    const int u = blockIdx.y, re = r_eff[u];
    unsigned char *dst = img + (int64_t)u * L::kImgStride;
    const int nth = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + threadIdx.x;
    for (int e = t0; e < RP * CPR; e += nth) {
        const int row = e / CPR, cc = e % CPR;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row < re) v = __ldg(reinterpret_cast<const uint4 *>(KS + ((int64_t)u * r + row) * D) + cc);
        *reinterpret_cast<uint4 *>(dst + umma::sw128_offset(row, cc * 8, RP)) = v;
    }
    // X read row-major (coalesced), written transposed into the swizzled images; column D is w
    float *wd = reinterpret_cast<float *>(dst + L::kImgKX);
    const float *Xu = X + (int64_t)u * r * DC;
    for (int e = t0; e < RP * DC; e += nth) {
        const int s2 = e / DC, c = e % DC;
        const float x = (s2 < re) ? __ldg(Xu + e) : 0.f;
        if (c == D) {
            wd[s2] = x;
            continue;
        }
        const __nv_bfloat16 xh = __float2bfloat16_rn(x);
        *reinterpret_cast<__nv_bfloat16 *>(dst + (L::kOffXh - L::kOffK) + umma::sw128_offset(c, s2, D)) = xh;
        if (L::kSplitX)
            *reinterpret_cast<__nv_bfloat16 *>(dst + (L::kOffXl - L::kOffK) + umma::sw128_offset(c, s2, D)) =
                __float2bfloat16_rn(x - __bfloat162float(xh));
    }
}

// NT threads: NT / 128 threads per query row (TMEM lane), each owning 1 / (NT / 128) of the S and O
// columns; NT = 512 for d = 128, r > 64 (shorter softmax / epilogue per thread), else 256.
template <int D, int RP, int NT>
__global__ void __launch_bounds__(NT, 1)
    attend_tc_kernel(const __nv_bfloat16 *__restrict__ Q, const __nv_bfloat16 *__restrict__ KS,
                     const float *__restrict__ X, const int32_t *__restrict__ r_eff,
                     const __nv_bfloat16 *__restrict__ vmin, const __nv_bfloat16 *__restrict__ vmax, int64_t m,
                     int r, int group, int hq, int hkv, float beta, int clip, __nv_bfloat16 *__restrict__ O,
                     int64_t tiles_per_head, int64_t total_tiles, const unsigned char *__restrict__ img,
                     unsigned long long *atrace) {
    pdl_wait();
    using L = TcSmem<D, RP>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;  // offset 0 of the CTA's shared window: 1024-aligned
    if (smem_u32(sm) & 1023u) __trap();
    unsigned char *sQ = sm + L::kOffQ, *sK = sm + L::kOffK, *sXh = sm + L::kOffXh, *sXl = sm + L::kOffXl;
    unsigned char *sP = sm + L::kOffP;
    float *sW = reinterpret_cast<float *>(sm + L::kOffW);
    __nv_bfloat16 *sVmin = reinterpret_cast<__nv_bfloat16 *>(sm + L::kOffV), *sVmax = sVmin + D;
    // row exchange between the NSPLIT column parts; aliases the Q tile, which is idle from the
    // retirement of GEMM1 until the next tile's Q is stored (after a barrier)
    float (*xch)[128] = reinterpret_cast<float (*)[128]>(sQ);
    uint64_t &bar = *reinterpret_cast<uint64_t *>(sm + L::kOffBar);
    uint64_t &ibar = *reinterpret_cast<uint64_t *>(sm + L::kOffBarI);
    uint32_t &tbase = *reinterpret_cast<uint32_t *>(sm + L::kOffTb);
    const int tid = threadIdx.x, w = tid >> 5;
    constexpr int NSPLIT = NT / 128;
    const int row = tid & 127, half = tid >> 7;  // TMEM lane (query row) and column part
    constexpr int DC = D + 1;
    uint32_t iphase = 0;

    if (w == 0) umma::tmem_alloc(&tbase, 512);
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_init(&ibar, 1);
        fence_mbar_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tS = tbase, tO = tbase + 256;
    const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
    uint32_t phase = 0;
    int cur_unit = -1, re = 0;
    const float bl2 = beta * 1.4426950408889634f;

    // contiguous tile ranges per CTA: consecutive tiles share the unit, so K_S / X are staged rarely.
    // Pipeline per tile t (one TMEM S accumulator, one O accumulator, one mbarrier, commits waited
    // in issue order): GEMM1(t) -> softmax(t) -> GEMM2(t) [Q(t+1) loads in flight] -> Q(t+1) into
    // sQ (free since GEMM1(t) retired) -> GEMM1(t+1) issued -> epilogue(t) from O while GEMM1(t+1)
    // runs (S and O are disjoint TMEM columns; sP is next written by softmax(t+1), after GEMM2(t)).
    const int64_t tpc = ceil_div(total_tiles, (int64_t)gridDim.x);
    const int64_t t_begin = (int64_t)blockIdx.x * tpc, t_end = std::min<int64_t>(total_tiles, t_begin + tpc);
    constexpr int CPR = D / 8;                   // 16-byte chunks per row
    constexpr int NQ = 128 * CPR / NT;           // Q chunks per thread
    auto unit_of = [&](int64_t tile) {
        const int64_t head = tile / tiles_per_head;
        return (int)(head / hq) * hkv + (int)(head % hq) / group;
    };
    auto load_q = [&](int64_t tile, uint4 (&qv)[NQ]) {
        const int64_t head = tile / tiles_per_head, q0 = (tile % tiles_per_head) * 128;
        const __nv_bfloat16 *Qh = Q + head * m * D;
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            const int e = tid + k * NT, row = e / CPR, cc = e % CPR;
            qv[k] = (q0 + row < m) ? __ldg(reinterpret_cast<const uint4 *>(Qh + (q0 + row) * D) + cc)
                                   : make_uint4(0, 0, 0, 0);
        }
    };
    auto store_q = [&](const uint4 (&qv)[NQ]) {
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            const int e = tid + k * NT, row = e / CPR, cc = e % CPR;
            *reinterpret_cast<uint4 *>(sQ + umma::sw128_offset(row, cc * 8, 128)) = qv[k];
        }
    };
    // K_S, X (hi / lo) of unit u: one bulk copy of its prepared image; w and the value range
    auto stage_unit = [&](int u) {
        re = r_eff[u];
        const unsigned char *iu = img + (int64_t)u * L::kImgStride;
        if (tid == 0) {
            mbar_arrive_expect_tx(&ibar, (uint32_t)L::kImgKX);
            bulk_g2s(sK, iu, (uint32_t)L::kImgKX, &ibar);
        }
        const float *wu = reinterpret_cast<const float *>(iu + L::kImgKX);
        for (int s2 = tid; s2 < RP; s2 += NT) sW[s2] = __ldg(wu + s2);
        for (int c = tid; c < D; c += NT) {
            sVmin[c] = vmin[(int64_t)u * D + c];
            sVmax[c] = vmax[(int64_t)u * D + c];
        }
        mbar_wait(&ibar, iphase);
        iphase ^= 1u;
        cur_unit = u;
    };
    auto sync_for_mma = [&]() {
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        umma::fence_after_sync();
    };
    auto issue_gemm1 = [&]() {
        if (tid == 0) {
            umma::gemm_128xNxK(tS, smem_u32(sQ), smem_u32(sK), RP, D, false);
            umma::commit(&bar);
        }
    };
    if (t_begin < t_end) {
        uint4 qv[NQ];
        load_q(t_begin, qv);
        store_q(qv);
        stage_unit(unit_of(t_begin));
        sync_for_mma();
        issue_gemm1();
    }
    for (int64_t tile = t_begin; tile < t_end; ++tile) {
        if (atrace && blockIdx.x == 0 && threadIdx.x == 0 && tile - t_begin < 64)
            atrace[(tile - t_begin) * 8] = atrace[(tile - t_begin) * 8 + 1] = gtimer_a();
        const int64_t head = tile / tiles_per_head;  // b * hq + h
        const int64_t q0 = (tile % tiles_per_head) * 128;
        // ---- S = Q K_S^T (issued at the end of the previous tile, or above)
        mbar_wait(&bar, phase);
        phase ^= 1u;
        umma::fence_after_sync();
        if (atrace && blockIdx.x == 0 && threadIdx.x == 0 && tile - t_begin < 64) atrace[(tile - t_begin) * 8 + 2] = gtimer_a();
        // ---- softmax epilogue (two threads per row, RP/2 columns each, all in registers):
        // row max, P = exp2(beta log2e (S - max)) in bf16 -> smem, den = P . w (4 partial sums)
        {
            constexpr int HC = RP / NSPLIT;  // columns per thread
            constexpr int NCH = HC / 32 > 0 ? HC / 32 : 1;
            const int cbase = half * HC;
            float v[HC >= 32 ? HC : 32];
#pragma unroll
            for (int q = 0; q < NCH; ++q) umma::ld32(tS + lane_off + cbase + q * 32, v + q * 32);
            float mx = -INFINITY;
#pragma unroll
            for (int i2 = 0; i2 < HC; ++i2)
                if (cbase + i2 < re) mx = fmaxf(mx, v[i2]);
            xch[half][row] = mx;
            __syncthreads();
#pragma unroll
            for (int q2 = 0; q2 < NSPLIT; ++q2) mx = fmaxf(mx, xch[q2][row]);
            const float mb = mx * bl2;
            float dn[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int g8 = 0; g8 < HC / 8; ++g8) {
                uint32_t pk[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int cl = g8 * 8 + 2 * i, s0 = cbase + cl;
                    const float p0 = (s0 < re) ? ex2_approx(fmaf(v[cl], bl2, -mb)) : 0.f;
                    const float p1 = (s0 + 1 < re) ? ex2_approx(fmaf(v[cl + 1], bl2, -mb)) : 0.f;
                    const __nv_bfloat162 pb = __floats2bfloat162_rn(p0, p1);
                    dn[i] = fmaf(__bfloat162float(pb.x), sW[s0], dn[i]);
                    dn[i] = fmaf(__bfloat162float(pb.y), sW[s0 + 1], dn[i]);
                    pk[i] = *reinterpret_cast<const uint32_t *>(&pb);
                }
                *reinterpret_cast<uint4 *>(sP + umma::sw128_offset(row, cbase + g8 * 8, 128)) =
                    make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
            const float dpart = (dn[0] + dn[1]) + (dn[2] + dn[3]);
            __syncthreads();  // xch reused
            xch[half][row] = dpart;
        }
        sync_for_mma();
        if (atrace && blockIdx.x == 0 && threadIdx.x == 0 && tile - t_begin < 64) atrace[(tile - t_begin) * 8 + 3] = gtimer_a();
        float den = 0.f;
#pragma unroll
        for (int q2 = 0; q2 < NSPLIT; ++q2) den += xch[q2][row];
        // ---- O = P X_hi (+ P X_lo); the next tile's Q loads fly meanwhile
        if (tid == 0) {
            umma::gemm_128xNxK(tO, smem_u32(sP), smem_u32(sXh), D, RP, false);
            if (L::kSplitX) umma::gemm_128xNxK(tO, smem_u32(sP), smem_u32(sXl), D, RP, true);
            umma::commit(&bar);
        }
        const bool has_next = tile + 1 < t_end;
        const bool same_unit = has_next && unit_of(tile + 1) == cur_unit;
        uint4 qv[NQ];
        if (has_next) load_q(tile + 1, qv);
        mbar_wait(&bar, phase);
        phase ^= 1u;
        umma::fence_after_sync();
        if (atrace && blockIdx.x == 0 && threadIdx.x == 0 && tile - t_begin < 64) atrace[(tile - t_begin) * 8 + 4] = gtimer_a();
        if (same_unit) {  // S(t+1) overlaps this tile's output epilogue
            __syncthreads();  // every thread has read den from xch (the Q tile) before it is refilled
            store_q(qv);
            sync_for_mma();
            issue_gemm1();
        }
        // ---- output epilogue: each thread finishes D/NSPLIT columns of its row.  When the bf16 tile
        // fits the (idle) P buffer it is assembled there (16-byte chunks XOR-swizzled by row, so
        // both the row writes and the chunk reads are bank-conflict free) and, its rows being
        // consecutive rows of O, leaves as one contiguous run of 16-byte stores.
        {
            constexpr bool kStaged = 128 * D * 2 <= L::kP;
            constexpr int RB = D * 2;  // output row bytes
            const int64_t qi = q0 + row;
            const float inv = den > 0.f ? 1.f / den : 0.f;
            constexpr int HD = D / NSPLIT;
#pragma unroll
            for (int c0 = 0; c0 < HD; c0 += 32) {
                const int cc0 = half * HD + c0;
                float v[32];
                umma::ld32(tO + lane_off + cc0, v);
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float o0 = v[2 * i] * inv, o1 = v[2 * i + 1] * inv;
                    if (clip) {
                        o0 = fminf(fmaxf(o0, __bfloat162float(sVmin[cc0 + 2 * i])), __bfloat162float(sVmax[cc0 + 2 * i]));
                        o1 = fminf(fmaxf(o1, __bfloat162float(sVmin[cc0 + 2 * i + 1])), __bfloat162float(sVmax[cc0 + 2 * i + 1]));
                    }
                    const __nv_bfloat162 ob = __floats2bfloat162_rn(o0, o1);
                    pk[i] = *reinterpret_cast<const uint32_t *>(&ob);
                }
                if constexpr (kStaged) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int ch = cc0 / 8 + i;  // 16-byte chunk of the row
                        *reinterpret_cast<uint4 *>(sP + row * RB + ((ch ^ (row & 7)) * 16)) =
                            make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
                    }
                } else if (qi < m) {
                    uint4 *dst = reinterpret_cast<uint4 *>(O + (head * m + qi) * D + cc0);
#pragma unroll
                    for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
                }
            }
            if constexpr (kStaged) {
                __syncthreads();
                constexpr int CPRO = RB / 16;  // 16-byte chunks per output row (>= 8)
                const int nrows = (int)std::min<int64_t>(128, m - q0);
                uint4 *dst = reinterpret_cast<uint4 *>(O + (head * m + q0) * D);
                for (int e = tid; e < nrows * CPRO; e += NT) {
                    const int rr = e / CPRO, ch = e % CPRO;
                    dst[e] = *reinterpret_cast<const uint4 *>(sP + rr * RB + ((ch ^ (rr & 7)) * 16));
                }
            }
        }
        if (has_next && !same_unit) {  // new unit: restage K_S / X, then S(t+1)
            store_q(qv);
            stage_unit(unit_of(tile + 1));
            sync_for_mma();
            issue_gemm1();
        }
        if (atrace && blockIdx.x == 0 && threadIdx.x == 0 && tile - t_begin < 64) atrace[(tile - t_begin) * 8 + 5] = gtimer_a();
    }
    if (w == 0) umma::tmem_dealloc(tbase, 512);
}

template <int D, int RP>
int launch_attend_tc(const Dims &Dm, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                     const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws, cudaStream_t st) {
    using L = TcSmem<D, RP>;
    if (!ws) return -1;
    unsigned char *img = static_cast<unsigned char *>(ws);
    launch_pdl(attend_img_prep_kernel<D, RP>, dim3(RP / 4, (unsigned)Dm.units()), dim3(256), 0, st,
               static_cast<const __nv_bfloat16 *>(KS), X, r_eff, Dm.r, img);
    constexpr int NT = (D == 128 && RP >= 128) ? 512 : kTcThreads;
    auto kern = attend_tc_kernel<D, RP, NT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    const int64_t tph = ceil_div(Dm.m, 128);
    const int64_t total = tph * Dm.hq * Dm.batch;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>(total, sms);
    static const bool tracing = std::getenv("WC_ATTEND_TRACE") != nullptr;
    unsigned long long *atrace = nullptr;
    if (tracing) {
        cudaMalloc(&atrace, 64 * 8 * sizeof(unsigned long long));
        cudaMemsetAsync(atrace, 0, 64 * 8 * sizeof(unsigned long long), st);
    }
    launch_pdl(kern, dim3(grid), dim3(NT), (size_t)L::kTotal, st, static_cast<const __nv_bfloat16 *>(Q),
               static_cast<const __nv_bfloat16 *>(KS), X, r_eff, static_cast<const __nv_bfloat16 *>(vmin),
               static_cast<const __nv_bfloat16 *>(vmax), Dm.m, Dm.r, Dm.group(), Dm.hq, Dm.hkv, (float)beta, clip,
               static_cast<__nv_bfloat16 *>(O), tph, total, (const unsigned char *)img, atrace);
    if (atrace) {  // debug: phase durations of CTA 0's tiles (ns)
        unsigned long long h[64 * 8];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, atrace, sizeof(h), cudaMemcpyDeviceToHost);
        cudaFree(atrace);
        double acc[5] = {0};
        int cnt = 0;
        for (int t = 1; t < 64; ++t) {
            if (!h[t * 8 + 5]) continue;
            for (int k = 0; k < 5; ++k) acc[k] += (double)(h[t * 8 + k + 1] - h[t * 8 + k]);
            ++cnt;
        }
        if (cnt)
            std::fprintf(stderr, "[atrace] tiles=%d stage=%.0f gemm1=%.0f softmax=%.0f gemm2=%.0f epi=%.0f ns\n", cnt,
                         acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

// =====================================================================================
// tcgen05 path for r > 256 (bf16, d in {64, 128}): the coreset is streamed through shared memory
// in chunks of RC = 128 rows, with the online (lazy) max rescaling of A5 (exact,
// since the shift cancels in num/den).  A prep kernel writes, per (unit, chunk), one contiguous
// "image" = [K_S chunk (K-major SW128) | X_hi^T chunk | X_lo^T chunk (if it fits) | w chunk fp32],
// already in the swizzled shared-memory layout, so each chunk is ONE cp.async.bulk copy into a
// double-buffered ring (issued as soon as the buffer's GEMM2 retires, so the next chunk lands
// while the current one is computed).
// Rescaling is lazy: the running max m only moves when a chunk's max exceeds it by more than
// 2^8 (log2 domain), so P <= 2^8 and O / den stay exact ratios; when it moves, the warp rescales
// its rows' O columns in TMEM (tcgen05.ld, multiply, tcgen05.st) and its running den.
// =====================================================================================
template <int D> struct TcLong {
    static constexpr int RC = 128;
    static constexpr int kQ = 128 * D * 2, kK = RC * D * 2, kX = D * RC * 2, kP = 128 * RC * 2;
    static constexpr bool kSplitX = kQ + kP + 2 * (kK + 2 * kX + RC * 4 + 1024) <= 224 * 1024;
    static constexpr int kImgK = 0, kImgXh = kK, kImgXl = kK + kX, kImgW = kK + (kSplitX ? 2 : 1) * kX;
    static constexpr int kImg = kImgW + RC * 4;  // bytes per chunk image (multiple of 16)
    static constexpr int kBuf = (kImg + 1023) & ~1023;
    static constexpr int kOffQ = 0, kOffP = kQ, kOffB0 = kQ + kP;
    static constexpr int kOffV = kOffB0 + 2 * kBuf, kOffXch = kOffV + 2 * D * 2, kOffBar = kOffXch + 2 * 128 * 4;
    static constexpr int kOffTb = kOffBar + 3 * 8, kTotal = kOffTb + 8;
};

// Per (unit, chunk, part): blockIdx.z = part of kPrepParts splits the chunk's K rows and X columns, so
// a one-unit call still spreads the image build over many SMs.
constexpr int kPrepParts = 16;
template <int D>
__global__ void __launch_bounds__(256)
    attend_long_prep_kernel(const __nv_bfloat16 *__restrict__ KS, const float *__restrict__ X,
                            const int32_t *__restrict__ r_eff, int r, int nch, unsigned char *__restrict__ img) {
    pdl_wait();
    using L = TcLong<D>;
    constexpr int RC = L::RC, DC = D + 1, CPR = D / 8;
    const int ch = blockIdx.x, u = blockIdx.y, part = blockIdx.z, tid = threadIdx.x;
    const int re = r_eff[u], s0 = ch * RC;
    unsigned char *dst = img + ((int64_t)u * nch + ch) * L::kImg;
    constexpr int KR = RC / kPrepParts;  // K rows of this part
    for (int e = tid; e < KR * CPR; e += blockDim.x) {
        const int row = part * KR + e / CPR, cc = e % CPR;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (s0 + row < re) v = __ldg(reinterpret_cast<const uint4 *>(KS + ((int64_t)u * r + s0 + row) * D) + cc);
        *reinterpret_cast<uint4 *>(dst + L::kImgK + umma::sw128_offset(row, cc * 8, RC)) = v;
    }
    // X rows of this part read row-major (coalesced over the d + 1 columns), written transposed
    for (int e = tid; e < KR * DC; e += blockDim.x) {
        const int sl = part * KR + e / DC, c = e % DC;
        const float x = (s0 + sl < re) ? __ldg(X + ((int64_t)u * r + s0 + sl) * DC + c) : 0.f;
        if (c == D) {
            reinterpret_cast<float *>(dst + L::kImgW)[sl] = x;
            continue;
        }
        const __nv_bfloat16 xh = __float2bfloat16_rn(x);
        *reinterpret_cast<__nv_bfloat16 *>(dst + L::kImgXh + umma::sw128_offset(c, sl, D)) = xh;
        if (L::kSplitX)
            *reinterpret_cast<__nv_bfloat16 *>(dst + L::kImgXl + umma::sw128_offset(c, sl, D)) =
                __float2bfloat16_rn(x - __bfloat162float(xh));
    }
}

template <int D>
__global__ void __launch_bounds__(kTcThreads, 1)
    attend_tc_long_kernel(const __nv_bfloat16 *__restrict__ Q, const unsigned char *__restrict__ img,
                          const int32_t *__restrict__ r_eff, const __nv_bfloat16 *__restrict__ vmin,
                          const __nv_bfloat16 *__restrict__ vmax, int64_t m, int nch_max, int group, int hq, int hkv,
                          float beta, int clip, __nv_bfloat16 *__restrict__ O, int64_t tiles_per_head,
                          int64_t total_tiles) {
    using L = TcLong<D>;
    constexpr int RC = L::RC;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;
    if (smem_u32(sm) & 1023u) __trap();
    unsigned char *sQ = sm + L::kOffQ, *sP = sm + L::kOffP;
    __nv_bfloat16 *sVmin = reinterpret_cast<__nv_bfloat16 *>(sm + L::kOffV), *sVmax = sVmin + D;
    float (*xch)[128] = reinterpret_cast<float (*)[128]>(sm + L::kOffXch);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + L::kOffBar);  // [0] MMA done, [1 + b] buffer b full
    uint32_t &tbase = *reinterpret_cast<uint32_t *>(sm + L::kOffTb);
    const int tid = threadIdx.x, w = tid >> 5;
    const int row = tid & 127, half = tid >> 7;

    if (w == 0) umma::tmem_alloc(&tbase, 256);
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_mbar_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tS = tbase, tO = tbase + RC;
    const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
    const float bl2 = beta * 1.4426950408889634f;

    const int64_t tpc = ceil_div(total_tiles, (int64_t)gridDim.x);
    const int64_t t_begin = (int64_t)blockIdx.x * tpc, t_end = std::min<int64_t>(total_tiles, t_begin + tpc);
    auto unit_of = [&](int64_t tile) {
        const int64_t head = tile / tiles_per_head;
        return (int)(head / hq) * hkv + (int)(head % hq) / group;
    };
    // producer state (thread 0): the chunk stream is (tile, ch < nch(unit(tile))) in order
    int64_t p_tile = t_begin;
    int p_ch = 0, p_n = 0;
    uint32_t issued = 0;
    if (tid == 0 && p_tile < t_end) p_n = (int)ceil_div(r_eff[unit_of(p_tile)], RC);
    auto issue = [&]() {
        while (p_tile < t_end && p_ch >= p_n) {
            ++p_tile;
            p_ch = 0;
            if (p_tile < t_end) p_n = (int)ceil_div(r_eff[unit_of(p_tile)], RC);
        }
        if (p_tile >= t_end) return;
        const int b = issued & 1;
        mbar_arrive_expect_tx(&bars[1 + b], L::kImg);
        bulk_g2s(sm + L::kOffB0 + b * L::kBuf, img + ((int64_t)unit_of(p_tile) * nch_max + p_ch) * L::kImg, L::kImg,
                 &bars[1 + b]);
        ++issued;
        ++p_ch;
    };
    if (tid == 0) {
        issue();
        issue();
    }
    uint32_t j = 0, mph = 0;
    int cur_unit = -1;
    for (int64_t tile = t_begin; tile < t_end; ++tile) {
        const int64_t head = tile / tiles_per_head;
        const int64_t q0 = (tile % tiles_per_head) * 128;
        const int u = unit_of(tile);
        const int re = r_eff[u];
        const int nch = (int)ceil_div(re, RC);
        const __nv_bfloat16 *Qh = Q + head * m * D;
        constexpr int CPR = D / 8;
        for (int e = tid; e < 128 * CPR; e += kTcThreads) {
            const int rw = e / CPR, cc = e % CPR;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (q0 + rw < m) v = __ldg(reinterpret_cast<const uint4 *>(Qh + (q0 + rw) * D) + cc);
            *reinterpret_cast<uint4 *>(sQ + umma::sw128_offset(rw, cc * 8, 128)) = v;
        }
        if (u != cur_unit) {
            for (int c = tid; c < D; c += kTcThreads) {
                sVmin[c] = vmin[(int64_t)u * D + c];
                sVmax[c] = vmax[(int64_t)u * D + c];
            }
            cur_unit = u;
        }
        float mrun = -INFINITY, dn = 0.f;
        for (int ch = 0; ch < nch; ++ch, ++j) {
            const int b = j & 1;
            const unsigned char *sB = sm + L::kOffB0 + b * L::kBuf;
            umma::fence_async_smem();
            umma::fence_before_sync();
            __syncthreads();
            umma::fence_after_sync();
            mbar_wait(&bars[1 + b], (j >> 1) & 1u);
            if (tid == 0) {
                umma::gemm_128xNxK(tS, smem_u32(sQ), smem_u32(sB + L::kImgK), RC, D, false);
                umma::commit(&bars[0]);
            }
            mbar_wait(&bars[0], mph);
            mph ^= 1u;
            umma::fence_after_sync();
            {
                constexpr int HC = RC / 2;
                const int cbase = half * HC, sg = ch * RC + cbase;
                const float *sW = reinterpret_cast<const float *>(sB + L::kImgW);
                float v[HC];
#pragma unroll
                for (int q = 0; q < HC / 32; ++q) umma::ld32(tS + lane_off + cbase + q * 32, v + q * 32);
                float mx = -INFINITY;
#pragma unroll
                for (int i = 0; i < HC; ++i)
                    if (sg + i < re) mx = fmaxf(mx, v[i]);
                xch[half][row] = mx;
                __syncthreads();
                const float mb = fmaxf(xch[0][row], xch[1][row]) * bl2;
                bool resc = false;
                float fac = 1.f;
                if (ch == 0) {
                    mrun = mb;
                } else if (mb > mrun + 8.f) {
                    fac = ex2_approx(mrun - mb);
                    mrun = mb;
                    dn *= fac;
                    resc = true;
                }
                if (__any_sync(0xffffffffu, resc)) {  // warp-uniform: rescale this warp's rows of O
                    constexpr int HD = D / 2;
#pragma unroll
                    for (int c0 = 0; c0 < HD; c0 += 32) {
                        float o[32];
                        umma::ld32(tO + lane_off + half * HD + c0, o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= fac;
                        umma::st32(tO + lane_off + half * HD + c0, o);
                    }
                }
                float dd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int g8 = 0; g8 < HC / 8; ++g8) {
                    uint32_t pk[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int cl = g8 * 8 + 2 * i;
                        const float p0 = (sg + cl < re) ? ex2_approx(fmaf(v[cl], bl2, -mrun)) : 0.f;
                        const float p1 = (sg + cl + 1 < re) ? ex2_approx(fmaf(v[cl + 1], bl2, -mrun)) : 0.f;
                        const __nv_bfloat162 pb = __floats2bfloat162_rn(p0, p1);
                        dd[i] = fmaf(__bfloat162float(pb.x), sW[cbase + cl], dd[i]);
                        dd[i] = fmaf(__bfloat162float(pb.y), sW[cbase + cl + 1], dd[i]);
                        pk[i] = *reinterpret_cast<const uint32_t *>(&pb);
                    }
                    *reinterpret_cast<uint4 *>(sP + umma::sw128_offset(row, cbase + g8 * 8, 128)) =
                        make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                dn += (dd[0] + dd[1]) + (dd[2] + dd[3]);
            }
            umma::fence_async_smem();
            umma::fence_before_sync();
            __syncthreads();
            umma::fence_after_sync();
            if (tid == 0) {
                umma::gemm_128xNxK(tO, smem_u32(sP), smem_u32(sB + L::kImgXh), D, RC, ch > 0);
                if (L::kSplitX) umma::gemm_128xNxK(tO, smem_u32(sP), smem_u32(sB + L::kImgXl), D, RC, true);
                umma::commit(&bars[0]);
            }
            mbar_wait(&bars[0], mph);
            mph ^= 1u;
            umma::fence_after_sync();
            if (tid == 0) issue();  // buffer b retired: prefetch the chunk after next into it
        }
        __syncthreads();  // xch free
        xch[half][row] = dn;
        __syncthreads();
        const float den = xch[0][row] + xch[1][row];
        {
            const int64_t qi = q0 + row;
            const float inv = (nch > 0 && den > 0.f) ? 1.f / den : 0.f;
            constexpr int HD = D / 2;
#pragma unroll
            for (int c0 = 0; c0 < HD; c0 += 32) {
                const int cc0 = half * HD + c0;
                float v[32];
                umma::ld32(tO + lane_off + cc0, v);
                if (qi < m) {
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        float o0 = inv != 0.f ? v[2 * i] * inv : 0.f, o1 = inv != 0.f ? v[2 * i + 1] * inv : 0.f;
                        if (clip) {
                            o0 = fminf(fmaxf(o0, __bfloat162float(sVmin[cc0 + 2 * i])), __bfloat162float(sVmax[cc0 + 2 * i]));
                            o1 = fminf(fmaxf(o1, __bfloat162float(sVmin[cc0 + 2 * i + 1])), __bfloat162float(sVmax[cc0 + 2 * i + 1]));
                        }
                        const __nv_bfloat162 ob = __floats2bfloat162_rn(o0, o1);
                        pk[i] = *reinterpret_cast<const uint32_t *>(&ob);
                    }
                    uint4 *dst = reinterpret_cast<uint4 *>(O + (head * m + qi) * D + cc0);
#pragma unroll
                    for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
                }
            }
        }
        umma::fence_before_sync();
        __syncthreads();
        umma::fence_after_sync();
    }
    if (w == 0) umma::tmem_dealloc(tbase, 256);
}

template <int D>
int launch_attend_tc_long(const Dims &Dm, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                          const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws,
                          cudaStream_t st) {
    using L = TcLong<D>;
    if (!ws) return -1;
    const int nch = (int)ceil_div(Dm.r, L::RC);
    unsigned char *img = static_cast<unsigned char *>(ws);
    launch_pdl(attend_long_prep_kernel<D>, dim3(nch, (unsigned)Dm.units(), kPrepParts), dim3(256), 0, st,
               static_cast<const __nv_bfloat16 *>(KS), X, r_eff, Dm.r, nch, img);
    auto kern = attend_tc_long_kernel<D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    const int64_t tph = ceil_div(Dm.m, 128);
    const int64_t total = tph * Dm.hq * Dm.batch;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>(total, sms);
    kern<<<grid, kTcThreads, L::kTotal, st>>>(static_cast<const __nv_bfloat16 *>(Q), img, r_eff,
                                              static_cast<const __nv_bfloat16 *>(vmin),
                                              static_cast<const __nv_bfloat16 *>(vmax), Dm.m, nch, Dm.group(), Dm.hq,
                                              Dm.hkv, (float)beta, clip, static_cast<__nv_bfloat16 *>(O), tph, total);
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

// =====================================================================================
// Warp-specialised tcgen05 attend (bf16, d in {64, 128}, any r): A5 / Alg 3 with two
// 128-query tiles in flight per CTA (a "pair" of tiles of one unit), the coreset streamed in chunks of
// RC = 128 rows (the TcLong images above: [K_S chunk | X_hi^T (| X_lo^T) | w]).
//   warp 0        producer: Q tiles by TMA tensor copies (128-byte swizzle, the UMMA K-major layout),
//                 coreset chunk images by 1-D bulk copies into a 2-buffer ring;
//   warp 1        MMA issuer (one thread): per chunk c, for each tile t of the pair
//                   GEMM2(t, c-1): O_t += P_t X_{c-1}  (A = P from tensor memory)
//                   GEMM1(t, c):   S_t  = Q_t K_c^T
//                 (in-order tensor-core execution makes GEMM1(t, c) overwrite S_t / P_t only after
//                 GEMM2(t, c-1) has read them);
//   warps 4-7     softmax / epilogue of tile slot 0, warps 8-11 of slot 1 (thread = query row = TMEM
//                 lane): row max of the chunk, lazy running max (moves only by > 2^8, then O_t and den
//                 are rescaled in place), P = exp2(beta log2e s - M) -> bf16 packed into S_t's own
//                 columns (tcgen05.st), den += P w; after the last chunk O / den, clip (Z14, Z15),
//                 bf16 rows staged in the slot's Q buffer and written by one bulk copy per tile.
// TMEM: slot t uses columns [256 t, 256 t + 128) for S_t / P_t and [256 t + 128, 256 t + 128 + d) for O_t.
// =====================================================================================
constexpr int kWsThreads = 384;

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(x),
                 "r"(y), "r"(z), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void tma_store_commit_wait_read() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// mbarrier wait that traps after ~4 s instead of hanging the GPU (a protocol error then fails the call)
__device__ __forceinline__ void mbar_wait_ws(uint64_t *bar, uint32_t parity, int tag) {
    if (mbar_try_wait(bar, parity)) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    while (!mbar_try_wait(bar, parity)) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
        if (t1 - t0 > 4000000000ull) {
            printf("[attend_ws] block %d thread %d: barrier wait %d timed out\n", blockIdx.x, threadIdx.x, tag);
            __trap();
        }
    }
}
__device__ __forceinline__ void wg_sync(int id) {  // named barrier of one 128-thread warpgroup
    asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

template <int D> struct WsSmem {
    using L = TcLong<D>;
    static constexpr int RC = L::RC;
    static constexpr int kQ = 128 * D * 2;
    static constexpr int kOffQ = 0;                    // [2][kQ]: Q tiles (then the output staging)
    static constexpr int kOffRing = 2 * kQ;            // [2][L::kBuf] chunk images
    static constexpr int kOffBar = kOffRing + 2 * L::kBuf;
    // barriers: qfull[2], qempty[2], cfull[2], cempty[2], sfull[2], pfull[2], ofull[2]
    static constexpr int kOffTb = kOffBar + 14 * 8;
    static constexpr int kTotal = kOffTb + 16;
};

template <int D>
__global__ void __launch_bounds__(kWsThreads, 1)
    attend_ws_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap omap,
                     const unsigned char *__restrict__ img,
                     const int32_t *__restrict__ r_eff, const __nv_bfloat16 *__restrict__ vmin,
                     const __nv_bfloat16 *__restrict__ vmax, int64_t m, int nch_max, int group, int hq, int hkv,
                     float beta, int clip, int64_t tiles_per_head, int64_t total_tiles) {
    pdl_wait();
    using L = TcLong<D>;
    using W = WsSmem<D>;
    constexpr int RC = W::RC;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;
    if (smem_u32(sm) & 1023u) __trap();
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + W::kOffBar);
    uint64_t *qfull = bars, *qempty = bars + 2, *cfull = bars + 4, *cempty = bars + 6, *sfull = bars + 8;
    uint64_t *pfull = bars + 10, *ofull = bars + 12;
    uint32_t &tbase = *reinterpret_cast<uint32_t *>(sm + W::kOffTb);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;

    if (w == 0) umma::tmem_alloc(&tbase, 512);
    if (tid == 0) {
        for (int t = 0; t < 2; ++t) {
            mbar_init(&qfull[t], 1);
            mbar_init(&qempty[t], 1);
            mbar_init(&cfull[t], 1);
            mbar_init(&cempty[t], 1);
            mbar_init(&sfull[t], 1);
            mbar_init(&pfull[t], 128);
            mbar_init(&ofull[t], 1);
        }
        fence_mbar_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tb = tbase;

    const int64_t tpc = ceil_div(total_tiles, (int64_t)gridDim.x);
    const int64_t t_begin = (int64_t)blockIdx.x * tpc, t_end = std::min<int64_t>(total_tiles, t_begin + tpc);
    auto unit_of = [&](int64_t tile) {
        const int64_t head = tile / tiles_per_head;
        return (int)(head / hq) * hkv + (int)(head % hq) / group;
    };
    // the pair sequence: tile A = t, tile B = t + 1 when it exists and shares A's unit (and its chunks)
    auto pair_b = [&](int64_t t) { return (t + 1 < t_end && unit_of(t + 1) == unit_of(t)) ? t + 1 : (int64_t)-1; };
    auto nchunks = [&](int u) { return (int)std::max<int64_t>(1, ceil_div(r_eff[u], RC)); };

    if (w == 0) {
        // ================= producer =================
        if (lane == 0) {
            uint32_t nq[2] = {0, 0}, cseq = 0;
            for (int64_t t = t_begin; t < t_end;) {
                const int64_t tB = pair_b(t);
                const int u = unit_of(t);
                for (int s = 0; s < 2; ++s) {
                    const int64_t tt = s == 0 ? t : tB;
                    if (tt < 0) continue;
                    mbar_wait_ws(&qempty[s], (nq[s] & 1u) ^ 1u, 1);
                    ++nq[s];
                    const int64_t head = tt / tiles_per_head, q0 = (tt % tiles_per_head) * 128;
                    mbar_arrive_expect_tx(&qfull[s], (uint32_t)W::kQ);
                    unsigned char *dq = sm + W::kOffQ + s * W::kQ;
#pragma unroll
                    for (int kb = 0; kb < D / 64; ++kb)  // rows >= m: zero-filled out-of-bounds box rows
                        tma_load_3d(dq + kb * 128 * 128, &qmap, kb * 64, (int)q0, (int)head, &qfull[s]);
                }
                const int C = nchunks(u);
                for (int c = 0; c < C; ++c, ++cseq) {
                    const int b = cseq & 1;
                    mbar_wait_ws(&cempty[b], ((cseq >> 1) & 1u) ^ 1u, 2);
                    mbar_arrive_expect_tx(&cfull[b], (uint32_t)L::kImg);
                    bulk_g2s(sm + W::kOffRing + b * L::kBuf, img + ((int64_t)u * nch_max + c) * L::kImg, (uint32_t)L::kImg,
                             &cfull[b]);
                }
                t = tB >= 0 ? tB + 1 : t + 1;
            }
        }
    } else if (w == 1) {
        // ================= MMA issuer =================
        if (lane == 0) {
            uint32_t nq[2] = {0, 0}, np[2] = {0, 0}, cseq = 0;
            const uint32_t tS[2] = {tb, tb + 256}, tO[2] = {tb + 128, tb + 384};
            auto gemm1 = [&](int s, const unsigned char *chunk) {
                umma::gemm_128xNxK(tS[s], smem_u32(sm + W::kOffQ + s * W::kQ), smem_u32(chunk + L::kImgK), RC, D, false);
                umma::commit(&sfull[s]);
            };
            auto gemm2 = [&](int s, const unsigned char *chunk, bool acc) {
                mbar_wait_ws(&pfull[s], np[s] & 1u, 3);
                ++np[s];
                umma::fence_after_sync();
                umma::gemm_128xNxK_tmem_a(tO[s], tS[s], smem_u32(chunk + L::kImgXh), D, RC, acc);
                if (L::kSplitX) umma::gemm_128xNxK_tmem_a(tO[s], tS[s], smem_u32(chunk + L::kImgXl), D, RC, true);
            };
            for (int64_t t = t_begin; t < t_end;) {
                const int64_t tB = pair_b(t);
                const int ns = tB >= 0 ? 2 : 1;
                const int C = nchunks(unit_of(t));
                for (int s = 0; s < ns; ++s) {
                    mbar_wait_ws(&qfull[s], nq[s] & 1u, 4);
                    ++nq[s];
                }
                const unsigned char *prev = nullptr;
                for (int c = 0; c < C; ++c, ++cseq) {
                    const int b = cseq & 1;
                    const unsigned char *chunk = sm + W::kOffRing + b * L::kBuf;
                    mbar_wait_ws(&cfull[b], (cseq >> 1) & 1u, 5);
                    umma::fence_after_sync();
                    for (int s = 0; s < ns; ++s) {
                        if (c > 0) gemm2(s, prev, c > 1);
                        gemm1(s, chunk);
                    }
                    if (c > 0) umma::commit(&cempty[(cseq - 1) & 1]);  // chunk c-1: both GEMM2 issued
                    prev = chunk;
                }
                for (int s = 0; s < ns; ++s) {
                    gemm2(s, prev, C > 1);
                    umma::commit(&ofull[s]);
                }
                umma::commit(&cempty[(cseq - 1) & 1]);
                t = tB >= 0 ? tB + 1 : t + 1;
            }
        }
    } else if (w >= 4) {
        // ================= softmax / epilogue warpgroups =================
        const int s = (w - 4) >> 2;             // tile slot
        const int row = tid & 127;              // query row of the tile = TMEM lane
        const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
        const uint32_t tS = tb + 256 * s + lane_off, tO = tb + 256 * s + 128 + lane_off;
        const float bl2 = beta * 1.4426950408889634f;
        uint32_t ns_ph = 0, no_ph = 0, cseq = 0;
        unsigned char *stage = sm + W::kOffQ + s * W::kQ;
        for (int64_t t = t_begin; t < t_end;) {
            const int64_t tB = pair_b(t);
            const int u = unit_of(t);
            const int re = r_eff[u];
            const int C = nchunks(u);
            const int64_t tt = s == 0 ? t : tB;
            if (tt < 0) {  // slot 1 idle for this pair: follow the chunk sequence only
                cseq += C;
                t = t + 1;
                continue;
            }
            float M = -INFINITY, den = 0.f;
            for (int c = 0; c < C; ++c, ++cseq) {
                const unsigned char *chunk = sm + W::kOffRing + (cseq & 1) * L::kBuf;
                const float *sW = reinterpret_cast<const float *>(chunk + L::kImgW);
                mbar_wait_ws(&sfull[s], ns_ph, 6);
                ns_ph ^= 1u;
                umma::fence_after_sync();
                const int lim = re - c * RC;  // valid columns of this chunk
                // pass 1: the chunk's row max over valid columns (two TMEM loads in flight per wait)
                float mx = -INFINITY;
#pragma unroll
                for (int g = 0; g < RC / 32; ++g) {
                    float v[32];
                    umma::ld32(tS + g * 32, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (g * 32 + i < lim) mx = fmaxf(mx, v[i]);
                }
                const float mb = mx * bl2;
                bool resc = false;
                float fac = 1.f;
                if (c == 0) {
                    M = mb;
                } else if (mb > M + 8.f) {  // lazy: P <= 2^8 otherwise
                    fac = ex2_approx(M - mb);
                    M = mb;
                    den *= fac;
                    resc = true;
                }
                // warp-uniform (tcgen05.ld / st are warp-collective): rows without a new max scale by 1.
                // O_t of chunks < c is complete (this chunk's S commit follows their GEMM2)
                if (__any_sync(0xffffffffu, resc)) {
#pragma unroll
                    for (int c0 = 0; c0 < D; c0 += 32) {
                        float o[32];
                        umma::ld32(tO + c0, o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= fac;
                        umma::st32(tO + c0, o);
                    }
                }
                const float Mx = (M == -INFINITY) ? 0.f : M;  // a row with no valid column: all P = 0
                // pass 2: P = exp2(bl2 s - M) -> bf16 pairs into S_t's columns [0, RC/2) (group g's
                // pairs overwrite columns already read); den += P w with the fp32 P
                float dd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int g = 0; g < RC / 32; ++g) {
                    float v[32];
                    umma::ld32(tS + g * 32, v);
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int cl = g * 32 + 2 * i;
                        const float2 w2 = *reinterpret_cast<const float2 *>(sW + cl);
                        const float p0 = (cl < lim) ? ex2_approx(fmaf(v[2 * i], bl2, -Mx)) : 0.f;
                        const float p1 = (cl + 1 < lim) ? ex2_approx(fmaf(v[2 * i + 1], bl2, -Mx)) : 0.f;
                        dd[(2 * i) & 3] = fmaf(p0, w2.x, dd[(2 * i) & 3]);
                        dd[(2 * i + 1) & 3] = fmaf(p1, w2.y, dd[(2 * i + 1) & 3]);
                        const __nv_bfloat162 pb = __floats2bfloat162_rn(p0, p1);
                        pk[i] = *reinterpret_cast<const uint32_t *>(&pb);
                    }
                    umma::st16u(tS + g * 16, pk);
                }
                den += (dd[0] + dd[1]) + (dd[2] + dd[3]);
                umma::fence_before_sync();
                mbar_arrive(&pfull[s]);
            }
            // ---- epilogue: O / den, clip, bf16 rows staged in the slot's Q buffer, one bulk store
            mbar_wait_ws(&ofull[s], no_ph, 7);
            no_ph ^= 1u;
            umma::fence_after_sync();
            const int64_t head = tt / tiles_per_head, q0 = (tt % tiles_per_head) * 128;
            const float inv = den > 0.f ? 1.f / den : 0.f;
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) {
                float v[32];
                umma::ld32(tO + c0, v);
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int col = c0 + 2 * i;
                    float o0 = v[2 * i] * inv, o1 = v[2 * i + 1] * inv;
                    if (clip) {
                        o0 = fminf(fmaxf(o0, __bfloat162float(vmin[(int64_t)u * D + col])), __bfloat162float(vmax[(int64_t)u * D + col]));
                        o1 = fminf(fmaxf(o1, __bfloat162float(vmin[(int64_t)u * D + col + 1])),
                                   __bfloat162float(vmax[(int64_t)u * D + col + 1]));
                    }
                    const __nv_bfloat162 ob = __floats2bfloat162_rn(o0, o1);
                    pk[i] = *reinterpret_cast<const uint32_t *>(&ob);
                }
                // the 128-byte-swizzled K-major layout of the O tensor map (bank-conflict free by row)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int col = c0 + 8 * q;
                    *reinterpret_cast<uint4 *>(stage + umma::sw128_offset(row, col, 128)) =
                        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                }
            }
            fence_proxy_async_smem();
            wg_sync(3 + s);
            if (row == 0) {  // rows >= m of the head are outside the O tensor map: clipped by the TMA unit
#pragma unroll
                for (int kb = 0; kb < D / 64; ++kb)
                    tma_store_3d(&omap, stage + kb * 128 * 128, kb * 64, (int)q0, (int)head);
                tma_store_commit_wait_read();
                mbar_arrive(&qempty[s]);  // the Q buffer is free for the producer
            }
            t = tB >= 0 ? tB + 1 : t + 1;
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (w == 0) umma::tmem_dealloc(tbase, 512);
}

template <int D>
int launch_attend_ws(const Dims &Dm, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                     const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws, cudaStream_t st) {
    using L = TcLong<D>;
    using W = WsSmem<D>;
    if (!ws) return -1;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult qr;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess || !fn)
            return -1;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // Q and O as 3-D tensors [batch * hq][m][D] bf16; boxes of 64 columns x 128 rows x 1 head with the
    // 128-byte swizzle of the UMMA K-major layout: rows past m of a head are out of bounds (zero on
    // load, dropped on store)
    CUtensorMap qmap, omap;
    const cuuint64_t gdim[3] = {(cuuint64_t)D, (cuuint64_t)Dm.m, (cuuint64_t)Dm.batch * Dm.hq};
    const cuuint64_t gstride[2] = {(cuuint64_t)D * 2, (cuuint64_t)Dm.m * D * 2};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    for (int k = 0; k < 2; ++k)
        if (encode(k ? &omap : &qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(k ? O : Q), gdim, gstride,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -1;
    const int nch = (int)ceil_div(Dm.r, L::RC);
    unsigned char *img = static_cast<unsigned char *>(ws);
    launch_pdl(attend_long_prep_kernel<D>, dim3(nch, (unsigned)Dm.units(), kPrepParts), dim3(256), 0, st,
               static_cast<const __nv_bfloat16 *>(KS), X, r_eff, Dm.r, nch, img);
    auto kern = attend_ws_kernel<D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, W::kTotal);
    const int64_t tph = ceil_div(Dm.m, 128);
    const int64_t total = tph * Dm.hq * Dm.batch;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // whole pairs per CTA: an even tile count per CTA keeps the pairs of a head aligned
    int64_t tpc = ceil_div(total, (int64_t)sms);
    tpc += tpc & 1;
    const int grid = (int)ceil_div(total, tpc);
    launch_pdl(kern, dim3(grid), dim3(kWsThreads), (size_t)W::kTotal, st, qmap, omap, (const unsigned char *)img, r_eff,
               static_cast<const __nv_bfloat16 *>(vmin), static_cast<const __nv_bfloat16 *>(vmax), Dm.m, nch,
               Dm.group(), Dm.hq, Dm.hkv, (float)beta, clip, tph, total);
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

template <typename T, int D>
int launch_attend_td(const Dims &Dm, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                     const void *vmin, const void *vmax, double beta, int clip, void *O, cudaStream_t st) {
    if (Dm.m == 0) return 0;
    constexpr int DC = D + 1;
    const size_t smem = ((size_t)kBM * (D + 1) + (size_t)kRT * (D + 1) + (size_t)kRT * (DC + 1) +
                         (size_t)kBM * (kRT + 1) + kBM) * sizeof(float);
    auto kern = attend_kernel<T, D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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

// 0: CUDA-core kernel, 1: tcgen05 kernel with the coreset resident, 2: tcgen05 kernel streaming r > 256,
// 3: decode kernel (kvcache.cu) for m <= kDecodeMaxM queries per q-head, 4: warp-specialised tcgen05
// kernel (two query tiles in flight, TMA, P in tensor memory)
static int attend_path(const Dims &D) {
    const char *mode = std::getenv("WC_ATTEND");  // "cuda" / "tc" / "ws": force a path (A/B tests)
    if (mode && std::strcmp(mode, "cuda") == 0) return 0;
    if (D.m > 0 && D.m <= kDecodeMaxM) return 3;
    if (!(D.dtype == 1 && (D.d == 64 || D.d == 128) && D.m > 0)) return 0;
    if (mode && std::strcmp(mode, "tc") == 0) return D.r <= 256 ? 1 : 2;  // the round-1 tcgen05 kernels
    return 4;
}

static int attend_rp(const Dims &D) { return D.r <= 32 ? 32 : D.r <= 64 ? 64 : D.r <= 128 ? 128 : 256; }
template <int D> static int img_stride(int rp) {
    switch (rp) {
        case 32: return TcSmem<D, 32>::kImgStride;
        case 64: return TcSmem<D, 64>::kImgStride;
        case 128: return TcSmem<D, 128>::kImgStride;
        default: return TcSmem<D, 256>::kImgStride;
    }
}

size_t attend_ws_bytes(const Dims &D) {
    if (attend_path(D) == 3) return attend_decode_ws_bytes(D);
    if (attend_path(D) == 1) {
        const int rp = attend_rp(D);
        const int stride = D.d == 64 ? img_stride<64>(rp) : img_stride<128>(rp);
        return (size_t)D.units() * stride;
    }
    if (attend_path(D) != 2 && attend_path(D) != 4) return 0;
    const size_t img = D.d == 64 ? TcLong<64>::kImg : TcLong<128>::kImg;
    return D.units() * (size_t)ceil_div(D.r, 128) * img;
}

int launch_attend(const Dims &D, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                  const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws, cudaStream_t st) {
    const int path = attend_path(D);
    if (path == 3) return launch_attend_decode(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
    if (path == 4) {
        if (D.d == 64) return launch_attend_ws<64>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
        return launch_attend_ws<128>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
    }
    if (path == 2) {
        if (D.d == 64) return launch_attend_tc_long<64>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
        return launch_attend_tc_long<128>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
    }
    if (path == 1) {
        const int rp = attend_rp(D);
        if (D.d == 64) {
            switch (rp) {
                case 32: return launch_attend_tc<64, 32>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
                case 64: return launch_attend_tc<64, 64>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
                case 128: return launch_attend_tc<64, 128>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
                default: return launch_attend_tc<64, 256>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
            }
        }
        switch (rp) {
            case 32: return launch_attend_tc<128, 32>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
            case 64: return launch_attend_tc<128, 64>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
            case 128: return launch_attend_tc<128, 128>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
            default: return launch_attend_tc<128, 256>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, ws, st);
        }
    }
    if (D.dtype == 0) return launch_attend_t<float>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, st);
    return launch_attend_t<__nv_bfloat16>(D, Q, KS, X, r_eff, vmin, vmax, beta, clip, O, st);
}

}  // namespace wc
