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

constexpr int kBMax = 32;  // largest supported block size b (candidate slots of the NSL = 32 plan)

// Warp roles: compute warps 0..kCW-1, the TMA producer warp kWP, the rejection warp kWE.  The
// rejection warp is warp 11, on SM sub-partition 3 (warps 9 and 10 leave at once): sub-partition 3
// hosts compute warps 3 and 7, the last warps of a super-tile, which are the ones idle in a partial
// tile, so the sequential rejection chain is not starved of issue slots by two DMMA streams.  12 warps
// cost no registers over 10 (the register file is allocated in 4-warp units: 168 per thread either way).
constexpr int kWP = kCW, kWE = kCW + 3;
constexpr int kBThreads = kCT + 128;
// named barrier 2: the compute warps and the rejection warp (hand-over of H and of the accepted pivots)
__device__ __forceinline__ void ce_sync() { asm volatile("bar.sync 2, %0;" ::"n"(kCT + 32) : "memory"); }

__device__ __forceinline__ double accept_uniform(uint64_t seed, uint32_t cand, uint64_t unit) {
    uint32_t c[4] = {cand, (uint32_t)unit, (uint32_t)(unit >> 32), 0x41435054u};  // 'ACPT'
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double x = (double)(c[0] >> 5), y = (double)(c[1] >> 6);
    return (x * 67108864.0 + y) * (1.0 / 9007199254740992.0);
}

// -x by the sign bit (an integer op: no fp64-pipe instruction ahead of the DMMA that consumes it)
__device__ __forceinline__ double dneg(double x) {
    return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x));
}

// 1/sqrt(h) in fp64: MUFU rsqrt of the float value, then two Newton steps (2^-23 -> 2^-46 -> fp64
// rounding); the library rsqrt(double) carries a much longer dependent chain.
__device__ __forceinline__ double rsqrt_nr(double h) {
    if (!(h > 1e-30 && h < 1e30)) return 1.0 / sqrt(h);
    double y = (double)rsqrtf((float)h);
    y = y * fma(-0.5 * h * y, y, 1.5);
    y = y * fma(-0.5 * h * y, y, 1.5);
    return y;
}

struct BlkArgs {
    const void *K;
    double *stats;
    const double *nrm2;
    double *p;      // [2][units][n]
    double *F;      // per unit tile-major [cpu][nst][r][BT]
    double *part;   // [units][2][kMaxCpu]
    unsigned *bar;  // [units]
    double *gsum;   // [units][2][ngroups] residual sums of 32-key groups
    double *rej;    // [units][kRejStride]: flag (u64 epoch), na, Fx, rinvA, sA, jA, perm of the last block
    int32_t *S;
    int32_t *r_eff;
    double *L;
    int64_t n;                 // keys per sub-unit buffer (the largest sub-unit)
    int bins;                  // sub-unit geometry (Dims::bins, nb, unit_n; sub_unit())
    int64_t nb, unit_n;
    int units, r, cpu, b;
    uint64_t seed;
    uint64_t unit0;  // Philox id of sub-unit 0 (wc_opts.unit_offset [x B]); unit u draws stream unit0 + u
    unsigned long long *trace;  // debug (WC_SELECT_TRACE): [r][16] globaltimer stamps of CTA 0 per block
};

constexpr int kTS = 32;  // trace stamps per block
// a.rej layout per unit (doubles): [0] flag = 1 + the block index of the result (u64 bits), [1] na,
// then Fx [kBMax^2], rinvA, sA, jA, perm [kBMax each] (the ints as exact doubles)
constexpr int kRjFx = 8, kRjRinv = kRjFx + 32 * 32, kRjSA = kRjRinv + 32, kRjJA = kRjSA + 32, kRjPerm = kRjJA + 32;
static_assert(kRjPerm + 32 <= kRejStride, "rejection result layout");
__device__ __forceinline__ unsigned long long btimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define WC_BTR(k)                                                                                   \
    do {                                                                                            \
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && blk < a.r) a.trace[blk * kTS + (k)] = btimer(); \
    } while (0)
#define WC_BTRE(k)                                                                                  \
    do {                                                                                            \
        if (a.trace && blockIdx.x == 0 && lane == 0 && blk < a.r) a.trace[blk * kTS + (k)] = btimer(); \
    } while (0)

constexpr int kBR = 4;  // F rows per quad = per ring stage = one DMMA k-step

// F layout (per unit, quad-interleaved tile-major): the CTA slices [cpu][chunk keys], each cut into
// super-tiles of BT keys (the last one wk <= BT wide); within a super-tile the rows come in quads
// (rows 4Q .. 4Q + 3) stored key-major, F[q, key] at  ((q / 4) * wk + key) * 4 + q % 4.  A quad of a
// super-tile is one contiguous run (one bulk copy per ring stage) and a candidate's column is one
// 32-byte sector per quad (the gather reads r4 / 4 sectors instead of r scattered doubles).
__host__ __device__ __forceinline__ int f_r4(int r) { return (r + 3) & ~3; }

// Plan of the candidate-slot count NSL (16 or 32): NT 8-column MMA n-tiles of slots, MT 8-key MMA
// row tiles per compute warp (MT * NT * 2 = 32 fp64 accumulators per thread either way), BT keys per
// super-tile (the tile-major F width); a ring stage holds one quad [BT][4] (an A-fragment load of
// 8 keys x 4 rows is 32 consecutive doubles: conflict-free).
template <int NSL> struct BPlan {
    static constexpr int NT = NSL / 8;
    static constexpr int MT = 128 / NSL;
    static constexpr int KPW = 8 * MT;    // keys per compute warp per super-tile
    static constexpr int KPL = KPW / 32;  // keys per lane in the per-key triangle
    static constexpr int BT = kCW * KPW;  // keys per super-tile (512 for NSL = 16, 256 for NSL = 32)
    static constexpr int STAGE = BT * kBR;  // doubles per ring stage
    static constexpr int SPITCH = NSL + 1;  // staging row pitch (doubles) of the per-key triangle
};

// fp64 tensor-core MMA (DMMA) m8n8k4: C += A B with A 8x4 row-major (lane l holds A[l/4][l%4]),
// B 4x8 column-major (lane l holds B[l%4][l/4]), C 8x8 (lane l holds C[l/4][2(l%4) + {0,1}]).
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// MMA-operand layouts of the candidate pivot columns (NSL slots p):
//   Fcol: F[q, s_p] as NSL rows of stride ldc = 16k + 4 doubles: lane (tq, g) of the k-step at q0
//        reads Fcol[(8 nt + g) * ldc + q0 + tq];
//   kcB: centred key k_sp - kbar at dim = tq * (D/4) + t (lane tq owns a contiguous run of D/4 dims),
//        stored at ((t * NT + p/8) * 8 + p%8) * 4 + tq: a half-warp of 64-bit loads hits 16 distinct
//        consecutive doubles.
template <int D, int NSL> __device__ __forceinline__ int kcb(int dim, int p) {
    constexpr int DQ = D / 4;
    return (((dim % DQ) * (NSL / 8) + (p >> 3)) * 8 + (p & 7)) * 4 + dim / DQ;
}

// TC consecutive raw key elements of one row held as 32-bit words; elem() widens exactly to fp64.
template <typename T, int TC> struct KChunk {
    static constexpr int kWords = TC * (int)sizeof(T) / 4;
    uint32_t w[kWords];
    __device__ __forceinline__ void load(const T *p) {
        if constexpr (kWords == 2) {
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
            w[0] = v.x; w[1] = v.y;
        } else {
#pragma unroll
            for (int q = 0; q < kWords / 4; ++q) {
                const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p) + q);
                w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
            }
        }
    }
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int q = 0; q < kWords; ++q) w[q] = 0u;
    }
    __device__ __forceinline__ double elem(int tt) const {
        if constexpr (sizeof(T) == 2) {
            const uint32_t x = w[tt >> 1];
            return (double)__uint_as_float((tt & 1) ? (x & 0xffff0000u) : (x << 16));
        } else {
            return (double)__uint_as_float(w[tt]);
        }
    }
};

// Per-key triangle of KSN keys per lane at once (independent fp64 chains interleaved):
//   F[i+aa, l] = (G[l, aa] - sum_{a2<aa} F[i+a2, l] F[i+a2, s_aa]) * (1 / sqrt(p_{s_aa}))
// for the accepted slots aa < na in acceptance order, the residual downdate with the clamp (Z4) and
// p_s <- 0.  stg: the staged G rows [32 KSN keys][NSL + 1].  DIRECT: F[i + aa, key] is stored (key < hi)
// at frow[h] + ((i + aa) / 4) * 4 wk + (i + aa) % 4 (frow[h]: the key's column in quad 0 of its
// super-tile) as soon as it is computed; else it replaces G[key, aa] in stg (read just before) for the
// coalesced write_f_rows.  Measured: the staged write-out wins on full interleaved super-tiles (the
// headline), the direct stores on short contiguous slices (ViT).
template <int NSL, int KSN>
__device__ __forceinline__ void key_triangle_staged(double *stg, int lane, const double *Fx, const double *rinvA,
                                             const int *sA, int na, const int64_t (&key)[KSN],
                                             double (&f)[KSN][NSL], double (&pl)[KSN]) {
    constexpr int SP = NSL + 1;
#pragma unroll
    for (int aa = 0; aa < NSL; ++aa) {
#pragma unroll
        for (int h = 0; h < KSN; ++h) f[h][aa] = 0.0;
        if (aa < na) {
            const double *fx = Fx + aa * NSL;
            double c0v[KSN], c1v[KSN];  // two partial sums per key shorten the dependent chain
#pragma unroll
            for (int h = 0; h < KSN; ++h) {
                c0v[h] = stg[(32 * h + lane) * SP + aa];
                c1v[h] = 0.0;
            }
#pragma unroll
            for (int a2 = 0; a2 < aa; ++a2) {
                const double x = fx[a2];
#pragma unroll
                for (int h = 0; h < KSN; ++h) {
                    if (a2 & 1) c1v[h] = fma(-f[h][a2], x, c1v[h]);
                    else c0v[h] = fma(-f[h][a2], x, c0v[h]);
                }
            }
            const double ra = rinvA[aa];
            const int sa = sA[aa];
#pragma unroll
            for (int h = 0; h < KSN; ++h) {
                const double fv = (c0v[h] + c1v[h]) * ra;
                f[h][aa] = fv;
                stg[(32 * h + lane) * SP + aa] = fv;
                const double qd = __dadd_rn(pl[h], -__dmul_rn(fv, fv));
                pl[h] = (qd > 0.0 && key[h] != sa) ? qd : 0.0;
            }
        }
    }
}

// The same triangle with each F[i + aa, key] stored (key < hi) as soon as it is computed, at frow[h] +
// ((i + aa) / 4) * 4 wk + (i + aa) % 4 (frow[h]: the key's column in quad 0 of its super-tile), and zeros
// to the end of the last quad.  Measured: the staged write-out (key_triangle_staged + write_f_rows) wins
// on full interleaved super-tiles (the headline), these direct stores on short contiguous slices (ViT).
template <int NSL, int KSN>
__device__ __forceinline__ void key_triangle_direct(double *stg, int lane, const double *Fx, const double *rinvA,
                                                    const int *sA, int na, const int64_t (&key)[KSN], int64_t hi,
                                                    double *const (&frow)[KSN], int wk, int i,
                                                    double (&f)[KSN][NSL], double (&pl)[KSN]) {
    constexpr int SP = NSL + 1;
#pragma unroll
    for (int aa = 0; aa < NSL; ++aa) {
#pragma unroll
        for (int h = 0; h < KSN; ++h) f[h][aa] = 0.0;
        if (aa < na) {
            const double *fx = Fx + aa * NSL;
            double c0v[KSN], c1v[KSN];  // two partial sums per key shorten the dependent chain
#pragma unroll
            for (int h = 0; h < KSN; ++h) {
                c0v[h] = stg[(32 * h + lane) * SP + aa];
                c1v[h] = 0.0;
            }
#pragma unroll
            for (int a2 = 0; a2 < aa; ++a2) {
                const double x = fx[a2];
#pragma unroll
                for (int h = 0; h < KSN; ++h) {
                    if (a2 & 1) c1v[h] = fma(-f[h][a2], x, c1v[h]);
                    else c0v[h] = fma(-f[h][a2], x, c0v[h]);
                }
            }
            const double ra = rinvA[aa];
            const int sa = sA[aa];
            const int64_t fo = (int64_t)((i + aa) >> 2) * wk * kBR + ((i + aa) & 3);
#pragma unroll
            for (int h = 0; h < KSN; ++h) {
                const double fv = (c0v[h] + c1v[h]) * ra;
                f[h][aa] = fv;
                if (key[h] < hi) frow[h][fo] = fv;  // interleaved with the triangle's arithmetic
                const double qd = __dadd_rn(pl[h], -__dmul_rn(fv, fv));
                pl[h] = (qd > 0.0 && key[h] != sa) ? qd : 0.0;
            }
        }
    }
    // rows i + na .. the end of their quad are written as zeros, so every row of a streamed quad is
    // finite (the F-prefix DMMAs multiply rows >= i by zero B values without a predicate)
    for (int rr = i + na; rr < ((i + na + 3) & ~3); ++rr) {
        const int64_t fo = (int64_t)(rr >> 2) * wk * kBR + (rr & 3);
#pragma unroll
        for (int h = 0; h < KSN; ++h)
            if (key[h] < hi) frow[h][fo] = 0.0;
    }
}

// Staging row of the warp-local key j (0 .. 63): within each 32-key half, key 8 m + g sits in row 4 g + m,
// i.e. lane L of the per-key triangle owns key 8 (L & 3) + (L >> 2) of the half.  With the row pitch
// NSL + 1 the triangle's column reads (row = lane) and the write-out's reads (8 keys x 4 rows) are both
// conflict-free.
__device__ __forceinline__ int srow_of(int j) { return (j & ~31) + 4 * (j & 7) + ((j >> 3) & 3); }
__device__ __forceinline__ int key_of_lane(int lane) { return 8 * (lane & 3) + (lane >> 2); }


// Write-out of the new F rows i .. i + na - 1 of 8 KR consecutive warp-local keys (staging rows
// srow_of(j) hold F[i + aa, key j] at [row][aa]), plus zeros from row i + na to the end of its quad (so
// every row of a streamed quad is finite: the F-prefix DMMAs multiply rows >= i by zero B values without a
// predicate).  Per (row tile, quad) one warp store of 8 keys x 4 rows = 32 consecutive doubles of the
// quad layout; rows < i of a partial first quad are left alone.  koff: local key -> super-tile offset.
template <int NSL, int KR, typename KOff>
__device__ __forceinline__ void write_f_rows(const double *stg, int lane, KOff koff, int64_t t0, int64_t hi,
                                             double *Fk, int wk, int i, int na) {
    constexpr int SP = NSL + 1;
    const int q0 = i >> 2, q1 = (i + na + 3) >> 2;
    const int t = lane & 3;
    // the KR row tiles' offsets once; per quad all KR values are read before the KR stores are issued
    // (distinct registers: a store does not wait for the previous one to release its operands)
    int off[KR];
    bool kin[KR];
#pragma unroll
    for (int rt = 0; rt < KR; ++rt) {
        off[rt] = koff(rt * 8 + (lane >> 2));
        kin[rt] = t0 + off[rt] < hi;
    }
    for (int q = q0; q < q1; ++q) {
        const int row = 4 * q + t, aa = row - i;
        double v[KR];
#pragma unroll
        for (int rt = 0; rt < KR; ++rt) v[rt] = aa < na ? stg[srow_of(rt * 8 + (lane >> 2)) * SP + aa] : 0.0;
        double *fq = Fk + (int64_t)q * wk * kBR + t;
#pragma unroll
        for (int rt = 0; rt < KR; ++rt)
            if (row >= i && kin[rt]) fq[off[rt] * kBR] = v[rt];
    }
}

// Shared-memory carve of the kernel (the launcher sizes it with the same function).
template <int D, int NSL> struct BSmem {
    double *ring, *Fcol, *kcB, *H0, *Fcand, *Fx, *colbuf, *cp, *c0r, *vac, *unif, *rinvA, *kb, *scr, *c0p, *spart, *cpre,
        *sv, *sinc, *rts;
    int *cs, *sA, *jA, *perm;
    uint64_t *full, *empty;
    size_t bytes;
    __host__ __device__ BSmem(unsigned char *base, int NS, int ldc, int cpu) {
        using PL = BPlan<NSL>;
        size_t o = 0;
        // (base == nullptr: only the size is wanted)
        auto at = [&](size_t bytes) { unsigned char *q = base ? base + o : nullptr; o += bytes; return q; };
        auto td = [&](size_t cnt) { return reinterpret_cast<double *>(at(cnt * sizeof(double))); };
        ring = td((size_t)NS * PL::STAGE);
        Fcol = td((size_t)NSL * ldc);
        kcB = td((size_t)D * NSL);
        H0 = td(NSL * NSL);
        Fcand = td(NSL * NSL);
        Fx = td(NSL * NSL);
        colbuf = td(2 * NSL);
        cp = td(NSL);
        c0r = td(NSL);
        vac = td(NSL);
        unif = td(NSL);
        rinvA = td(NSL);
        kb = td(D + D / 8);
        scr = td(40);
        c0p = td(kCT);
        spart = td(cpu);
        cpre = td(cpu);
        rts = td(PL::BT / 8);
        sv = td(32);
        sinc = td(32);
        cs = reinterpret_cast<int *>(at(NSL * sizeof(int)));
        sA = reinterpret_cast<int *>(at(NSL * sizeof(int)));
        jA = reinterpret_cast<int *>(at(NSL * sizeof(int)));
        perm = reinterpret_cast<int *>(at(NSL * sizeof(int)));
        o = (o + 15) & ~size_t(15);
        full = reinterpret_cast<uint64_t *>(at(NS * sizeof(uint64_t)));
        empty = reinterpret_cast<uint64_t *>(at(NS * sizeof(uint64_t)));
        bytes = o;
    }
};

// ILV: warps own interleaved row tiles (w, w + 8, ..) of a super-tile, else contiguous 64-key spans
// (slices of at most BT / 2 keys: one warp per SM sub-partition, the empty warps idle).
template <typename T, int D, int NSL, bool ILV>
__global__ void __launch_bounds__(kBThreads, 1) rpc_select_blocked_kernel(BlkArgs a, int NS) {
    pdl_wait();  // the prologue's stats / nrm2 (programmatic dependent launch)
    using PL = BPlan<NSL>;
    constexpr int NT = PL::NT, MT = PL::MT, KPW = PL::KPW, KPL = PL::KPL, BT = PL::BT, STAGE = PL::STAGE;
    static_assert(MT == 4 * KPL, "row tiles 4h .. 4h + 3 hold the keys 32h .. 32h + 31 of a warp");
    constexpr int SP = PL::SPITCH;
    constexpr int DQ = D / 4;             // dims per lane per key in the kernel-dot MMA
    constexpr int TC = 4;                 // k-steps per register chunk of the K row (8 or 16 bytes per key)
    using KC = KChunk<T, TC>;
    extern __shared__ __align__(128) unsigned char smraw[];
    const int ldc = ((a.r + 15) & ~15) + 4;
    BSmem<D, NSL> sm(smraw, NS, ldc, a.cpu);
    double *ring = sm.ring, *Fcol = sm.Fcol, *kcB = sm.kcB, *H0 = sm.H0, *Fcand = sm.Fcand, *Fx = sm.Fx;
    double *colbuf = sm.colbuf, *cp = sm.cp, *c0r = sm.c0r, *vac = sm.vac, *rinvA = sm.rinvA, *kb = sm.kb;
    double *rts = sm.rts;  // per row tile residual sums of the current super-tile
    double *scr = sm.scr, *spart = sm.spart, *cpre = sm.cpre, *sv = sm.sv, *sinc = sm.sinc, *unif = sm.unif;
    int *cs = sm.cs, *sA = sm.sA, *jA = sm.jA, *perm = sm.perm;
    uint64_t *full = sm.full, *empty = sm.empty;
    __shared__ volatile int sh_stop;
    __shared__ volatile long long sh_req;  // request number << 32 | super-tile << 16 | F rows to stream
    __shared__ int sh_na, sh_cmd;

    const int tid = threadIdx.x, lane = tid & 31, w = warp_index();
    const int gid = lane >> 2, tq = lane & 3;
    const int u = blockIdx.x / a.cpu, c = blockIdx.x % a.cpu;
    const SubUnit sub = sub_unit(u, a.n, a.bins, a.nb, a.unit_n);
    const int64_t n = sub.count;  // this sub-unit's keys (a.n: the buffer stride)
    // with >= kRejMinCpu CTAs the last CTA of the unit (is_R) owns no keys: it runs the block
    // rejection and publishes the result to a.rej; the other CTAs' idle rejection warp relays it
    const bool rej_cta = a.cpu >= kRejMinCpu;
    const bool is_R = rej_cta && c == a.cpu - 1;
    const int kcta = key_ctas(a.cpu);
    const int64_t chunk = ((ceil_div(n, kcta) + 31) / 32) * 32;
    const int64_t chunk_max = ((ceil_div(a.n, kcta) + 31) / 32) * 32;
    const int64_t lo = std::min<int64_t>(n, (int64_t)c * chunk), hi = std::min<int64_t>(n, lo + chunk);
    const int nst = (int)ceil_div(hi - lo, BT);
    const int bsz = a.b;
    const uint64_t uid = a.unit0 + (uint64_t)u;
    // the per-key triangle stages both of a lane's keys at once when the ring holds [64][SP] per warp
    const bool two_keys = (size_t)NS * STAGE >= (size_t)kCW * 64 * SP;

    const T *Ku = static_cast<const T *>(a.K) + sub.base * D;
    double *st = a.stats + (int64_t)u * (kStatsHead + D);
    const int r4 = f_r4(a.r);
    double *Fu = a.F + (int64_t)u * a.cpu * chunk_max * r4;
    double *Fc = Fu + (int64_t)c * chunk * r4;
    auto tile_w = [&](int k) -> int { return (int)std::min<int64_t>(BT, chunk - (int64_t)k * BT); };

    if (tid == 0) {
        for (int q = 0; q < NS; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kCW);
        }
        flag_st(&sh_stop, 0);
        flag_st64(&sh_req, 0);
        fence_mbar_init();
    }
    __syncthreads();  // the only CTA-wide barrier: everything after is role-specific

    if (w == kWP) {
        // ============ producer warp: streams F[0:i, own slice] once per block (one bulk copy per row) ============
        if (lane == 0) {
            int stage = 0;
            uint32_t ph = 0, issued = 0, par = 0;
            long long seen = 0;
            const uint64_t pol = policy_evict_first();
            while (true) {
                long long req;
                while (((req = flag_ld64(&sh_req)) >> 32) == seen) {
                    if (flag_ld(&sh_stop)) goto drain;
                    __nanosleep(64);
                }
                seen = req >> 32;
                const int rows = (int)(req & 0xffffLL), k = (int)((req >> 16) & 0xffffLL);
                {
                    const double *blkp = Fc + (int64_t)k * r4 * BT;
                    const int wk = tile_w(k);
                    const uint32_t qb = (uint32_t)(wk * kBR * sizeof(double));  // one quad of the super-tile
                    for (int j0 = 0; j0 < rows; j0 += kBR) {
                        while (!mbar_try_wait(&empty[stage], ph ^ 1u)) {
                            if (flag_ld(&sh_stop)) goto drain;
                            __nanosleep(128);  // ring full: do not steal issue slots from the compute warp of this SMSP
                        }
                        mbar_arrive_expect_tx(&full[stage], qb);
                        double *dst = ring + (size_t)stage * STAGE;
                        // F streams through L2 evict-first so that K, p and the group sums stay resident (keeping
                        // the first F rows evict-last instead was measured slower: the 126 MB L2 thrashes); rows
                        // >= i of the last quad are streamed too and ignored by the consumer
                        bulk_g2s_hint(dst, blkp + (int64_t)j0 * wk, qb, &full[stage], pol);
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

    if (w > kWP && w < kWE) return;  // spare warps (register-allocation granularity)
    if (w == kWE && rej_cta && !is_R) {
        // ============ relay warp (a key-owning CTA of a unit with a rejection CTA): per block, wait for
        // the rejection CTA's published result, copy it into shared memory, write the L rows / S of the
        // accepted pivots this CTA owns; the compute warps pick it up at ce_sync B ============
        const double *rj = a.rej + (int64_t)u * kRejStride;
        int i = 0, blk = 0;
        while (true) {
            ce_sync();  // A: the candidates and their F columns are in shared memory (or the stop command)
            if (sh_cmd == 0) break;
            if (lane == 0) {
                while (true) {
                    unsigned long long f;
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(rj) : "memory");
                    if (f >= (unsigned long long)(blk + 1)) break;
                    __nanosleep(256);
                }
            }
            __syncwarp();
            const int nacc = (int)__ldcg(rj + 1);
            for (int idx = lane; idx < NSL * NSL; idx += 32) Fx[idx] = __ldcg(rj + kRjFx + idx);
            if (lane < NSL) {
                rinvA[lane] = __ldcg(rj + kRjRinv + lane);
                sA[lane] = (int)__ldcg(rj + kRjSA + lane);
                jA[lane] = (int)__ldcg(rj + kRjJA + lane);
                perm[lane] = (int)__ldcg(rj + kRjPerm + lane);
            }
            __syncwarp();
            for (int x = 0; x < nacc; ++x) {
                const int s = sA[x];
                if (s >= lo && s < hi) {
                    const int sl = jA[x];
                    for (int q = lane; q < i; q += 32) a.L[((int64_t)u * a.r + i + x) * a.r + q] = Fcol[(size_t)sl * ldc + q];
                    if (lane == 0) a.S[(int64_t)u * a.r + i + x] = s;
                }
            }
            if (lane == 0) sh_na = nacc;
            WC_BTRE(14);
            i += nacc;
            ++blk;
            ce_sync();  // B
        }
        return;
    }
    if (w == kWE) {
        // ============ rejection warp: per block, the sequential accept / eliminate loop of step 3 ============
        // (lane e = column e of the symmetric H in registers; column j is published through shared
        // memory).  Accepting j subtracts F_x F_e with F_x = H[x][j] / sqrt(H[j][j]), which is also
        // F[i+aa, s_x] for the later candidates x: the coefficients of every key's triangle.
        // It runs while the compute warps start the round-update GEMMs (kernel dots and F prefix over
        // all candidate slots do not depend on acceptance); they pick up its results at ce_sync B.
        int i = 0, blk = 0;
        while (true) {
            ce_sync();  // A: H0 of this block (or the stop command) is in shared memory
            if (sh_cmd == 0) break;
            // NSL = 16: the two half-warps split the rows of each column (lane = column e, rows
            // XR * h .. XR * h + XR - 1 of it), halving the fp64 instructions per step that share the
            // pipe with the compute warps' DMMA; the arithmetic per entry is unchanged
            constexpr int XH = NSL == 16 ? 2 : 1, XR = NSL / XH;
            const int e = XH == 2 ? (lane & 15) : lane, h = XH == 2 ? (lane >> 4) : 0;
            double hc[XR];
#pragma unroll
            for (int xx = 0; xx < XR; ++xx) {
                const int x = XR * h + xx;
                hc[xx] = (e < bsz && x < bsz) ? H0[x * NSL + e] : 0.0;
            }
            const int my_cs = e < bsz ? cs[e] : -1;
            const double my_vp = e < bsz ? __dmul_rn(vac[e], cp[e]) : 0.0;  // v_e p[s_e]
            bool my_acc = false;
            int nacc = 0;
#pragma unroll 1
            for (int j = 0; j < bsz && i + nacc < a.r; ++j) {
                // the lanes of column j publish it through shared memory (double-buffered by step
                // parity: the previous user of this buffer finished before the last __syncwarp); H stays
                // bitwise symmetric, so H[j][e] = H[e][j] = col[e]
                double *col = colbuf + (j & 1) * NSL;
                if (e == j) {
#pragma unroll
                    for (int xx = 0; xx < XR; ++xx) col[XR * h + xx] = hc[xx];
                }
                __syncwarp();
                const double hjj = col[j];
                const double hej = e < NSL ? col[e] : 0.0;  // H[j][e]
                const int sj = __shfl_sync(0xffffffffu, my_cs, j);
                const double vp = __shfl_sync(0xffffffffu, my_vp, j);
                const bool dup = __any_sync(0xffffffffu, my_acc && my_cs == sj);
                if (!dup && vp < hjj) {
                    const double rinv = rsqrt_nr(hjj);
                    const double fe = hej * rinv;  // F[i+nacc, s_e] = H[j][e] / sqrt(H[j][j])
                    if (h == 0 && e < NSL) Fcand[nacc * NSL + e] = (e > j && e < bsz) ? fe : 0.0;
#pragma unroll
                    for (int xx = 0; xx < XR; ++xx) {
                        const int x = XR * h + xx;
                        const double fx = col[x] * rinv;  // H[x][j] / sqrt(H[j][j])
                        if (e > j && x > j) hc[xx] = fma(-fx, fe, hc[xx]);
                    }
                    if (lane == 0) {
                        sA[nacc] = sj;
                        jA[nacc] = j;
                        rinvA[nacc] = rinv;
                    }
                    my_acc |= (e == j);
                    ++nacc;
                }
            }
            // bookkeeping of the accepted pivots: Fx[aa][a2] = F[i+a2, s_aa], perm (slot -> acceptance
            // index), the owner CTA's L rows L[i+x][0:i] = F[0:i, s_x] and S
            __syncwarp();
            for (int idx = lane; idx < NSL * NSL; idx += 32) {
                const int aa = idx / NSL, a2 = idx % NSL;
                Fx[idx] = (aa < nacc && a2 < aa) ? Fcand[a2 * NSL + jA[aa]] : 0.0;
            }
            if (lane < NSL) {
                int pa = -1;
                for (int x = 0; x < nacc; ++x) pa = (jA[x] == lane) ? x : pa;
                perm[lane] = pa;
            }
            for (int x = 0; x < nacc; ++x) {
                const int s = sA[x];
                if (s >= lo && s < hi) {
                    const int sl = jA[x];
                    for (int q = lane; q < i; q += 32) a.L[((int64_t)u * a.r + i + x) * a.r + q] = Fcol[(size_t)sl * ldc + q];
                    if (lane == 0) a.S[(int64_t)u * a.r + i + x] = s;
                }
            }
            if (lane == 0) sh_na = nacc;
            if (is_R) {  // publish the block's result for the relay warps of the other CTAs
                __syncwarp();
                double *rj = a.rej + (int64_t)u * kRejStride;
                for (int idx = lane; idx < NSL * NSL; idx += 32) rj[kRjFx + idx] = Fx[idx];
                if (lane < NSL) {
                    rj[kRjRinv + lane] = rinvA[lane];
                    rj[kRjSA + lane] = (double)sA[lane];
                    rj[kRjJA + lane] = (double)jA[lane];
                    rj[kRjPerm + lane] = (double)perm[lane];
                }
                if (lane == 0) rj[1] = (double)nacc;
                __threadfence();
                __syncwarp();
                if (lane == 0)
                    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(rj), "l"((unsigned long long)(blk + 1)) : "memory");
            }
            WC_BTRE(14);
            i += nacc;
            ++blk;
            ce_sync();  // B: the compute warps read na, Fx, perm, sA, rinvA
        }
        return;
    }

    // ================= compute warps (256 threads) =================
    const double g = st[1], mstar = st[2];
    double *p0 = a.p + (int64_t)u * a.n;
    double *p1 = a.p + ((int64_t)a.units + u) * a.n;
    double *partu = a.part + (int64_t)u * 2 * kMaxCpu;
    for (int j = tid; j < D; j += kCT) kb[j + j / 8] = st[kStatsHead + j];  // padded (bank-conflict free reads)

    // p <- kernel diagonal h~(k_l, k_l) (Alg 1); 32-key group sums (one warp per group)
    double loc = 0.0;
    {
        const int ngr0 = (int)((a.n + 31) / 32);  // group-sum stride per sub-unit (buffer size)
        double *g0s = a.gsum + (int64_t)u * 2 * ngr0;
        for (int64_t gb = lo + 32 * w; gb < hi; gb += kCT) {
            const int64_t l = gb + lane;
            double v = 0.0;
            if (l < hi) {
                v = exp(__dadd_rn(__dmul_rn(g, a.nrm2[sub.base + l]), -mstar));
                p0[l] = v;
            }
            v = warp_sum(v);
            if (lane == 0) g0s[gb / 32] = v;
            loc += lane == 0 ? v : 0.0;
        }
    }
    loc = cw_sum(loc, scr);
    // Grid-group barrier of the compute threads (as cw_group_barrier); while thread 0 waits for the
    // other CTAs, warps 1-2 draw the Philox pivot and accept uniforms of the next block's candidates
    // (they depend only on the candidate counter).
    auto block_barrier = [&](unsigned ep, uint32_t cb) {
        cw_sync();
        if (tid == 0) {
            if (a.cpu > 1) {
                asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.bar + u), "r"(1u) : "memory");
                const unsigned target = ep * (unsigned)a.cpu;
                unsigned v;
                while (true) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar + u) : "memory");
                    if (v >= target) break;
                    __nanosleep(20);
                }
            } else {
                __threadfence();
            }
        } else if (tid >= 32 && tid < 32 + 2 * NSL) {
            const int jj = (tid - 32) % NSL;
            if (tid - 32 < NSL) unif[jj] = pivot_uniform(a.seed, cb + (uint32_t)jj, uid);
            else vac[jj] = accept_uniform(a.seed, cb + (uint32_t)jj, uid);
        }
        cw_sync();
    };
    if (tid == 0) partu[c] = loc;
    unsigned epoch = 1;
    block_barrier(epoch++, 0u);

    int rstage = 0;
    uint32_t rph = 0;
    double T0 = 0.0, theta = 0.0;
    int i = 0, blk = 0;
    uint32_t cbase = 0;
    double fread = 0.0, fdot = 0.0;
    long long nreq = 0;  // requests published to the producer (thread 0)
    while (i < a.r) {
        double *cur = (blk & 1) ? p1 : p0;
        double *nxt = (blk & 1) ? p0 : p1;
        const double *pc = partu + (blk & 1) * kMaxCpu;
        double *pn = partu + ((blk + 1) & 1) * kMaxCpu;
        WC_BTR(0);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && blk < a.r) a.trace[blk * kTS + 12] = clock64();

        // ---- 1a (warp 0): per-CTA residual sums -> shared memory (one L2 read per CTA), lane
        // partition sums and their inclusive prefix, total T (fixed order)
        const int ngr = (int)((a.n + 31) / 32);
        const double *gcur = a.gsum + ((int64_t)u * 2 + (blk & 1)) * ngr;
        double *gnxt = a.gsum + ((int64_t)u * 2 + ((blk + 1) & 1)) * ngr;
        const int per = (a.cpu + 31) / 32;
        if (w == 0) {
            const int b0 = lane * per, b1 = min(a.cpu, b0 + per);
            double v = 0.0;
            if (per <= 8) {  // all of the lane's loads in flight, then the fixed-order sum
                double xs[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) xs[q] = (b0 + q < b1) ? __ldcg(pc + b0 + q) : 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (b0 + q < b1) {
                        spart[b0 + q] = xs[q];
                        v += xs[q];
                    }
                }
                WC_BTR(20);
            } else {
                for (int cc = b0; cc < b1; ++cc) {
                    const double x = __ldcg(pc + cc);
                    spart[cc] = x;
                    v += x;
                }
            }
            double incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            sv[lane] = v;
            sinc[lane] = incl;
            // inclusive prefix of the CTA sums in this order: the level-1 search of every candidate
            double ex = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) ex = 0.0;
            for (int cc = b0; cc < b1; ++cc) {
                ex += spart[cc];
                cpre[cc] = ex;
            }
        }
        cw_sync();
        const double Ttot = sinc[31];
        if (blk == 0) {
            T0 = Ttot;
            theta = 1000.0 * (double)a.r * 2.220446049250313e-16 * T0;
        }
        if (Ttot <= theta) break;  // exhausted (reading Z3), tested at block starts
        if (tid == 0) flag_st64(&sh_req, ((long long)(++nreq) << 32) | (long long)i);  // producer: F[0:i] of super-tile 0
        WC_BTR(10);

        // ---- 1b: candidates: each half-warp draws one candidate per pass (warp w: j = w + 8 h + 16 pass)
        // by the Eq. 4 inverse CDF with strict '>', hierarchically: owning CTA (prefix of CTA sums) ->
        // 32-key group (prefix of the group sums of that CTA's slice) -> key (scan of the group's 32
        // residuals).  Each level falls back to its last positive entry if rounding leaves no crossing
        // (reading Z2).
#pragma unroll 1
        for (int pass = 0; pass < NSL / 16; ++pass) {
            const int h16 = lane >> 4, l16 = lane & 15;
            const unsigned hm = 0xFFFFu << (16 * h16);
            const int j = w + kCW * (h16 + 2 * pass);
            const bool jok = j < bsz;
            const int per16 = (a.cpu + 15) / 16;
            const int b0 = l16 * per16, b1 = min(a.cpu, b0 + per16);
            const double Tw = cpre[a.cpu - 1];  // the total in the prefix's order
            const double t = jok ? unif[j] * Tw : 0.0;
            // level 1: the first CTA whose inclusive prefix exceeds t (strict '>'), else the last CTA with a
            // positive sum; tp = t - the exclusive prefix of that CTA
            int fh = -1, lp = -1;
#pragma unroll 4
            for (int cc = b0; cc < b1; ++cc) {
                const double pv = cpre[cc], sp = spart[cc];
                if (fh < 0 && pv > t) fh = cc;
                if (sp > 0.0) lp = cc;
            }
            const unsigned hit = (__ballot_sync(0xffffffffu, fh >= 0) & hm) >> (16 * h16);
            const unsigned pos = (__ballot_sync(0xffffffffu, lp >= 0) & hm) >> (16 * h16);
            const int Ln = hit ? __ffs(hit) - 1 : 31 - __clz(pos);
            const int cstar = __shfl_sync(0xffffffffu, hit ? fh : lp, Ln, 16);
            const double tp = t - (cstar > 0 ? cpre[cstar - 1] : 0.0);
            if (pass == 0) WC_BTR(16);
            // level 2: 32-key group inside c*'s slice
            const int64_t slo = std::min<int64_t>(n, (int64_t)cstar * chunk);
            const int64_t shi = std::min<int64_t>(n, slo + chunk);
            const int g0 = (int)(slo / 32), gn = (int)((shi - slo + 31) / 32);
            const int gper = (gn + 15) / 16;
            const int q0 = g0 + l16 * gper, q1 = min(g0 + gn, q0 + gper);
            constexpr int kG = 8;  // fast path: <= 128 groups per slice, kept in registers
            double gv[kG];
            double v2 = 0.0;
            if (gper <= kG) {
#pragma unroll
                for (int q = 0; q < kG; ++q) gv[q] = (q0 + q < q1) ? __ldcg(gcur + q0 + q) : 0.0;
#pragma unroll
                for (int q = 0; q < kG; ++q) v2 += gv[q];
            } else {
                for (int q = q0; q < q1; ++q) v2 += __ldcg(gcur + q);
            }
            double inc2 = v2;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, inc2, o, 16);
                if (l16 >= o) inc2 += y;
            }
            const unsigned hit2 = (__ballot_sync(0xffffffffu, q1 > q0 && inc2 > tp) & hm) >> (16 * h16);
            const unsigned pos2 = (__ballot_sync(0xffffffffu, q1 > q0 && v2 > 0.0) & hm) >> (16 * h16);
            const int L2 = hit2 ? __ffs(hit2) - 1 : 31 - __clz(pos2);
            int gstar = 0;
            double tq2 = 0.0;
            if (l16 == L2) {
                double acc = inc2 - v2;
                int gsel = -1, last = -1;
                double excl = 0.0, last_excl = 0.0;
                auto scan = [&](int q, double gg) {
                    if (gg > 0.0) { last = q; last_excl = acc; }
                    const double nacc = acc + gg;
                    if (gsel < 0 && hit2 && nacc > tp) { gsel = q; excl = acc; }
                    acc = nacc;
                };
                if (gper <= kG) {  // static register indices (no local-memory copy of gv)
#pragma unroll
                    for (int z = 0; z < kG; ++z)
                        if (z < q1 - q0) scan(q0 + z, gv[z]);
                } else {
                    for (int q = q0; q < q1; ++q) scan(q, __ldcg(gcur + q));
                }
                if (gsel < 0) { gsel = last; excl = last_excl; }
                gstar = gsel;
                tq2 = tp - excl;
            }
            gstar = __shfl_sync(0xffffffffu, gstar, L2, 16);
            tq2 = __shfl_sync(0xffffffffu, tq2, L2, 16);
            if (pass == 0) WC_BTR(17);
            // level 3: key inside the group, two keys per lane (in key order)
            const int64_t k0 = (int64_t)gstar * 32 + 2 * l16;
            const double pa = k0 < shi ? __ldcg(cur + k0) : 0.0;
            const double pb = k0 + 1 < shi ? __ldcg(cur + k0 + 1) : 0.0;
            const double v3 = pa + pb;
            double inc3 = v3;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, inc3, o, 16);
                if (l16 >= o) inc3 += y;
            }
            const unsigned hit3 = (__ballot_sync(0xffffffffu, inc3 > tq2) & hm) >> (16 * h16);
            const unsigned pos3 = (__ballot_sync(0xffffffffu, v3 > 0.0) & hm) >> (16 * h16);
            const int L3 = hit3 ? __ffs(hit3) - 1 : 31 - __clz(pos3);
            int s3 = 0;
            double psv = 0.0;
            if (l16 == L3) {  // which of the lane's two keys: strict '>' in key order, fallback to the last positive
                const double ex = inc3 - v3;
                if (hit3 && ex + pa > tq2) { s3 = 0; psv = pa; }
                else if (hit3) { s3 = 1; psv = pb; }
                else if (pb > 0.0) { s3 = 1; psv = pb; }
                else { s3 = 0; psv = pa; }
            }
            s3 = __shfl_sync(0xffffffffu, s3, L3, 16);
            psv = __shfl_sync(0xffffffffu, psv, L3, 16);
            const int sj = (int)(gstar * 32 + 2 * L3 + s3);
            if (pass == 0) WC_BTR(18);
            if (l16 == 0 && jok) {
                cs[j] = sj;
                cp[j] = psv;
            }
            // ---- 2 (the same half-warp, right after its draw): the candidate's column F[0:i, s_j], one
            // 32-byte quad sector per 4 rows of the owner's tile-major F (written by the owner CTAs in
            // earlier blocks; L2 only: an L1 line read earlier may straddle into a row another CTA wrote
            // since), and its centred key (fp64, MMA layout) with c0[j] = <kbar, k_sj - kbar>.  Slots
            // j >= b and the rows [i, i4) are zero.
            {
                double *fdst = Fcol + (size_t)j * ldc;
                const int nq = (i + 3) >> 2;
                constexpr int EPC = 16 / (int)sizeof(T);  // key elements per 16-byte chunk
                constexpr int KCH = D / EPC;              // 16-byte chunks per key row
                constexpr int KCL = (KCH + 15) / 16;      // chunks per lane
                uint4 kr[KCL];
                const double *fsrc = Fu;
                int wkj = 0;
                if (jok) {
                    const int64_t cc = sj / chunk, off = sj - cc * chunk, kk = off / BT;
                    wkj = (int)std::min<int64_t>(BT, chunk - kk * BT);
                    fsrc = Fu + cc * chunk * r4 + kk * r4 * BT + (off - kk * BT) * kBR;
#pragma unroll
                    for (int z = 0; z < KCL; ++z) {
                        const int ch = l16 + 16 * z;
                        if (ch < KCH) kr[z] = __ldg(reinterpret_cast<const uint4 *>(Ku + (int64_t)sj * D) + ch);
                    }
                }
                constexpr int kQ = 4;  // quads per lane in flight per pass (64 rows per half-warp pass)
                for (int qb = 0; qb < nq; qb += 16 * kQ) {
                    double2 v[kQ][2];
#pragma unroll
                    for (int z = 0; z < kQ; ++z) {
                        const int Q = qb + 16 * z + l16;
                        if (jok && Q < nq) {
                            const double2 *src = reinterpret_cast<const double2 *>(fsrc + (int64_t)Q * wkj * kBR);
                            v[z][0] = __ldcg(src);
                            v[z][1] = __ldcg(src + 1);
                        } else {
                            v[z][0] = v[z][1] = make_double2(0.0, 0.0);
                        }
                    }
#pragma unroll
                    for (int z = 0; z < kQ; ++z) {
                        const int Q = qb + 16 * z + l16;
                        if (Q < nq) {
                            const int q = 4 * Q;
                            fdst[q] = v[z][0].x;
                            fdst[q + 1] = q + 1 < i ? v[z][0].y : 0.0;
                            fdst[q + 2] = q + 2 < i ? v[z][1].x : 0.0;
                            fdst[q + 3] = q + 3 < i ? v[z][1].y : 0.0;
                        }
                    }
                }
                double s0 = 0.0;
#pragma unroll
                for (int z = 0; z < KCL; ++z) {
                    const int ch = l16 + 16 * z;
                    if (ch < KCH) {
                        const T *ke = reinterpret_cast<const T *>(&kr[z]);
#pragma unroll
                        for (int t = 0; t < EPC; ++t) {
                            const int e = ch * EPC + t;
                            const double kbe = kb[e + e / 8];
                            const double kc = jok ? __dadd_rn(to_f64(ke[t]), -kbe) : 0.0;
                            kcB[kcb<D, NSL>(e, j)] = kc;
                            s0 = fma(kbe, kc, s0);
                        }
                    }
                }
#pragma unroll
                for (int o = 8; o >= 1; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o, 16);
                if (l16 == 0) c0r[j] = s0;
            }
            if (pass == 0) WC_BTR(19);
            if (blk == 0 && j == 0) WC_BTR(11);
        }
        cw_sync();  // candidates, their F columns, centred keys and c0 are in shared memory
        WC_BTR(1);
        WC_BTR(2);
        const int i4 = (i + 3) & ~3;
        // ---- 3: H = h~(K_C, K_C) - F[0:i, C]^T F[0:i, C] on the fp64 tensor cores, one 8x8 tile
        // (mt, nt) per warp and pass (all k-steps of the tile in one accumulator, fixed k order: the
        // (x, e) and (e, x) tiles get the same bits, so H is bitwise symmetric).  Kernel-dot k-steps
        // first (now), F k-steps once the gather has landed.
        constexpr int NTILE = NT * NT, TPW = (NTILE + kCW - 1) / kCW;
        if (!rej_cta || is_R) {  // (a CTA that relays the rejection CTA's result needs no H)
        double hk[TPW][2], hf[TPW][2];
#pragma unroll
        for (int q = 0; q < TPW; ++q) hk[q][0] = hk[q][1] = hf[q][0] = hf[q][1] = 0.0;
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int tile = w + kCW * q;
            if (tile < NTILE) {
                const int mh = tile / NT, nh = tile % NT;
                double h2[2] = {0.0, 0.0};  // odd k-steps: a second independent DMMA chain
#pragma unroll 4
                for (int t = 0; t < DQ; t += 2) {
                    const double *b0 = kcB + (size_t)t * NSL * 4, *b1 = b0 + NSL * 4;
                    dmma(hk[q][0], hk[q][1], b0[(mh * 8 + gid) * 4 + tq], b0[(nh * 8 + gid) * 4 + tq]);
                    dmma(h2[0], h2[1], b1[(mh * 8 + gid) * 4 + tq], b1[(nh * 8 + gid) * 4 + tq]);
                }
                hk[q][0] += h2[0];
                hk[q][1] += h2[1];
            }
        }
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int tile = w + kCW * q;
            if (tile < NTILE) {
                const int mh = tile / NT, nh = tile % NT;
                for (int kq = 0; kq < i4 / 4; ++kq) {
                    const double f0 = Fcol[(size_t)(mh * 8 + gid) * ldc + 4 * kq + tq];
                    const double f1 = Fcol[(size_t)(nh * 8 + gid) * ldc + 4 * kq + tq];
                    dmma(hf[q][0], hf[q][1], f0, f1);
                }
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int x = mh * 8 + gid, e = nh * 8 + 2 * tq + hh;
                    H0[x * NSL + e] = (x == e) ? cp[x < bsz ? x : 0]
                                               : exp(__dadd_rn(__dmul_rn(g, hk[q][hh]), -mstar)) - hf[q][hh];
                }
            }
        }
        }
        if (tid == 0) sh_cmd = 1;
        ce_sync();  // A: H0, c0r complete; the rejection warp starts
        WC_BTR(3);

        // ---- 4: na F-form rounds over this CTA's keys.  Per BT-key super-tile, warp w owns keys
        // [KPW w, KPW w + KPW) as MT MMA row-tiles of 8; over the NSL candidate slots,
        //   G = h~(K_tile, K_C) - F[0:i, tile]^T F[0:i, C]
        // is accumulated on the fp64 tensor cores (kernel dot, exp in registers, then the F prefix
        // with negated ring operands); each lane then runs the triangle of its key(s) over the
        // accepted slots in acceptance order.
        int na = 0;
        loc = 0.0;
        for (int k = 0; k < nst; ++k) {
            const int64_t t0 = lo + (int64_t)k * BT;
            const int wk = tile_w(k);
            double *Fk = Fc + (int64_t)k * r4 * BT;
            // warp w owns the row tiles w, w + 8, .. of the super-tile (8 keys each, interleaved so that a
            // partial super-tile spreads over all four SM sub-partitions' DMMA pipes); its warp-local key
            // j (row tile j / 8, row j % 8) sits at super-tile offset koff(j)
            // (ILV = false, short slices: contiguous 64-key warp spans instead)
            constexpr int wsr = ILV ? 1 : MT, msr = ILV ? kCW : 1;  // row-tile index = w * wsr + mt * msr
            auto rto = [&](int mt) { return 8 * (w * wsr + mt * msr); };
            auto koff = [&](int j) { return rto(j >> 3) + (j & 7); };
            const bool wact = t0 + 8 * w * wsr < hi;
            double C[MT][NT][2];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) C[mt][nt][0] = C[mt][nt][1] = 0.0;
            if (wact) {
                KC kc[2][MT];  // double-buffered K chunks: chunk c + 1 is in flight while c feeds the MMAs
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int64_t key = t0 + rto(mt) + gid;
                    if (key < hi) kc[0][mt].load(Ku + key * D + tq * DQ);
                    else kc[0][mt].zero();
                }
#pragma unroll
                for (int t0c = 0; t0c < DQ; t0c += TC) {
                    const int cb = (t0c / TC) & 1;
                    if (t0c + TC < DQ) {
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const int64_t key = t0 + rto(mt) + gid;
                            if (key < hi) kc[cb ^ 1][mt].load(Ku + key * D + tq * DQ + t0c + TC);
                            else kc[cb ^ 1][mt].zero();
                        }
                    }
#pragma unroll
                    for (int tt = 0; tt < TC; ++tt) {
                        const int t = t0c + tt;
                        double bk[NT];
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) bk[nt] = kcB[((t * NT + nt) * 8 + gid) * 4 + tq];
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const double av = kc[cb][mt].elem(tt);
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) dmma(C[mt][nt][0], C[mt][nt][1], av, bk[nt]);
                        }
                    }
                }
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int sl = 8 * nt + 2 * tq + hh;
                        const double cz = c0r[sl];
                        if (sl < bsz) {  // every drawn candidate (acceptance is not known yet)
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt)
                                C[mt][nt][hh] = exp(__dadd_rn(__dmul_rn(g, C[mt][nt][hh] - cz), -mstar));
                        }
                    }
            }
            if (k == 0) WC_BTR(6);
            // F-prefix dots: rows 0..i-1 of this super-tile from the ring (one k-step per stage),
            // C -= F[.., tile]^T F[.., C] as C += A (-B): the 2 B values per stage are negated (sign bit),
            // not the 8 A values.  Rows [i, i4) of the last quad are zero in F (zero-filled after the
            // triangle) and in Fcol,
            // so no row predicate is needed.  The stage is released by the mbarrier arrive (release
            // semantics; every lane's loads have been consumed by its DMMAs before the __syncwarp).
            {
                int aoff[MT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) aoff[mt] = (rto(mt) + gid) * kBR + tq;
                const double *bcol = Fcol + (size_t)gid * ldc + tq;
                for (int j0 = 0; j0 < i; j0 += kBR) {
                    mbar_wait(&full[rstage], rph);
                    if (wact) {
                        const double *sb = ring + (size_t)rstage * STAGE;
                        double bf[NT];
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) bf[nt] = dneg(bcol[(size_t)nt * 8 * ldc + j0]);
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const double av = sb[aoff[mt]];
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) dmma(C[mt][nt][0], C[mt][nt][1], av, bf[nt]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[rstage]);
                    if (++rstage == NS) {
                        rstage = 0;
                        rph ^= 1u;
                    }
                }
            }
            if (k == 0) WC_BTR(7);
            cw_sync();  // every warp is done with the ring before it is reused as staging
            if (k == 0) {
                ce_sync();  // B: the rejection warp's na, Fx, perm, sA, rinvA are in shared memory
                na = sh_na;
                WC_BTR(4);
                WC_BTR(5);
            }
            int pm[NT * 2];  // acceptance index of this lane's C columns (slots 8 nt + 2 tq + hh), -1: rejected
#pragma unroll
            for (int z = 0; z < NT * 2; ++z) pm[z] = perm[8 * (z >> 1) + 2 * tq + (z & 1)];
            // per-key triangle over the accepted pivots in acceptance order: G is transposed through the
            // ring (idle until the next request) so that lane k owns keys 32 h + k of its warp with all
            // their G values at hand; left-looking:
            //   F[i+aa, l] = (G[l, aa] - sum_{a2<aa} F[i+a2, l] F[i+a2, s_aa]) / sqrt(p_{s_aa})
            // then the F row writes (coalesced), the downdate with the clamp (Z4), p_s <- 0, the L
            // entries of pivot keys, and the 32-key group sums.
            if (wact) {
                double plh[KPL];  // the residuals of the lane's keys, loaded before the staging
#pragma unroll
                for (int h = 0; h < KPL; ++h) {
                    const int64_t key = t0 + koff(32 * h + key_of_lane(lane));
                    plh[h] = key < hi ? __ldcg(cur + key) : 0.0;
                }
                // per key (lane, half h) after its triangle: residual, L rows of an accepted pivot, and
                // the sum of its row tile (8 lanes; the 32-key group sums follow once all warps are done)
                auto key_epilogue = [&](int h, const double (&f)[NSL], double pl) {
                    const int64_t key = t0 + koff(32 * h + key_of_lane(lane));
                    if (key < hi) {
                        nxt[key] = pl;
                        int xm = -1;  // acceptance index if this key is an accepted pivot (branch-free search)
#pragma unroll
                        for (int x = 0; x < NSL; ++x) xm = (x < na && sA[x] == key) ? x : xm;
                        if (xm >= 0) {  // L[i+x][i..i+x] = F[i..i+x, s_x]
                            double *Lr = a.L + ((int64_t)u * a.r + i + xm) * a.r + i;
#pragma unroll
                            for (int a2 = 0; a2 < NSL; ++a2)
                                if (a2 <= xm) Lr[a2] = f[a2];
                        }
                    }
                    double rs = key < hi ? pl : 0.0;  // one row tile: lanes m, m + 4, .., m + 28 (fixed butterfly)
#pragma unroll
                    for (int o = 4; o < 32; o <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
                    if (lane < 4) rts[w * wsr + (4 * h + lane) * msr] = rs;
                };
                // stage G rows (keys 8 mt + gid of the warp) for row tiles [mt0, mt0 + 4 KSN) at stg
                auto stage = [&](double *stg, int mt0, int nmt) {
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh) {
                                const int ai = pm[nt * 2 + hh];
                                if (ai >= 0 && mt >= mt0 && mt < mt0 + nmt)
                                    stg[srow_of(8 * (mt - mt0) + gid) * SP + ai] = C[mt][nt][hh];
                            }
                };
                if (KPL == 2 && two_keys) {
                    // both of the lane's keys staged at once, their triangles interleaved
                    double *stg = ring + (size_t)w * 64 * SP;
                    if (k == 0) WC_BTR(21);
                    stage(stg, 0, MT);
                    __syncwarp();
                    if (k == 0) WC_BTR(24);
                    const int64_t keys[2] = {t0 + koff(key_of_lane(lane)), t0 + koff(32 + key_of_lane(lane))};
                    double f[2][NSL];
                    double pl[2] = {plh[0], plh[KPL - 1]};
                    if constexpr (ILV) {
                        key_triangle_staged<NSL, 2>(stg, lane, Fx, rinvA, sA, na, keys, f, pl);
                        __syncwarp();
                        if (k == 0) WC_BTR(15);
                        write_f_rows<NSL, 8>(stg, lane, koff, t0, hi, Fk, wk, i, na);
                    } else {
                        double *const frows[2] = {Fk + (int64_t)koff(key_of_lane(lane)) * kBR,
                                                  Fk + (int64_t)koff(32 + key_of_lane(lane)) * kBR};
                        key_triangle_direct<NSL, 2>(stg, lane, Fx, rinvA, sA, na, keys, hi, frows, wk, i, f, pl);
                    }
                    if (k == 0) WC_BTR(22);
                    __syncwarp();
                    key_epilogue(0, f[0], pl[0]);
                    key_epilogue(1, f[1], pl[1]);
                    if (k == 0) WC_BTR(23);
                } else {
                    double *stg = ring + (size_t)w * 32 * SP;  // [32 keys][SP] per warp
#pragma unroll
                    for (int h = 0; h < KPL; ++h) {  // 32 keys of the warp at a time (row tiles 4h .. 4h + 3)
                        stage(stg, 4 * h, 4);
                        __syncwarp();
                        const int64_t keys[1] = {t0 + koff(32 * h + key_of_lane(lane))};
                        double f[1][NSL];
                        double pl[1] = {plh[h]};
                        if constexpr (ILV) {
                            key_triangle_staged<NSL, 1>(stg, lane, Fx, rinvA, sA, na, keys, f, pl);
                        } else {
                            double *const frows[1] = {Fk + (int64_t)koff(32 * h + key_of_lane(lane)) * kBR};
                            key_triangle_direct<NSL, 1>(stg, lane, Fx, rinvA, sA, na, keys, hi, frows, wk, i, f, pl);
                        }
                        __syncwarp();
                        if constexpr (ILV) {
                            write_f_rows<NSL, 4>(stg, lane, [&](int jl) { return koff(32 * h + jl); }, t0, hi, Fk, wk,
                                                 i, na);
                            __syncwarp();  // the staging of this half is consumed
                        }
                        key_epilogue(h, f[0], pl[0]);
                    }
                }
            } else if (lane < MT) {
                rts[w * wsr + lane * msr] = 0.0;  // row tiles past the slice
            }
            // the 32-key group sums (row tiles 4g .. 4g + 3, fixed order) and this CTA's running sum
            cw_sync();
            if (tid < BT / 32 && t0 + 32 * tid < hi) {
                const double gs = (rts[4 * tid] + rts[4 * tid + 1]) + (rts[4 * tid + 2] + rts[4 * tid + 3]);
                gnxt[t0 / 32 + tid] = gs;
                loc += gs;
            }
            fence_proxy_async_smem();  // the staging accesses to the ring precede the next bulk copies into it
            if (k + 1 < nst) {  // the ring (used as staging above) is free: stream the next super-tile
                cw_sync();
                if (tid == 0) flag_st64(&sh_req, ((long long)(++nreq) << 32) | ((long long)(k + 1) << 16) | (long long)i);
            }
        }
        if (nst == 0) {  // a CTA without keys still needs the accepted count
            ce_sync();
            na = sh_na;
        }
        WC_BTR(8);
        fence_proxy_async_global();  // this block's F rows are read by later TMA copies
        loc = cw_sum(loc, scr);
        if (tid == 0) pn[c] = loc;
        WC_BTR(9);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && blk < a.r) a.trace[blk * kTS + 13] = clock64();
        fread += (double)i;
        fdot += (double)i * (double)na;
        i += na;
        cbase += (uint32_t)bsz;
        ++blk;
        block_barrier(epoch++, cbase);
    }
    if (tid == 0) {
        flag_st(&sh_stop, 1);
        sh_cmd = 0;
    }
    ce_sync();  // A with the stop command: the rejection warp leaves its loop
    if (c == 0 && tid == 0) {
        a.r_eff[u] = i;
        st[5] = T0;
        st[6] = (double)blk;    // blocks run
        st[7] = (double)cbase;  // candidates drawn
        st[8] = fread;          // F rows re-read: sum over blocks of the block-start i
        st[9] = fdot;           // F-prefix dot work: sum over blocks of i * (pivots accepted)
    }
}

// Debug: per-block phase durations of CTA 0 (ns), printed per block.
void dump_block_trace(unsigned long long *dtrace, int r, cudaStream_t st) {
    std::vector<unsigned long long> h((size_t)kTS * r);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dtrace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(dtrace);
    // stamps in program order: 0 start, 1 candidates, 2 gather, 3 H, 6 kernel dots of super-tile 0
    // (the rejection runs meanwhile on the last compute warp), 7 F prefix, 4 na / Fx / perm,
    // 5 owners' L rows, 8 per-key triangle + writes, 9 sum, then the grid barrier (next block's 0)
    const int order[] = {1, 2, 3, 6, 7, 4, 5, 8, 9, 16};
    const char *names[] = {"cand", "gather", "H", "t0_kdot(+elim)", "t0_fdot", "na/Fx", "Lrows", "tiles", "sum",
                           "gbar"};
    for (int b = 0; b < r; ++b) {
        const unsigned long long *t = &h[(size_t)b * kTS];
        if (!t[0] || !t[9]) break;
        std::fprintf(stderr, "[btrace] block %3d:", b);
        unsigned long long last = t[0];
        for (int k = 0; k < 10; ++k) {
            const unsigned long long v = order[k] == 16 ? (b + 1 < r ? h[(size_t)(b + 1) * kTS] : 0) : t[order[k]];
            if (!v) continue;
            std::fprintf(stderr, " %s=%llu", names[k], v - last);
            last = v;
        }
        if (b == 0 && t[10] && t[11]) std::fprintf(stderr, " [1a=%llu cand0=%llu]", t[10] - t[0], t[11] - t[10]);
        if (t[14] > t[3]) std::fprintf(stderr, " [elim=%llu]", t[14] - t[3]);
        if (t[20] && t[16] && t[17] && t[18] && t[19])
            std::fprintf(stderr, " [poll=%llu L1=%llu L2=%llu L3=%llu gath=%llu]", t[20] - t[0], t[16] - t[20], t[17] - t[16],
                         t[18] - t[17], t[19] - t[18]);
        if (t[21] && t[22] && t[23])
            std::fprintf(stderr, " [pre=%llu stage=%llu tri=%llu wr=%llu epi=%llu gs=%llu]", t[21] - t[5], t[24] - t[21],
                         t[15] - t[24], t[22] - t[15], t[23] - t[22], t[8] - t[23]);
        if (t[13] > t[12] && t[9] > t[0]) std::fprintf(stderr, " MHz=%.0f", 1e3 * (double)(t[13] - t[12]) / (double)(t[9] - t[0]));
        std::fprintf(stderr, "\n");
    }
}

// Static shared memory of the kernel the plan allows for (ptxas reports 1152 bytes on sm_100a with
// nvcc 12.9; the launch re-checks against cudaFuncGetAttributes).
constexpr size_t kSmemStatic = 2048;

// Shared-memory plan of the kernel: NS ring stages (0 if r does not fit the plan); min_only: the
// smallest ring the per-key staging needs.
template <int D, int NSL> int blocked_stages(int r, int cpu, bool min_only = false) {
    using PL = BPlan<NSL>;
    const int ldc = ((r + 15) & ~15) + 4;
    const size_t stage_bytes = (size_t)PL::STAGE * sizeof(double);
    const size_t fixed = BSmem<D, NSL>(nullptr, 0, ldc, cpu).bytes + 64;
    // the per-key triangle stages G ([32 keys][NSL + 1] per compute warp) through the idle ring
    const size_t stg = (size_t)kCW * 32 * PL::SPITCH * sizeof(double);
    const int ns_min = (int)std::max<size_t>(3, (stg + stage_bytes - 1) / stage_bytes);
    constexpr size_t kSmemMax = 227 * 1024 - kSmemStatic;  // shared memory per CTA (sm_100) minus statics
    if (fixed + (size_t)ns_min * (stage_bytes + 16) > kSmemMax) return 0;
    if (min_only) return ns_min;
    return (int)std::min<size_t>(12, (kSmemMax - fixed) / (stage_bytes + 16));
}

template <typename T, int D, int NSL>
int launch_blocked_tdn(const Dims &Dm, const void *K, double *stats, SelectBufs b, uint64_t seed, uint64_t unit0,
                       int block, int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    using PL = BPlan<NSL>;
    BlkArgs a;
    a.K = K; a.stats = stats; a.nrm2 = b.nrm2; a.p = b.p; a.F = b.F; a.part = b.part; a.bar = b.bar;
    a.gsum = b.gsum;
    a.rej = b.rej;
    a.S = S; a.r_eff = r_eff; a.L = L; a.n = Dm.n; a.units = Dm.units(); a.r = Dm.r;
    a.bins = Dm.bins; a.nb = Dm.nb; a.unit_n = Dm.unit_n;
    a.cpu = select_ctas_per_unit(Dm); a.b = block; a.seed = seed; a.unit0 = unit0; a.trace = nullptr;
    const int ldc = ((Dm.r + 15) & ~15) + 4;
    int NS = blocked_stages<D, NSL>(Dm.r, a.cpu);
    if (NS == 0) return -2;  // r too large for this plan
    (void)sizeof(PL);
    auto kt = rpc_select_blocked_kernel<T, D, NSL, true>;
    if constexpr (NSL == 16) {  // slices of at most BT / 2 keys: contiguous warp spans (see ILV)
        const int kc = key_ctas(a.cpu);
        const int64_t chunk = ((ceil_div(Dm.n, (int64_t)kc) + 31) / 32) * 32;
        if (chunk <= PL::BT / 2) kt = rpc_select_blocked_kernel<T, D, NSL, false>;
    }
    // the plan reserves kSmemStatic bytes for the kernel's static shared memory: take any excess
    // (toolchain-dependent) out of the ring, down to the plan's minimum
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kt) != cudaSuccess) return -1;
    const size_t extra = fa.sharedSizeBytes > kSmemStatic ? fa.sharedSizeBytes - kSmemStatic : 0;
    const int drop = (int)((extra + PL::STAGE * sizeof(double) + 15) / (PL::STAGE * sizeof(double) + 16));
    if (drop > 0) {
        if (NS - drop < blocked_stages<D, NSL>(Dm.r, a.cpu, true)) return -2;
        NS -= drop;
    }
    const size_t smem = BSmem<D, NSL>(nullptr, NS, ldc, a.cpu).bytes + 64;
    static const bool tracing = std::getenv("WC_SELECT_TRACE") != nullptr;
    if (tracing && cudaMalloc(&a.trace, sizeof(unsigned long long) * kTS * Dm.r) == cudaSuccess)
        cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long) * kTS * Dm.r, st);
    if (cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
    if (cudaMemsetAsync(b.bar, 0, sizeof(unsigned) * a.units, st) != cudaSuccess) return -1;
    if (cudaMemsetAsync(b.part, 0, sizeof(double) * 2 * kMaxCpu * a.units, st) != cudaSuccess) return -1;
    if (a.cpu >= kRejMinCpu &&
        cudaMemset2DAsync(b.rej, kRejStride * sizeof(double), 0, sizeof(double), a.units, st) != cudaSuccess)
        return -1;  // the flags of the published rejection results
    const dim3 grid(a.units * a.cpu);
    if (a.cpu > 1) {
        // cooperative (co-resident CTAs for the grid barrier) + programmatic stream serialisation
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kBThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        if (cudaLaunchKernelEx(&cfg, kt, a, NS) != cudaSuccess) return -1;
    } else {
        launch_pdl(kt, grid, dim3(kBThreads), smem, st, a, NS);
    }
    if (a.trace) dump_block_trace(a.trace, Dm.r, st);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// b <= 16: 16 candidate slots (512-key super-tiles); 16 < b <= 32: 32 slots (256-key super-tiles),
// whose candidate columns must fit shared memory next to the ring (r up to ~300).
template <typename T, int D>
int launch_blocked_td(const Dims &Dm, const void *K, double *stats, SelectBufs b, uint64_t seed, uint64_t unit0,
                      int block, int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    if (block <= 16) return launch_blocked_tdn<T, D, 16>(Dm, K, stats, b, seed, unit0, block, S, r_eff, L, st);
    return launch_blocked_tdn<T, D, 32>(Dm, K, stats, b, seed, unit0, block, S, r_eff, L, st);
}

template <typename T>
int launch_blocked_t(const Dims &Dm, const void *K, double *stats, SelectBufs b, uint64_t seed, uint64_t unit0, int block,
                     int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    switch (Dm.d) {
        case 16: return launch_blocked_td<T, 16>(Dm, K, stats, b, seed, unit0, block, S, r_eff, L, st);
        case 32: return launch_blocked_td<T, 32>(Dm, K, stats, b, seed, unit0, block, S, r_eff, L, st);
        case 64: return launch_blocked_td<T, 64>(Dm, K, stats, b, seed, unit0, block, S, r_eff, L, st);
        case 128: return launch_blocked_td<T, 128>(Dm, K, stats, b, seed, unit0, block, S, r_eff, L, st);
    }
    return -1;
}

}  // namespace

int select_blocked_max_block() { return kBMax; }

bool select_blocked_plan_ok(const Dims &D, int block) {
    if (block < 2 || block > kBMax) return false;
    const int cpu = select_ctas_per_unit(D);
    const bool s16 = block <= 16;
    switch (D.d) {
        case 16: return (s16 ? blocked_stages<16, 16>(D.r, cpu) : blocked_stages<16, 32>(D.r, cpu)) > 0;
        case 32: return (s16 ? blocked_stages<32, 16>(D.r, cpu) : blocked_stages<32, 32>(D.r, cpu)) > 0;
        case 64: return (s16 ? blocked_stages<64, 16>(D.r, cpu) : blocked_stages<64, 32>(D.r, cpu)) > 0;
        case 128: return (s16 ? blocked_stages<128, 16>(D.r, cpu) : blocked_stages<128, 32>(D.r, cpu)) > 0;
    }
    return false;
}

int launch_select_blocked(const Dims &D, const void *K, double *stats, SelectBufs b, uint64_t seed, uint64_t unit0, int block,
                          int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    if (block < 2 || block > kBMax) return -1;
    if (D.dtype == 0) return launch_blocked_t<float>(D, K, stats, b, seed, unit0, block, S, r_eff, L, st);
    return launch_blocked_t<__nv_bfloat16>(D, K, stats, b, seed, unit0, block, S, r_eff, L, st);
}

}  // namespace wc
