// kernels.h -- private host-side launchers of the WildCat sm_100a kernels (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace wc {

// Per-unit stats record: tau, g, mstar, R_K, R_Q, T0, nblocks, ncand, Fread, 0..., kbar[d]
// (WC_STATS_STRIDE(d) = kStatsHead + d in include/wildcat.h).
constexpr int kStatsHead = 16;
constexpr int kMaxR = 1024;  // largest r (or rb per bin) of a selection problem: the solve / blocked plans (WC_MAX_R)

struct Dims {
    int batch, hq, hkv, d, r, dtype;
    int64_t m, n;
    // Sub-unit geometry of Alg 2 binning (readings Z12, Z13): with bins > 1 a "unit" of these dims is
    // the sub-unit su = u * bins + b, whose keys are rows [b nb, b nb + count) of unit u's unit_n keys
    // (nb = floor(unit_n / bins); the last bin also holds the remainder); n is then the largest
    // sub-unit (the per-sub-unit buffer stride).  bins = 1: plain units of n keys.
    int bins = 1;
    int64_t nb = 0, unit_n = 0;
    int units() const { return batch * hkv; }
    int group() const { return hq / hkv; }
};

// Keys of sub-unit su (count) and the row of its first key in the unit-level K / V / nrm2 arrays.
struct SubUnit {
    int64_t count, base;
};
#ifdef __CUDACC__
__host__ __device__
#endif
inline SubUnit sub_unit(int su, int64_t n, int bins, int64_t nb, int64_t unit_n) {
    if (bins <= 1) return SubUnit{n, (int64_t)su * n};
    const int b = su % bins;
    return SubUnit{b == bins - 1 ? unit_n - (int64_t)(bins - 1) * nb : nb, (int64_t)(su / bins) * unit_n + (int64_t)b * nb};
}

// Workspace blocks used by the prologue (A0).
struct ProloguePartials {
    double *colsum;  // [units][P][d]
    float *vmin;     // [units][P][d]
    float *vmax;     // [units][P][d]
    double *rq2;     // [units][P]
    double *rk2;     // [units][P]
    int P;
    // optional output initialisation folded into pass 1 (instead of two memsets): S <- -1, L <- 0
    int32_t *fill_S = nullptr;
    int64_t nS = 0;
    double *zero_L = nullptr;
    int64_t nL = 0;
};

int prologue_num_splits(const Dims &D);

// Prologue options (wc_opts.flags): kPfTauOne -> tau = 1 (WC_TAU_ONE); kPfNoRecenter -> kbar = 0 (WC_NO_RECENTER).
constexpr int kPfTauOne = 1;
// WC_CHECK_FINITE: *flag |= 1 if x[0, count) (dtype 0 fp32, 1 bf16) holds a NaN / Inf.  Returns launches or -1.
int launch_check_finite(const void *x, int64_t count, int dtype, int *flag, cudaStream_t st);
constexpr int kPfNoRecenter = 2;

// A0: kbar, R_K, R_Q, tau, g, mstar -> stats[u][kStatsHead+d]; nrm2[u][l] = ||k_l - kbar||^2;
// vmin/vmax (dtype) when non-null.  Returns number of launches (>0) or -1 on error.
int launch_prologue(const Dims &D, const void *Q, const void *K, const void *V, double rq, double beta,
                    ProloguePartials pp, double *stats, double *nrm2, void *vmin, void *vmax, int pflags,
                    cudaStream_t st);

// The two streaming passes of the prologue on their own (the n-sharded path reduces across GPUs
// between them): pass 1 -> per-split column sums / V range / max ||q||^2; pass 2 -> nrm2, max rk^2.
int launch_prologue_pass1(const Dims &D, const void *Q, const void *K, const void *V, bool want_q,
                          ProloguePartials pp, cudaStream_t st);
int launch_prologue_pass2(const Dims &D, const void *K, ProloguePartials pp, const double *stats, double *nrm2,
                          cudaStream_t st);

// Columnwise range of V only (wildcat_weights).
int launch_vrange(const Dims &D, const void *V, ProloguePartials pp, void *vmin, void *vmax, cudaStream_t st);

struct SelectBufs {
    double *nrm2;   // [units][n]
    double *p;      // [2][units][n]
    double *F;      // [units][r][f_ld(n)]
    double *part;   // [units][2][kMaxCpu]
    unsigned *bar;  // [units]
    double *gsum;   // [units][2][ceil(n/32)] residual sums of 32-key groups (blocked selection)
    double *rej = nullptr;  // [units][kRejStride] the rejection CTA's published block result (blocked selection)
};
// Blocked selection with >= kRejMinCpu CTAs per unit: the last CTA owns no keys and runs the block
// rejection for the unit (its fp64 pipe free of the round-update DMMAs), publishing the result.
constexpr int kRejMinCpu = 32;
constexpr int kRejStride = 1280;
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int key_ctas(int cpu) { return cpu >= kRejMinCpu ? cpu - 1 : cpu; }
constexpr int kMaxCpu = 1024;
inline int64_t f_ld(int64_t n) { return (n + 31) / 32 * 32; }  // row stride of F (row-major kernel)
// Tile-major F of the TMA kernel: per unit [cpu][nst][r][256] doubles, nst = 256-key super-tiles per slice.
inline int f_tile_nst(int64_t n, int cpu) {
    const int64_t chunk = ((n + cpu - 1) / cpu + 31) / 32 * 32;
    return (int)((chunk + 255) / 256);
}
int select_ctas_per_unit(const struct Dims &D);
inline size_t f_elems_per_unit(int64_t n, int r, int cpu) {
    const size_t rowmajor = (size_t)r * f_ld(n);
    const int kc = key_ctas(cpu);  // (the sequential kernel's ceil(n / cpu) slices fit as well)
    const int64_t chunk = ((n + kc - 1) / kc + 31) / 32 * 32;
    // TMA kernels: [cpu][r4 x chunk] (the blocked kernel stores rows in quads: r rounded up to 4)
    const size_t tiles = (size_t)cpu * chunk * (size_t)((r + 3) & ~3);
    return rowmajor > tiles ? rowmajor : tiles;
}

int select_ctas_per_unit(const Dims &D);
// A1+A2: r rounds of RP-Cholesky.  Returns launches or -1.
// unit0: Philox id of the call's sub-unit 0 (wc_opts.unit_offset, times B with bins).
int launch_select(const Dims &D, const void *K, const double *stats, SelectBufs b, uint64_t seed, uint64_t unit0,
                  int32_t *S, int32_t *r_eff, double *L, cudaStream_t st);

// Blocked (accelerated) RPC, 2 <= block <= select_blocked_max_block().  Returns launches, -1 on a
// CUDA error, -2 when r does not fit the shared-memory plan.  stats[u][6..8] <- nblocks, ncand, Fread.
int launch_select_blocked(const Dims &D, const void *K, double *stats, SelectBufs b, uint64_t seed, uint64_t unit0,
                          int block, int32_t *S, int32_t *r_eff, double *L, cudaStream_t st);
int select_blocked_max_block();
// Whether the blocked kernel's shared-memory plan holds this r at this block size (host check, no launch).
bool select_blocked_plan_ok(const Dims &D, int block);

// Alg 2 binning (bins.cu): per-bin stats, pack (sub-unit -> unit layout), unpack (S only).
int launch_bins_stats(const Dims &D, int bins, double beta, const double *stats_u, const double *nrm2, double *stats_b,
                      int pflags, cudaStream_t st);
int launch_bins_pack(const Dims &D, int bins, int rb, const int32_t *Ssub, const int32_t *reff_sub, const void *KSsub,
                     const float *Xsub, int32_t *S, int32_t *reff, void *KS, float *X, cudaStream_t st);
int launch_bins_unpack(const Dims &D, int bins, int rb, const int32_t *S, int32_t *Ssub, int32_t *reff_sub,
                       cudaStream_t st);

int weights_num_splits(const Dims &D);
// A3+A4: X = L^{-T} L^{-1} h~(K_S,K)[V,1]; KS gather.  Ypart: [units][splits][r][d+1] fp32.
int launch_weights(const Dims &D, const void *K, const void *V, const int32_t *S, const int32_t *r_eff,
                   const double *L, const double *stats, float *Ypart, void *KS, float *X, cudaStream_t st);
// n-sharded variant, phase 1: fp64 partial Y~ over the local keys with the coreset rows given
// densely (KSin [units][r][d], dtype); Yfull receives the reduced local sum [units][r][d+1].
int launch_weights_partial_ks(const Dims &D, const void *K, const void *V, const void *KSin, const int32_t *r_eff,
                              const double *stats, float *Ypart, double *Yfull, cudaStream_t st);
// phase 2 (after the cross-GPU sum of Yfull): X = L^{-T} L^{-1} Y~.  Dinv: scratch of
// units * dinv_elems(r) doubles for the inverted 32 x 32 diagonal blocks of L.
int launch_weights_solve(const Dims &D, const double *Yfull, const double *L, const int32_t *r_eff, float *X,
                         double *Dinv, cudaStream_t st);
inline size_t dinv_elems(int r) { return (size_t)((r + 31) / 32) * 32 * 32; }
// Scratch of the inverse-based solve per unit (doubles): W = L^{-1} (R x R, R = 32 * 2^k >= r), the level
// products (R x R / 4) and W Y~ (R x (d + 1)).
inline size_t solve_scratch_elems(int r, int d) {
    size_t R = 32;
    while ((int)R < r) R *= 2;
    return R * R + R * R / 4 + R * (size_t)(d + 1);
}

// A5: attend.
int launch_attend(const Dims &D, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                  const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws, cudaStream_t st);
size_t attend_ws_bytes(const Dims &D);  // staging images for r > 256, decode partials (0 otherwise)

// Decode-shaped A5 (kvcache.cu), used by launch_attend when 0 < m <= kDecodeMaxM.
constexpr int kDecodeMaxM = 16;
size_t attend_decode_ws_bytes(const Dims &D);
int launch_attend_decode(const Dims &D, const void *Q, const void *KS, const float *X, const int32_t *r_eff,
                         const void *vmin, const void *vmax, double beta, int clip, void *O, void *ws,
                         cudaStream_t st);
// KV-cache assembly (reading Z24): KC / XC rows [first kf | last kl | middle coreset], c_eff, S (global).
// D: the full-context unit dims (n = all tokens).  Smid / reff_mid / KS / X of the middle may be null
// when R = 0.
int launch_kv_assemble(const Dims &D, const void *K, const void *V, int kf, int kl, int R, const void *KS,
                       const float *X, const int32_t *Smid, const int32_t *reff_mid, void *KC, void *VC, float *WC,
                       int32_t *c_eff, int32_t *S_out, cudaStream_t st);
// Decode over a compact KV cache (KC, VC dtype [units][C][d]; WC fp32 [units][C]): D.r = C, D.m <= kDecodeMaxM.
int launch_attend_decode_vw(const Dims &D, const void *Q, const void *KC, const void *VC, const float *WC,
                            const int32_t *c_eff, const void *vmin, const void *vmax, double beta, int clip, void *O,
                            void *ws, cudaStream_t st);
// (VC, WC) -> X fp32 rows [units * C][d + 1] (general attend over a compact cache).
int launch_vw_to_x(const Dims &D, const void *VC, const float *WC, float *X, cudaStream_t st);

// n-sharded forward (nshard.cu).  Single unit per call; NCCL resolved at run time.
size_t ns_workspace_bytes(const Dims &D);
int ns_forward(void *comm, const Dims &D, int64_t n_global, int64_t n_off, const struct wc_opts *o, double beta,
               double rq, const void *Q, const void *K, const void *V, void *O, int32_t *S, int32_t *reff, void *ws,
               cudaStream_t st, int *launches);
int ns_comm_unique_id(void *id128);
int ns_comm_init(void **out, const void *id128, int world, int rank);
int ns_comm_destroy(void *comm);
int ns_p2p_create(void **out, int world, int rank, size_t cap, void *handle64);
int ns_p2p_connect(void *comm, const void *handles);
int ns_comm_world(void *comm);

}  // namespace wc
