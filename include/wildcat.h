/*
 * wildcat.h -- C ABI of libwildcat.so: WildCat weighted-coreset attention
 * (Schroeder & Mackey, arxiv 2602.10056) on NVIDIA B200 (sm_100a).
 *
 * Citations "P:<line>" refer to PAPER.md of the paper; "Z<k>" to the readings
 * listed in DESIGN.md (where the paper is silent or ambiguous).
 *
 * Problem (Alg 4): queries Q, keys K, values V, scale beta, rank r
 *   -> O^ = WtdAttn(Q, CompressKV(K, V, R_Q, beta, r)),
 * computed independently for every "unit" u = b*heads_kv + h (one (batch,
 * kv-head) pair).  Query head hq uses unit (b, hq / (heads_q/heads_kv)).
 *
 * Binning (shape.bins = B > 1; Alg 2; readings Z12, Z13, Z23 of DESIGN.md):
 * the keys of a unit are recentred with the unit's kbar, then split into B contiguous bins of
 * nb = floor(n/B) keys, the last bin also holding the n - B nb remainder (reading Z13); bin b gets
 * its own R_K^b, tau_b (Eq. 7 with its size n_b) and RPNys at rank rb = min(ceil(r/B), nb) with the
 * Philox stream of sub-unit u*B + b; the bin coresets are concatenated.  Sizes below use R = B*rb
 * (= r when B = 1).
 *
 * Layouts (row-major, contiguous, device memory unless stated):
 *   Q, O   [batch][heads_q ][m][d]   dtype
 *   K, V   [batch][heads_kv][n][d]   dtype
 *   S      int32  [units][R]         key index (0..n-1) of the i-th pivot, -1 past r_eff; with
 *                                    bins, the bins' valid pivots concatenated in bin order
 *   r_eff  int32  [units]            number of pivots actually drawn (<= R, Z3; sum over bins)
 *   L      double [units][B][rb][rb] lower-triangular Cholesky factor of h~(K_S,K_S) in pivot
 *                                    order, L[a][b] = F[b, S[a]] (b <= a), 0 elsewhere (Z6);
 *                                    one factor per bin (row/column index bin-local)
 *   stats  double [units][B][WC_STATS_STRIDE(d)] = tau, g, mstar, R_K, R_Q, T0, nblocks, ncand,
 *                                    Fread, Fdot, 0 (x6), kbar[d].  Selection bookkeeping: nblocks =
 *                                    blocks (sequential: rounds) run, ncand = candidates drawn,
 *                                    Fread = sum over blocks of the F rows re-read at the block
 *                                    start (sequential: sum_i i) -- the F traffic is 8 n Fread bytes;
 *                                    Fdot = sum over blocks of (rows re-read x pivots accepted)
 *   KS     dtype  [units][R][d]      coreset keys, uncentred (Alg 2 "K_S <- K_S + kbar"), rows
 *                                    in the order of S, zero past r_eff
 *   X      float  [units][R][d+1]    [V_S, w] = W [V, 1_n]  (Alg 2 "Compress values"); with
 *                                    bins W is block diagonal (each bin's weights over its keys)
 *   vmin, vmax dtype [units][d]      columnwise range of V (Alg 4)
 *
 * Conventions:
 *   - Every call is asynchronous on `stream` (a cudaStream_t); nothing synchronises
 *     the host.  Argument errors are returned before any launch and nothing is
 *     written; launch errors are reported via cudaGetLastError as WC_ECUDA.
 *   - The caller owns every buffer including the workspace `ws` (ws_bytes >=
 *     wc_workspace_bytes(shape, op)); the library allocates nothing.
 *   - Reentrant for distinct workspaces; no global mutable state.
 *   - NaN/Inf inputs give undefined outputs.
 */
#ifndef WILDCAT_H_
#define WILDCAT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WC_OK 0
#define WC_EINVAL -1        /* null pointer, bad enum, unknown flag, opts->block > WC_MAX_BLOCK */
#define WC_ESHAPE -2        /* r < 1, r > n, bins < 1 or > r, heads_q % heads_kv != 0, d not in {16,32,64,128}, m < 0 */
#define WC_EDTYPE -3        /* dtype not WC_F32 / WC_BF16 */
#define WC_EWORKSPACE -4    /* ws too small or misaligned (needs 256-byte alignment) */
#define WC_ECUDA -5         /* CUDA launch / runtime error */
#define WC_ENCCL -6         /* NCCL error (n-sharded path) */
#define WC_EUNSUPPORTED -7  /* valid request this build does not implement */
#define WC_ENONFINITE -8    /* WC_CHECK_FINITE: an input element is NaN or +-Inf (nothing else is launched) */

#define WC_F32 0
#define WC_BF16 1

#define WC_OP_SELECT 0
#define WC_OP_WEIGHTS 1
#define WC_OP_ATTEND 2
#define WC_OP_FORWARD 3
#define WC_OP_FORWARD_NSHARD 4  /* per-rank workspace of wildcat_forward_nshard (shape = local shard) */

/* flags (wc_opts.flags; any other bit -> WC_EINVAL) */
#define WC_NO_CLIP 1u       /* skip the clip of Alg 3 (reading Z15) */
#define WC_TAU_ONE 2u       /* temperature tau = 1 instead of Eq. 7: the selection / weights kernel is
                               then h(a,b) = exp(beta <a - kbar, b - kbar>) -- the untempered softmax kernel of
                               P:124-129 on (recentred) keys; every bin (Alg 2) likewise */
#define WC_NO_RECENTER 4u   /* skip "Recenter keys" (Alg 2): kbar = 0, R_K = max ||k_l|| (P:304 with
                               uncentred keys); attention itself is invariant to the recentring, the
                               kernel the selection and the Nystrom weights approximate is not.  The kernel
                               values h~ span [exp(-2 mstar), 1]; the A3 weights run their exponentials in
                               fp32, so keys whose offset makes 2 mstar > ~80 (what recentring prevents)
                               lose the small entries to underflow */
#define WC_CHECK_FINITE 8u  /* debug: before any other work, scan Q, K, V for NaN / Inf (SPEC's finite-input
                               rule); synchronises `stream` once and returns WC_ENONFINITE if one is found */
#define WC_FLAGS_ALL 15u

#define WC_STATS_HEAD 16
#define WC_STATS_STRIDE(d) (WC_STATS_HEAD + (d))

typedef struct wc_shape {
    int32_t batch;     /* >= 1 */
    int32_t heads_q;   /* >= 1, multiple of heads_kv */
    int32_t heads_kv;  /* >= 1 */
    int32_t d;         /* head dim: 16, 32, 64 or 128 */
    int32_t r;         /* coreset size, 1 <= r <= n ("rank r") */
    int32_t bins;      /* B of Alg 2: 1 <= B <= r (remainder keys join the last bin) */
    int32_t dtype;     /* WC_F32 or WC_BF16 (element type of Q, K, V, O, KS, vmin, vmax) */
    int32_t reserved;
    int64_t m;         /* queries per q-head, >= 0 */
    int64_t n;         /* keys per kv-head, >= 1 */
} wc_shape;

typedef struct wc_opts {
    double beta;       /* softmax scale; <= 0 selects 1/sqrt(d) (reading Z7) */
    double rq;         /* R_Q of Alg 2; < 0 (or NaN) computes max ||q|| over the unit's query group */
    uint64_t seed;     /* Philox4x32-10 key for the pivot draws (reading Z2) */
    uint32_t flags;    /* WC_NO_CLIP | WC_TAU_ONE | WC_NO_RECENTER | WC_CHECK_FINITE */
    uint32_t block;    /* pivot selection: 0 or 1 = sequential RPCholesky, Alg 1;
                          2..WC_MAX_BLOCK = blocked ("accelerated") RPCholesky with b = block
                          candidates per block (P:678 future work; reading Z22): same pivot LAW
                          as Alg 1, a different pivot sequence for a given seed.  b <= 16 runs the
                          16-slot plan (any r <= WC_MAX_R); 16 < b <= 32 the 32-slot plan, whose
                          candidate columns must fit shared memory (r up to ~300, else
                          WC_EUNSUPPORTED before any launch). */
    uint64_t unit_offset; /* global id of this call's unit 0 (PAR2): unit u of the call draws
                          the Philox stream of unit unit_offset + u (bin b: sub-unit (unit_offset+u)*B + b;
                          reading Z2, Z23), so a GPU that holds units [u0, u0 + U) of a larger batch and
                          passes unit_offset = u0 selects exactly the pivots of the one-GPU run on those
                          units ("ForPar"; north_star "partitioned ... by (batch, head)").  The
                          n-sharded forward uses it as the id of its single unit. */
} wc_opts;

#define WC_MAX_BLOCK 32

/* Largest coreset size per selection problem (r, or rb = ceil(r/B) per bin) for wildcat_select /
 * wildcat_weights / wildcat_forward / wildcat_compress_kv / wildcat_forward_nshard: the r x r solve
 * and the blocked selection are planned for at most this many pivots; larger -> WC_EUNSUPPORTED
 * (before any launch).  wildcat_attend itself streams any number of coreset rows (decode caches). */
#define WC_MAX_R 1024

/* Bytes of workspace the op needs for this shape (0 on invalid shape). */
size_t wc_workspace_bytes(const wc_shape *shape, int op);

/* Alg 2 lines "Recenter keys" .. RPNys + Alg 1:
 * per unit, recentre K, compute R_K, R_Q (from Q, or opts->rq if >= 0; Q may then be
 * NULL), tau (Eq. 7), and run r rounds of randomly pivoted Cholesky on
 * h~(a,b) = exp(beta/tau^2 <a-kbar, b-kbar> - mstar) with the Philox pivot stream
 * (opts->block >= 2: the blocked variant, see wc_opts.block).
 * Writes S, r_eff, L, stats.  Outputs S, r_eff, L, stats are required. */
int wildcat_select(const wc_shape *shape, const wc_opts *opts, const void *Q, const void *K,
                   int32_t *S, int32_t *r_eff, double *L, double *stats,
                   void *ws, size_t ws_bytes, void *stream);

/* Nystrom weights applied to [V, 1_n] (Alg 2 "Compress values"):
 * X = h~(K_S,K_S)^{-1} h~(K_S,K) [V, 1_n], via L from wildcat_select; gathers KS = K[S]
 * and the value range vmin/vmax of V.  Inputs S, r_eff, L, stats come from wildcat_select. */
int wildcat_weights(const wc_shape *shape, const wc_opts *opts, const void *K, const void *V,
                    const int32_t *S, const int32_t *r_eff, const double *L, const double *stats,
                    void *KS, float *X, void *vmin, void *vmax,
                    void *ws, size_t ws_bytes, void *stream);

/* Alg 3 WtdAttn: O = clip( diag(A^ w)^{-1} A^ V_S where A^ w > 0 else 0, vmin, vmax ),
 * A^ = exp(beta Q K_S^T) over the first r_eff coreset rows.  `m` of the shape is the
 * number of queries per q-head (e.g. 1 for decode; 0 < m <= 16 selects the split-cache decode kernel).
 * Workspace: wc_workspace_bytes(shape, WC_OP_ATTEND) -- the per-unit operand image of the tcgen05
 * path (bf16, d in {64, 128}) or the decode kernel's split partials; 0 (ws may be NULL) otherwise. */
int wildcat_attend(const wc_shape *shape, const wc_opts *opts, const void *Q, const void *KS,
                   const float *X, const int32_t *r_eff, const void *vmin, const void *vmax,
                   void *O, void *ws, size_t ws_bytes, void *stream);

/* Alg 4 WildCat = select + weights + attend.  S and r_eff may be NULL
 * (then kept in the workspace). */
int wildcat_forward(const wc_shape *shape, const wc_opts *opts, const void *Q, const void *K,
                    const void *V, void *O, int32_t *S, int32_t *r_eff,
                    void *ws, size_t ws_bytes, void *stream);

/* ---- KV-cache compression (prefill) and decode.
 * The E3 protocol retains the first and last tokens of the context exactly and
 * compresses the rest: per unit, the first keep_first and last keep_last of the n tokens are kept,
 * and the n_mid = n - keep_first - keep_last middle tokens go through CompressKV (Alg 2,
 * P:297-313) at rank shape->r with shape->bins bins (B <= r <= n_mid; the last bin takes the
 * remainder, Z13; recentring, R_K and tau over the middle only; R_Q from Q's m prompt rows per q-head,
 * or opts->rq >= 0, Q then nullable; Philox unit ids as wildcat_forward; opts->block as wildcat_select).
 * Reading Z24: the cache is the union of exact and compressed entries, so WtdAttn over it
 * adds the retained tokens' exact terms to the Nystrom estimate of the middle's unnormalised sums.
 * The cache is compact -- per row a key, a value and a weight, keys and values in the model dtype:
 *   KC  dtype [units][C][d]    rows: first keep_first tokens | last keep_last tokens | the middle's
 *                              r_eff coreset keys (Alg 2 order) | zero rows
 *   VC  dtype [units][C][d]    matching values: v_l for retained tokens, V_S (rounded to the dtype)
 *                              for coreset rows, zero after
 *   WC  float [units][C]       matching weights: 1 for retained tokens, w for coreset rows, 0 after
 *   c_eff int32 [units]        keep_first + keep_last + r_eff (valid rows of the cache)
 *   vmin, vmax dtype [units][d] range of ALL n values
 *   S   int32 [units][R]       global token index of each coreset row, -1 past r_eff (nullable)
 * C = wc_kv_capacity(shape, keep_first, keep_last) = keep_first + keep_last + R, with R = B*rb of
 * the middle (R = 0 when n_mid = 0; then nothing is compressed and r, bins are not checked).
 * Errors: WC_ESHAPE for keep_* < 0 or n_mid < 0 and the wildcat_select shape rules applied to the
 * middle. */
size_t wc_kv_capacity(const wc_shape *shape, int32_t keep_first, int32_t keep_last);       /* 0 if invalid */
size_t wc_kv_workspace_bytes(const wc_shape *shape, int32_t keep_first, int32_t keep_last); /* 0 if invalid */
int wildcat_compress_kv(const wc_shape *shape, const wc_opts *opts, int32_t keep_first, int32_t keep_last,
                        const void *Q, const void *K, const void *V, void *KC, void *VC, float *WC, int32_t *c_eff,
                        void *vmin, void *vmax, int32_t *S, void *ws, size_t ws_bytes, void *stream);

/* Decode over the compact cache: WtdAttn (Alg 3) of shape->m new queries per q-head
 * (Q, O [batch][heads_q][m][d]) against the cache rows, with shape->r = C and shape->bins = 1
 * (shape->n only has to be >= C).  m <= 16 runs the split-cache decode kernel (fp32 scores and sums);
 * larger m expands the rows to [V_S, w] in the workspace and runs the prefill attend. */
size_t wc_decode_workspace_bytes(const wc_shape *shape);  /* 0 if invalid */
int wildcat_decode(const wc_shape *shape, const wc_opts *opts, const void *Q, const void *KC, const void *VC,
                   const float *WC, const int32_t *c_eff, const void *vmin, const void *vmax, void *O, void *ws,
                   size_t ws_bytes, void *stream);

/* ---- Key-dimension sharding of one long sequence across GPUs.
 * One process per GPU.  Rank 0 gets a 128-byte NCCL unique id from wc_comm_unique_id and shares
 * it (e.g. torch.distributed.broadcast_object_list); every rank then calls wc_comm_init after
 * selecting its device.  NCCL (libnccl.so.2) is resolved at run time; WC_EUNSUPPORTED if absent. */
int wc_comm_unique_id(void *id128);
int wc_comm_init(void **comm, const void *id128, int world, int rank);
int wc_comm_destroy(void *comm);

/* Device-initiated transport for the same n-sharded forward: no NCCL call per
 * round.  Each rank allocates a mailbox of 2 x world x capacity doubles (+ flags) in its own HBM
 * (the library's only allocation besides the comm) and exports it with CUDA IPC:
 *   wc_p2p_comm_create(&comm, world, rank, capacity, handle64)  -> this rank's 64-byte IPC handle
 *   (the caller all-gathers the handles, e.g. torch.distributed.all_gather_object, in rank order)
 *   wc_p2p_comm_connect(comm, handles)                          -> maps every peer's mailbox
 * Every exchange of wildcat_forward_nshard (prologue reductions, the per-round residual totals and
 * pivot packet, Y~) is then one kernel that stores this rank's vector into slot `rank` of every
 * peer's mailbox over NVLink (peer stores, system-scope release of a per-slot epoch flag) and one
 * kernel that acquires the world flags of the local mailbox and reduces the slots in rank order
 * (deterministic and identical on every rank).  capacity >= r (d + 1) doubles (the Y~ exchange);
 * smaller -> WC_EUNSUPPORTED at the forward.  world <= 8; world = 1 needs no connect.  A peer that
 * never posts makes the waiting kernel trap after 20 s (WC_ECUDA) instead of hanging the GPU.
 * wc_comm_destroy releases either kind of communicator. */
int wc_p2p_comm_create(void **comm, int world, int rank, size_t capacity, void *handle64);
int wc_p2p_comm_connect(void *comm, const void *handles);

/* Alg 4 on one (batch, kv-head) unit whose n_global keys are split across the communicator's ranks:
 * this rank holds keys/values [n_offset, n_offset + shape->n) (shape->n = local count >= 1, shape->batch
 * = shape->heads_kv = 1) and shape->m local queries per q-head (any query shard).  The pivot sequence
 * is drawn from the global residual diagonal with the same Philox stream and inverse-CDF rule as
 * wildcat_forward, so in exact arithmetic it does not depend on the number of ranks.  Collectives
 * per round: allgather of per-rank residual totals, allreduce(sum) of the pivot packet; plus the
 * prologue reductions and one allreduce of Y~.  S (global key indices) and r_eff are replicated.
 * R_Q from the local queries is max-reduced across ranks unless opts->rq >= 0. */
int wildcat_forward_nshard(void *comm, const wc_shape *local, int64_t n_global, int64_t n_offset,
                           const wc_opts *opts, const void *Q, const void *K, const void *V, void *O,
                           int32_t *S, int32_t *r_eff, void *ws, size_t ws_bytes, void *stream);

/* Human-readable status. */
const char *wc_strerror(int status);

/* Number of kernel launches the last successful call on this thread enqueued
 * (instrumentation for bench.py's gpu_launches; thread-local). */
int wc_last_launch_count(void);

/* Stage timing instrumentation (thread-local; off by default).  When enabled, the
 * calls record CUDA events on their stream between stages:
 *   wildcat_forward: [prologue, select, weights, attend];  wildcat_select: [prologue, select];
 *   wildcat_weights: [vrange, weights];  wildcat_attend: [attend].
 * wc_timing_read waits for the last event and writes the stage durations in ms; it
 * returns the number of stages written (<= cap), or a negative status. */
int wc_timing_enable(int on);
int wc_timing_read(float *ms, int cap);

/* ABI version (major*100 + minor). */
int wc_version(void);  /* 201: compact KV cache (KC, VC, WC) and wildcat_decode; 200: wc_opts.unit_offset, flags */

#ifdef __cplusplus
}
#endif
#endif /* WILDCAT_H_ */
