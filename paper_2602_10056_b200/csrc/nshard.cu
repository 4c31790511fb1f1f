// nshard.cu -- key-dimension sharding of one long sequence across GPUs.
//
// Each rank holds a contiguous shard [n_off, n_off + n_local) of the keys/values (and any shard of
// the queries).  The method is unchanged: the pivot of round i is drawn from the GLOBAL residual
// diagonal with the same Philox uniform and inverse-CDF rule (Eq. 4; reading Z2), so in
// exact arithmetic the pivot sequence equals the single-GPU one for any number of ranks.
// Per round (host-enqueued, no host synchronisation; NCCL over NVLink / NVSwitch):
//   ns_local_total -> ncclAllGather(per-rank residual totals)
//   ns_pick        -> owner rank finds s in its shard, writes the pivot packet
//                     {s, p_s, k_s, F[0:i, s]} (non-owners write zeros)
//   ncclAllReduce(sum) of the packet (an exact broadcast whose root is only known on the device)
//   ns_update      -> every rank: kernel column, rank update and downdate of its own keys
// Prologue: allreduce of column sums (kbar), of max ||q||^2 / value range, then of max rk^2.
// Weights: per-rank partial Y~ over local keys, allreduce(sum) of Y~, replicated r x r solve.
// Attend: local queries against the replicated coreset.
//
// Transport: NCCL, or device-initiated peer-memory exchange ("p2p").  In p2p
// mode every rank owns a mailbox [2 parities][world slots][cap] doubles + flags [2][world] in its
// own HBM, CUDA-IPC-mapped into every peer; an exchange is one single-CTA kernel that stores the
// rank's vector straight into slot `rank` of every peer's mailbox (NVLink P2P stores), fences at
// system scope and releases a flag = epoch per peer, and one single-CTA kernel that acquires the
// world flags of its own mailbox and reduces the slots in rank order (sum / max / gather) -- the
// same result on every rank, with no host round trip and no NCCL call per round.  Epochs are
// host-counted per exchange (all ranks run the same sequence); the parity double buffer is enough
// because a rank can only post exchange e+1 after every rank has posted e, i.e. finished e-1.
// Spins are bounded (globaltimer, 20 s) and trap instead of hanging the GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/wildcat.h"
#include "common.cuh"
#include "kernels.h"

namespace wc {

namespace {

// ------------------------------------------------------------------ NCCL (resolved at run time)
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    bool ok = false;
};

const NcclApi &nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
        a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
        a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.ok = a.getUniqueId && a.commInitRank && a.allReduce && a.allGather && a.commDestroy;
        return a;
    }();
    return api;
}

constexpr int kP2PMaxWorld = 8;

struct PeerPtrs {
    double *mbox[kP2PMaxWorld];
    unsigned long long *flags[kP2PMaxWorld];
};

struct Comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    int p2p = 0;                          // 1: device-initiated peer-memory transport
    size_t cap = 0;                       // doubles per mailbox slot
    char *base = nullptr;                 // local mailbox allocation (cudaMalloc, IPC-exported)
    PeerPtrs peers{};                     // mapped mailboxes of every rank (own rank: local)
    char *opened[kP2PMaxWorld] = {};      // IPC-opened peer bases (to close)
    unsigned long long epoch = 0;         // exchanges issued
};

size_t p2p_bytes(int world, size_t cap) {
    return ((2 * (size_t)world * cap * sizeof(double) + 255) & ~size_t(255)) + 2 * (size_t)world * 8;
}
void p2p_set_peer(Comm *c, int q, char *b) {
    c->peers.mbox[q] = reinterpret_cast<double *>(b);
    c->peers.flags[q] = reinterpret_cast<unsigned long long *>(
        b + ((2 * (size_t)c->world * c->cap * sizeof(double) + 255) & ~size_t(255)));
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtime_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Store src[0:count] into slot `rank` (parity `par`) of every rank's mailbox, then release the flags.
__global__ void __launch_bounds__(256) p2p_post(PeerPtrs pp, int world, int rank, size_t cap, const double *src,
                                                int count, int par, unsigned long long epoch) {
    for (int q = 0; q < world; ++q) {
        double *dst = pp.mbox[q] + ((size_t)par * world + rank) * cap;
        for (int e = threadIdx.x; e < count; e += blockDim.x) dst[e] = src[e];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < world) st_release_sys(pp.flags[threadIdx.x] + (size_t)par * world + rank, epoch);
}

// Acquire the world flags of the local mailbox (parity `par`), then reduce the slots in rank order:
// op 0 = sum, 1 = max, 2 = gather (dst[q * count + e] = slot_q[e]).
__global__ void __launch_bounds__(256) p2p_reduce(const double *mbox, const unsigned long long *flags, int world,
                                                  size_t cap, int count, int par, unsigned long long epoch, int op,
                                                  double *dst) {
    if (threadIdx.x < world) {
        const unsigned long long *f = flags + (size_t)par * world + threadIdx.x;
        const unsigned long long t0 = gtime_ns();
        while (ld_acquire_sys(f) < epoch) {
            if (gtime_ns() - t0 > 20000000000ull) __trap();  // a peer never posted: fail, do not hang
            __nanosleep(200);
        }
    }
    __syncthreads();
    __threadfence_system();
    const double *slot = mbox + (size_t)par * world * cap;
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        if (op == 2) {
            for (int q = 0; q < world; ++q) dst[(size_t)q * count + e] = __ldcv(slot + (size_t)q * cap + e);
        } else {
            double v = __ldcv(slot + e);
            for (int q = 1; q < world; ++q) {
                const double x = __ldcv(slot + (size_t)q * cap + e);
                v = op == 0 ? v + x : fmax(v, x);
            }
            dst[e] = v;
        }
    }
}

constexpr int kNsChunk = 2048;  // keys per chunk (one CTA of ns_update, one chunk total)
constexpr int kNsT = 256;

struct Ctl {  // device-side loop state
    int done;
    int r_eff;
    double T0;
    double theta;
    int i;      // blocked selection: pivots accepted so far
    int na;     // pivots accepted by the current block
    uint32_t cbase;  // candidates drawn so far (Philox counters, reading Z22)
    int nblocks;
};

// Acceptance uniform of blocked-selection candidate `cand` (Philox tag 'ACPT', reading Z22).
__device__ __forceinline__ double accept_uniform_ns(uint64_t seed, uint32_t cand, uint64_t unit) {
    uint32_t c[4] = {cand, (uint32_t)unit, (uint32_t)(unit >> 32), 0x41435054u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double x = (double)(c[0] >> 5), y = (double)(c[1] >> 6);
    return (x * 67108864.0 + y) * (1.0 / 9007199254740992.0);
}

// Per-round exchanges fused into the round kernels (p2p transport): the producer kernel stores its
// vector into every peer's mailbox and releases the flags; the consumer kernel acquires them.
struct P2PRound {
    int on, world, rank;
    size_t cap;
    PeerPtrs pp;
    unsigned long long ep;  // epoch of this exchange (parity = ep & 1)
};
// all threads of the block: post src[0:count] (already written, visible after __syncthreads)
__device__ __forceinline__ void p2p_post_block(const P2PRound &a, const double *src, int count) {
    const int par = (int)(a.ep & 1);
    for (int q = 0; q < a.world; ++q) {
        double *dst = a.pp.mbox[q] + ((size_t)par * a.world + a.rank) * a.cap;
        for (int e = threadIdx.x; e < count; e += blockDim.x) dst[e] = src[e];
    }
    __threadfence_system();
    __syncthreads();
    if ((int)threadIdx.x < a.world) st_release_sys(a.pp.flags[threadIdx.x] + (size_t)par * a.world + a.rank, a.ep);
}
// all threads of the block: wait until every rank posted exchange a.ep into the local mailbox
__device__ __forceinline__ void p2p_wait_block(const P2PRound &a) {
    const int par = (int)(a.ep & 1);
    if ((int)threadIdx.x < a.world) {
        const unsigned long long *f = a.pp.flags[a.rank] + (size_t)par * a.world + threadIdx.x;
        const unsigned long long t0 = gtime_ns();
        while (ld_acquire_sys(f) < a.ep) {
            if (gtime_ns() - t0 > 20000000000ull) __trap();
            __nanosleep(100);
        }
    }
    __syncthreads();
    __threadfence_system();
}
// element e of the rank-ordered sum of the posted vectors (after p2p_wait_block)
__device__ __forceinline__ double p2p_sum(const P2PRound &a, int e) {
    const double *slot = a.pp.mbox[a.rank] + (size_t)(a.ep & 1) * a.world * a.cap;
    double v = __ldcv(slot + e);
    for (int q = 1; q < a.world; ++q) v += __ldcv(slot + (size_t)q * a.cap + e);
    return v;
}

// ------------------------------------------------------------------ prologue reductions
__global__ void ns_pro_reduce1(int d, int P, const double *colsum, const float *vmin, const float *vmax,
                               const double *rq2, double *sumbuf, double *maxbuf) {
    // sumbuf[d] = local column sums; maxbuf = [rq2, -vmin[d], vmax[d]]
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        double t = 0.0;
        float a = 3.0e38f, b = -3.0e38f;
        for (int p = 0; p < P; ++p) {
            t += colsum[(int64_t)p * d + j];
            a = fminf(a, vmin[(int64_t)p * d + j]);
            b = fmaxf(b, vmax[(int64_t)p * d + j]);
        }
        sumbuf[j] = t;
        maxbuf[1 + j] = -(double)a;
        maxbuf[1 + d + j] = (double)b;
    }
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int p = 0; p < P; ++p) m = fmax(m, rq2[p]);
        maxbuf[0] = m;
    }
}

template <typename T>
__global__ void ns_pro_final1(int64_t n_global, int d, const double *sumbuf, const double *maxbuf, double *stats,
                              T *vmin, T *vmax, int no_recenter) {
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        stats[kStatsHead + j] = no_recenter ? 0.0 : sumbuf[j] / (double)n_global;  // WC_NO_RECENTER: kbar = 0
        vmin[j] = from_f32<T>((float)(-maxbuf[1 + j]));
        vmax[j] = from_f32<T>((float)maxbuf[1 + d + j]);
    }
}

__global__ void ns_pro_reduce2(int P, const double *rk2, double *rkbuf) {
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int p = 0; p < P; ++p) m = fmax(m, rk2[p]);
        rkbuf[0] = m;
    }
}

// tau (Eq. 7 with the global n), g, mstar; then the loop state.
__global__ void ns_tau(int64_t n_global, int r, const double *rkbuf, const double *maxbuf, double rq_given,
                       double beta, double *stats, Ctl *ctl, int tau_one) {
    if (threadIdx.x != 0) return;
    const double rk = sqrt(rkbuf[0]);
    const double rq = rq_given >= 0.0 ? rq_given : sqrt(maxbuf[0]);
    double tau = 1.0;
    if (!tau_one && rq * rk > 0.0) {
        const double rho0 = sqrt(1.0 + exp(lambert_w0_dev(2.0 / (2.718281828459045 * 2.718281828459045)) + 2.0));
        const double b0 = log((double)n_global) / (beta * rq * rk) + 2.0;
        const double w = lambert_w0_dev(b0 / (2.0 * rho0));
        tau = sqrt((rk / rq) * b0 / (2.0 * w));
    }
    const double g = beta / (tau * tau);
    stats[0] = tau;
    stats[1] = g;
    stats[2] = g * rk * rk;
    stats[3] = rk;
    stats[4] = rq;
    stats[5] = 0.0;
    ctl->done = 0;
    ctl->r_eff = r;
    ctl->T0 = 0.0;
    ctl->theta = 0.0;
    ctl->i = 0;
    ctl->na = 0;
    ctl->cbase = 0;
    ctl->nblocks = 0;
}

// p_l <- h~(k_l, k_l) (Alg 1) and the chunk totals.
__global__ void __launch_bounds__(kNsT) ns_init(int64_t n, const double *nrm2, const double *stats, double *p,
                                                double *ctot) {
    __shared__ double scr[40];
    const double g = stats[1], mstar = stats[2];
    const int64_t c0 = (int64_t)blockIdx.x * kNsChunk, c1 = std::min<int64_t>(n, c0 + kNsChunk);
    double loc = 0.0;
    for (int64_t l = c0 + threadIdx.x; l < c1; l += kNsT) {
        const double v = exp(__dadd_rn(__dmul_rn(g, nrm2[l]), -mstar));
        p[l] = v;
        loc += v;
    }
    loc = block_sum(loc, scr);
    if (threadIdx.x == 0) ctot[blockIdx.x] = loc;
}

__global__ void ns_local_total(int nchunks, const double *ctot, const Ctl *ctl, double *sendtot, P2PRound px) {
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int c = 0; c < nchunks; ++c) t += ctot[c];
        sendtot[0] = ctl->done ? 0.0 : t;
    }
    __syncthreads();
    if (px.on) p2p_post_block(px, sendtot, 1);  // this rank's total -> slot `rank` of every mailbox
}

template <typename T, int D>
__device__ __forceinline__ void ns_pick_owner(int i, int64_t n, int64_t n_off, int nchunks, const double *ctot,
                                              const double *p, const T *K, const double *F, double *packet,
                                              double *scr, int &sh_c, int &sh_s, int &sh_last, double &sh_t,
                                              double &sh_t2);

// Global pivot draw; the owner rank writes the pivot packet {s, p_s, k_s[d], F[0:i, s]}.
template <typename T, int D>
__global__ void __launch_bounds__(kNsT) ns_pick(int i, int r, int world, int rank, int64_t n, int64_t n_off,
                                                int nchunks, uint64_t seed, uint64_t unit_id, const double *ranktot,
                                                const double *ctot, const double *p, const T *K, const double *F,
                                                double *packet, Ctl *ctl, P2PRound pw, P2PRound px) {
    __shared__ double scr[40];
    __shared__ int sh_owner, sh_c, sh_s, sh_last, sh_done;
    __shared__ double sh_t, sh_t2;
    const int tid = threadIdx.x;
    const int plen = 2 + D + r;
    if (pw.on) {  // the rank totals of this round, gathered from the local mailbox
        p2p_wait_block(pw);
        if (tid < world) const_cast<double *>(ranktot)[tid] =
            __ldcv(pw.pp.mbox[pw.rank] + ((size_t)(pw.ep & 1) * world + tid) * pw.cap);
    }
    for (int j = tid; j < plen; j += kNsT) packet[j] = 0.0;
    __syncthreads();
    if (tid == 0) {
        sh_done = ctl->done;
        sh_owner = -1;
        if (!sh_done) {
            double Tt = 0.0;
            for (int q = 0; q < world; ++q) Tt += ranktot[q];
            if (i == 0) {
                ctl->T0 = Tt;
                ctl->theta = 1000.0 * (double)r * 2.220446049250313e-16 * Tt;
            }
            if (Tt <= ctl->theta) {
                ctl->done = 1;
                ctl->r_eff = i;
                sh_done = 1;
            } else {
                const double t = pivot_uniform(seed, (uint32_t)i, unit_id) * Tt;
                double acc = 0.0, excl = 0.0, last_excl = 0.0;
                int ow = -1, last = -1;
                for (int q = 0; q < world; ++q) {
                    const double v = ranktot[q];
                    if (v > 0.0) { last = q; last_excl = acc; }
                    const double na = acc + v;
                    if (ow < 0 && na > t) { ow = q; excl = acc; }
                    acc = na;
                }
                if (ow < 0) { ow = last; excl = last_excl; }
                sh_owner = ow;
                sh_t = t - excl;
            }
        }
    }
    __syncthreads();
    if (!(sh_done || sh_owner != rank)) ns_pick_owner<T, D>(i, n, n_off, nchunks, ctot, p, K, F, packet, scr, sh_c,
                                                            sh_s, sh_last, sh_t, sh_t2);
    if (px.on) {  // every rank posts its packet (non-owners: zeros); consumers sum in rank order
        __syncthreads();
        p2p_post_block(px, packet, plen);
    }
}

// owner rank of ns_pick: chunk by the local chunk totals (fixed order), then key inside the chunk
template <typename T, int D>
__device__ __forceinline__ void ns_pick_owner(int i, int64_t n, int64_t n_off, int nchunks, const double *ctot,
                                              const double *p, const T *K, const double *F, double *packet,
                                              double *scr, int &sh_c, int &sh_s, int &sh_last, double &sh_t,
                                              double &sh_t2) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        double acc = 0.0, excl = 0.0, last_excl = 0.0;
        int cs = -1, last = -1;
        for (int c = 0; c < nchunks; ++c) {
            const double v = ctot[c];
            if (v > 0.0) { last = c; last_excl = acc; }
            const double na = acc + v;
            if (cs < 0 && na > sh_t) { cs = c; excl = acc; }
            acc = na;
        }
        if (cs < 0) { cs = last; excl = last_excl; }
        sh_c = cs;
        sh_t2 = sh_t - excl;
        sh_s = 0x7fffffff;
        sh_last = -1;
    }
    __syncthreads();
    const int64_t c0 = (int64_t)sh_c * kNsChunk, c1 = std::min<int64_t>(n, c0 + kNsChunk);
    const int64_t per = ceil_div(c1 - c0, kNsT);
    const int64_t b0 = c0 + (int64_t)tid * per, b1 = std::min<int64_t>(c1, b0 + per);
    double v = 0.0;
    for (int64_t l = b0; l < b1; ++l) v += p[l];
    double tot;
    double run = block_exclusive_scan(v, scr, &tot);
    int found = -1, lastpos = -1;
    for (int64_t l = b0; l < b1; ++l) {
        const double pl = p[l];
        if (pl > 0.0) lastpos = (int)l;
        run += pl;
        if (found < 0 && run > sh_t2) found = (int)l;
    }
    if (found >= 0) atomicMin(&sh_s, found);
    if (lastpos >= 0) atomicMax(&sh_last, lastpos);
    __syncthreads();
    const int s = sh_s != 0x7fffffff ? sh_s : sh_last;
    if (tid == 0) {
        packet[0] = (double)(n_off + s);
        packet[1] = p[s];
    }
    for (int j = tid; j < D; j += kNsT) packet[2 + j] = to_f64(K[(int64_t)s * D + j]);
    for (int j = tid; j < i; j += kNsT) packet[2 + D + j] = F[(int64_t)j * n + s];
}

// Kernel column, rank update and downdate of this rank's keys (one CTA of 512 threads per 2048-key
// chunk, processed as 8 super-tiles of 256 keys).  Phase A: the 16 warps split the rows j of
// F[0:i, tile] (each lane keeps 8 + 8 independent coalesced loads in flight); phase B: the fp64
// kernel dot, two threads per key; phase C: fixed-order combine, F[i, :], residual, chunk sum.
constexpr int kNuT = 512, kNuW = kNuT / 32, kNuST = 256, kNuTK = kNuST / 32;

template <typename T, int D>
__global__ void __launch_bounds__(kNuT) ns_update(int i, int r, int64_t n, int64_t n_off, const T *K,
                                                  const double *stats, const double *packet, double *F, double *p,
                                                  double *ctot, int32_t *S, double *L, T *KS, const Ctl *ctl,
                                                  P2PRound pw) {
    extern __shared__ double nsm[];
    double *kcs = nsm;               // [D]
    double *fs = kcs + D;            // [r]
    double *kb = fs + r;             // [D]
    double *red = kb + D;            // [kNuW][kNuST]
    double *kd = red + kNuW * kNuST;  // [2][kNuST]
    double *scr = kd + 2 * kNuST;    // [40]
    if (ctl->done) return;
    const int tid = threadIdx.x, lane = tid & 31, w = warp_index();
    const double g = stats[1], mstar = stats[2];
    // the pivot packet: the NCCL-reduced buffer, or (p2p) the rank-ordered sum of the posted packets
    if (pw.on) p2p_wait_block(pw);
    auto pk = [&](int e) { return pw.on ? p2p_sum(pw, e) : packet[e]; };
    const int64_t s_glob = (int64_t)pk(0);
    const double ps = pk(1);
    for (int j = tid; j < D; j += kNuT) {
        kb[j] = stats[kStatsHead + j];
        kcs[j] = __dadd_rn(pk(2 + j), -stats[kStatsHead + j]);
    }
    for (int j = tid; j < i; j += kNuT) fs[j] = pk(2 + D + j);
    __syncthreads();
    const double rs = sqrt(ps);
    if (blockIdx.x == 0) {  // replicated outputs: S, L row i (L[i][i] = sqrt(p_s) = F[i, s] exactly), K_S row i
        for (int j = tid; j < i; j += kNuT) L[(int64_t)i * r + j] = fs[j];
        for (int j = tid; j < D; j += kNuT) KS[(int64_t)i * D + j] = from_f32<T>((float)pk(2 + j));
        if (tid == 0) {
            S[i] = (int32_t)s_glob;
            L[(int64_t)i * r + i] = rs;
        }
    }
    const int64_t c0 = (int64_t)blockIdx.x * kNsChunk, c1 = std::min<int64_t>(n, c0 + kNsChunk);
    double loc = 0.0;
    for (int64_t k0 = c0; k0 < c1; k0 += kNuST) {
        {  // phase A
            double acc[kNuTK];
#pragma unroll
            for (int t = 0; t < kNuTK; ++t) acc[t] = 0.0;
            int j = w;
            for (; j + kNuW < i; j += 2 * kNuW) {
                const double *F0 = F + (int64_t)j * n + k0 + lane;
                const double *F1 = F0 + (int64_t)kNuW * n;
                double x0[kNuTK], x1[kNuTK];
#pragma unroll
                for (int t = 0; t < kNuTK; ++t) {
                    const bool ok = k0 + 32 * t + lane < c1;
                    x0[t] = ok ? __ldcg(F0 + 32 * t) : 0.0;
                    x1[t] = ok ? __ldcg(F1 + 32 * t) : 0.0;
                }
                const double f0 = fs[j], f1 = fs[j + kNuW];
#pragma unroll
                for (int t = 0; t < kNuTK; ++t) acc[t] = fma(x1[t], f1, fma(x0[t], f0, acc[t]));
            }
            if (j < i) {
                const double *F0 = F + (int64_t)j * n + k0 + lane;
                const double f0 = fs[j];
#pragma unroll
                for (int t = 0; t < kNuTK; ++t) {
                    const bool ok = k0 + 32 * t + lane < c1;
                    acc[t] = fma(ok ? __ldcg(F0 + 32 * t) : 0.0, f0, acc[t]);
                }
            }
#pragma unroll
            for (int t = 0; t < kNuTK; ++t) red[w * kNuST + 32 * t + lane] = acc[t];
        }
        {  // phase B: two threads per key, D/2 elements each
            const int kk = tid % kNuST, half = tid / kNuST;
            const int64_t l = k0 + kk;
            double dot = 0.0;
            if (l < c1) {
                constexpr int Dh = D / 2;
                for (int jj = 0; jj < Dh; jj += 8) {
                    double kv[8];
                    Vec8<T>::load(K + l * D + half * Dh + jj, kv);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        dot = fma(__dadd_rn(kv[q], -kb[half * Dh + jj + q]), kcs[half * Dh + jj + q], dot);
                }
            }
            kd[half * kNuST + kk] = dot;
        }
        __syncthreads();
        if (tid < kNuST) {  // phase C
            const int64_t l = k0 + tid;
            if (l < c1) {
                double acc = 0.0;
#pragma unroll
                for (int ww = 0; ww < kNuW; ++ww) acc += red[ww * kNuST + tid];
                const double dot = kd[tid] + kd[kNuST + tid];
                const double hval = exp(__dadd_rn(__dmul_rn(g, dot), -mstar));
                const double f = (hval - acc) / rs;
                F[(int64_t)i * n + l] = f;
                double q = __dadd_rn(p[l], -__dmul_rn(f, f));
                q = q > 0.0 ? q : 0.0;
                if (n_off + l == s_glob) q = 0.0;
                p[l] = q;
                loc += q;
            }
        }
        __syncthreads();
    }
    loc = block_sum(loc, scr);
    if (tid == 0) ctot[blockIdx.x] = loc;
}

// ------------------------------------------------------------------ blocked selection (reading Z22)
// Per block of b candidates (host loop; the exchanges are the same two as the sequential rounds):
//   ns_local_total -> allgather of the rank totals (block-start residual)
//   ns_blk_pick    -> every rank draws the b candidates from the GLOBAL residual (Philox counters
//                     cbase + j, Eq. 4 inverse CDF over the rank totals, then the owner's chunk
//                     totals and keys) and writes the packets of the candidates it owns
//                     {s, p_s, k_s, F[0:i, s]} (b slots, zeros elsewhere)
//   allreduce(sum) of the b packets
//   ns_blk_elim    -> every rank (one CTA, identical fp64 arithmetic): H = h~(K_C, K_C) - F_C^T F_C
//                     with H_jj = p[s_j], the rejection of Z22 in candidate order, the accepted
//                     pivots' triangle coefficients; replicated S, L rows, K_S rows
//   ns_blk_update  -> every rank: the na F-form rounds on its own keys, one key per thread: the F
//                     prefix F[0:i, l] read ONCE for all accepted pivots (the blocked saving), the
//                     kernel dots, the per-key triangle, downdate with the clamp, chunk totals
constexpr int kNsBMax = 16;

struct BlkState {  // per block, written by ns_blk_elim (device memory)
    int jA[kNsBMax];      // candidate slot of accepted pivot a
    double rinv[kNsBMax];  // 1 / sqrt(H_jj at acceptance)
    double Fx[kNsBMax][kNsBMax];  // Fx[a][a2] = F[i + a2, s_a], a2 < a
};

template <typename T, int D>
__global__ void __launch_bounds__(kNsT) ns_blk_pick(int r, int b, int world, int rank, int64_t n, int64_t n_off,
                                                    int nchunks, uint64_t seed, uint64_t unit_id,
                                                    const double *ranktot, const double *ctot, const double *p,
                                                    const T *K, const double *F, double *packets, Ctl *ctl) {
    __shared__ double scr[40];
    __shared__ int sh_owner, sh_c, sh_s, sh_last, sh_done;
    __shared__ double sh_t, sh_t2;
    const int tid = threadIdx.x;
    const int plen = 2 + D + r;
    for (int e = tid; e < b * plen; e += kNsT) packets[e] = 0.0;
    __syncthreads();
    if (tid == 0) {
        sh_done = ctl->done || ctl->i >= r;
        if (!sh_done) {
            double Tt = 0.0;
            for (int q = 0; q < world; ++q) Tt += ranktot[q];
            if (ctl->nblocks == 0) {
                ctl->T0 = Tt;
                ctl->theta = 1000.0 * (double)r * 2.220446049250313e-16 * Tt;
            }
            if (Tt <= ctl->theta) {  // exhausted (reading Z3), tested at block starts
                ctl->done = 1;
                ctl->r_eff = ctl->i;
                sh_done = 1;
            }
            sh_t2 = Tt;  // (the total, read below)
        }
    }
    __syncthreads();
    if (sh_done) return;
    const double Tt = sh_t2;
    const int i = ctl->i;
    const uint32_t cbase = ctl->cbase;
    for (int j = 0; j < b; ++j) {
        if (tid == 0) {
            const double t = pivot_uniform(seed, cbase + (uint32_t)j, unit_id) * Tt;
            double acc = 0.0, excl = 0.0, last_excl = 0.0;
            int ow = -1, last = -1;
            for (int q = 0; q < world; ++q) {
                const double v = ranktot[q];
                if (v > 0.0) { last = q; last_excl = acc; }
                const double na = acc + v;
                if (ow < 0 && na > t) { ow = q; excl = acc; }
                acc = na;
            }
            if (ow < 0) { ow = last; excl = last_excl; }
            sh_owner = ow;
            sh_t = t - excl;
        }
        __syncthreads();
        if (sh_owner == rank)
            ns_pick_owner<T, D>(i, n, n_off, nchunks, ctot, p, K, F, packets + (size_t)j * plen, scr, sh_c, sh_s,
                                sh_last, sh_t, sh_t2);
        __syncthreads();
    }
}

// One CTA: H from the packets, the rejection, the replicated outputs.
template <typename T, int D>
__global__ void __launch_bounds__(kNsT) ns_blk_elim(int r, int b, uint64_t seed, uint64_t unit_id,
                                                    const double *stats, const double *packets, BlkState *bs,
                                                    int32_t *S, double *L, T *KS, Ctl *ctl) {
    __shared__ double H[kNsBMax][kNsBMax + 1];
    __shared__ double Fc[kNsBMax][kNsBMax];  // Fc[a][e] = F[i + a, s_e] (candidate e, accepted a)
    __shared__ double kc[kNsBMax][D];        // centred candidate keys
    __shared__ int acc_j[kNsBMax];
    __shared__ int sh_na;
    const int tid = threadIdx.x;
    if (ctl->done || ctl->i >= r) return;
    const int i = ctl->i;
    const int plen = 2 + D + r;
    const double g = stats[1], mstar = stats[2];
    for (int e = tid; e < b * D; e += kNsT) {
        const int j = e / D, c = e % D;
        kc[j][c] = __dadd_rn(packets[(size_t)j * plen + 2 + c], -stats[kStatsHead + c]);
    }
    __syncthreads();
    // H[x][e] = h~(k_x, k_e) - sum_{q<i} F[q, s_x] F[q, s_e]  (x != e), H[x][x] = p[s_x]; each entry
    // by one thread in a fixed order (the (x, e) and (e, x) sums are the same sequence of products)
    for (int e2 = tid; e2 < b * b; e2 += kNsT) {
        const int x = e2 / b, e = e2 % b;
        double v;
        if (x == e) {
            v = packets[(size_t)x * plen + 1];
        } else {
            const int lo_ = x < e ? x : e, hi_ = x < e ? e : x;  // symmetric order of the products
            double dot = 0.0;
            for (int c = 0; c < D; ++c) dot = fma(kc[lo_][c], kc[hi_][c], dot);
            double fs = 0.0;
            const double *fa = packets + (size_t)lo_ * plen + 2 + D, *fb = packets + (size_t)hi_ * plen + 2 + D;
            for (int q = 0; q < i; ++q) fs = fma(fa[q], fb[q], fs);
            v = exp(__dadd_rn(__dmul_rn(g, dot), -mstar)) - fs;
        }
        H[x][e] = v;
    }
    __syncthreads();
    if (tid == 0) {  // the rejection of Z22, in candidate order
        const uint32_t cbase = ctl->cbase;
        int na = 0;
        for (int j = 0; j < b && i + na < r; ++j) {
            const int64_t sj = (int64_t)packets[(size_t)j * plen];
            bool dup = false;
            for (int a = 0; a < na; ++a) dup |= (int64_t)packets[(size_t)acc_j[a] * plen] == sj;
            const double pj = packets[(size_t)j * plen + 1];
            const double v = accept_uniform_ns(seed, cbase + (uint32_t)j, unit_id);
            const double hjj = H[j][j];
            if (!dup && __dmul_rn(v, pj) < hjj) {
                const double rinv = 1.0 / sqrt(hjj);
                for (int e = 0; e < b; ++e) Fc[na][e] = (e > j) ? H[j][e] * rinv : 0.0;
                for (int x = j + 1; x < b; ++x)
                    for (int e = j + 1; e < b; ++e) H[x][e] = fma(-(H[x][j] * rinv), H[j][e] * rinv, H[x][e]);
                acc_j[na] = j;
                bs->jA[na] = j;
                bs->rinv[na] = rinv;
                ++na;
            }
        }
        sh_na = na;
        ctl->na = na;
    }
    __syncthreads();
    const int na = sh_na;
    for (int e = tid; e < kNsBMax * kNsBMax; e += kNsT) {
        const int a = e / kNsBMax, a2 = e % kNsBMax;
        bs->Fx[a][a2] = (a < na && a2 < a) ? Fc[a2][acc_j[a]] : 0.0;
    }
    // replicated outputs of the accepted pivots: S, K_S rows, L rows (L[i+x][q] = F[q, s_x])
    for (int x = 0; x < na; ++x) {
        const int j = acc_j[x];
        const double *pk = packets + (size_t)j * plen;
        for (int q = tid; q < i; q += kNsT) L[(int64_t)(i + x) * r + q] = pk[2 + D + q];
        for (int a2 = tid; a2 <= x; a2 += kNsT)
            L[(int64_t)(i + x) * r + i + a2] = a2 < x ? Fc[a2][j] : 1.0 / bs->rinv[x];
        for (int c = tid; c < D; c += kNsT) KS[(int64_t)(i + x) * D + c] = from_f32<T>((float)pk[2 + c]);
        if (tid == 0) S[i + x] = (int32_t)(int64_t)pk[0];
    }
}

// One key per thread: the na F-form rounds of the block on this rank's keys (F row-major [r][n]).
template <typename T, int D>
__global__ void __launch_bounds__(256) ns_blk_update(int r, int b, int64_t n, int64_t n_off, const T *K,
                                                     const double *stats, const double *packets, const BlkState *bs,
                                                     double *F, double *p, double *subtot, const Ctl *ctl) {
    __shared__ double fs[kNsBMax][128];  // F[q0 .. q0+127, s_a] of the accepted pivots (a chunk of rows)
    __shared__ double kcs[kNsBMax][D];   // their centred keys
    __shared__ double kb[D];
    __shared__ double scr[40];
    __shared__ int64_t sg[kNsBMax];
    if (ctl->done || ctl->i >= r) return;  // (ctl->i is advanced after this kernel)
    const int i = ctl->i, na = ctl->na;
    const int plen = 2 + D + r;
    const int tid = threadIdx.x;
    const double g = stats[1], mstar = stats[2];
    for (int c = tid; c < D; c += 256) kb[c] = stats[kStatsHead + c];
    for (int e = tid; e < na * D; e += 256) {
        const int a = e / D, c = e % D;
        kcs[a][c] = __dadd_rn(packets[(size_t)bs->jA[a] * plen + 2 + c], -stats[kStatsHead + c]);
    }
    if (tid < na) sg[tid] = (int64_t)packets[(size_t)bs->jA[tid] * plen];
    const int64_t l = (int64_t)blockIdx.x * 256 + tid;
    const bool ok = l < n;
    double G[kNsBMax];
#pragma unroll
    for (int a = 0; a < kNsBMax; ++a) G[a] = 0.0;
    // F prefix: G[a] -= sum_q F[q, l] F[q, s_a], rows in chunks of 128 staged in shared memory
    for (int q0 = 0; q0 < i; q0 += 128) {
        __syncthreads();
        for (int e = tid; e < na * 128; e += 256) {
            const int a = e / 128, q = q0 + e % 128;
            fs[a][e % 128] = q < i ? packets[(size_t)bs->jA[a] * plen + 2 + D + q] : 0.0;
        }
        __syncthreads();
        const int qe = min(128, i - q0);
        for (int q = 0; q < qe; ++q) {
            const double f = ok ? __ldcg(F + (int64_t)(q0 + q) * n + l) : 0.0;
#pragma unroll
            for (int a = 0; a < kNsBMax; ++a)
                if (a < na) G[a] = fma(-f, fs[a][q], G[a]);
        }
    }
    __syncthreads();
    // kernel dots: h~(k_l, k_sa) = exp(g <k_l - kbar, k_sa - kbar> - mstar)
    double dot[kNsBMax];
#pragma unroll
    for (int a = 0; a < kNsBMax; ++a) dot[a] = 0.0;
    if (ok) {
        for (int c0 = 0; c0 < D; c0 += 8) {
            double kv[8];
            Vec8<T>::load(K + l * D + c0, kv);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double kc = __dadd_rn(kv[q], -kb[c0 + q]);
#pragma unroll
                for (int a = 0; a < kNsBMax; ++a)
                    if (a < na) dot[a] = fma(kc, kcs[a][c0 + q], dot[a]);
            }
        }
    }
    double pl = ok ? p[l] : 0.0;
    double f[kNsBMax];
#pragma unroll
    for (int a = 0; a < kNsBMax; ++a) {
        f[a] = 0.0;
        if (a < na) {
            double cv = exp(__dadd_rn(__dmul_rn(g, dot[a]), -mstar)) + G[a];
#pragma unroll
            for (int a2 = 0; a2 < a; ++a2) cv = fma(-f[a2], bs->Fx[a][a2], cv);
            const double fv = cv * bs->rinv[a];
            f[a] = fv;
            if (ok) F[(int64_t)(i + a) * n + l] = fv;
            const double qd = __dadd_rn(pl, -__dmul_rn(fv, fv));
            pl = (qd > 0.0 && n_off + l != sg[a]) ? qd : 0.0;
        }
    }
    if (ok) p[l] = pl;
    // chunk totals (kNsChunk = 8 x 256 keys): the 8 CTAs of a chunk add in fixed order below
    const double bsum = block_sum(ok ? pl : 0.0, scr);
    if (tid == 0) subtot[blockIdx.x] = bsum;  // per-256-key totals; ns_blk_advance folds them per chunk
}

// Fold the per-256-key totals of ns_blk_update into the per-chunk totals (fixed order) and advance
// the block state.  One thread per chunk; thread 0 also advances i / cbase.
__global__ void ns_blk_advance(int nchunks, int nsub, int b, const double *sub_tot, double *ctot, Ctl *ctl, int r) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = !(ctl->done || ctl->i >= r);
    if (live && c < nchunks) {
        double t = 0.0;
        for (int k = 0; k < kNsChunk / 256; ++k)
            if (c * (kNsChunk / 256) + k < nsub) t += sub_tot[c * (kNsChunk / 256) + k];
        ctot[c] = t;
    }
    if (c == 0 && live) {
        ctl->i += ctl->na;
        ctl->cbase += (uint32_t)b;
        ctl->nblocks += 1;
        if (ctl->i >= r) ctl->r_eff = ctl->i;
    }
}

__global__ void ns_finish(const Ctl *ctl, int32_t *r_eff_out, double *stats) {
    if (threadIdx.x == 0) {
        *r_eff_out = ctl->r_eff;
        stats[5] = ctl->T0;
    }
}

struct NsWs {
    ProloguePartials pp;
    double *stats, *nrm2, *p, *F, *ctot, *sendtot, *ranktot, *packet, *sumbuf, *maxbuf, *rkbuf, *L, *Yfull, *Dinv;
    double *packets, *subtot;  // blocked selection: b candidate packets, per-256-key residual totals
    BlkState *bs;
    float *Ypart, *X;
    void *KS, *vmin, *vmax, *aimg;
    int32_t *S, *reff;
    Ctl *ctl;
};

struct Carve {
    char *base;
    size_t off = 0;
    template <typename U> U *take(size_t count) {
        off = (off + 255) & ~size_t(255);
        U *q = base ? reinterpret_cast<U *>(base + off) : nullptr;
        off += count * sizeof(U);
        return q;
    }
};

size_t ns_carve(const Dims &D, void *base, NsWs &w) {
    Carve c{static_cast<char *>(base)};
    const int P = prologue_num_splits(D);
    const int64_t nch = ceil_div(D.n, kNsChunk);
    const size_t e = D.dtype == 0 ? 4 : 2;
    w.pp.P = P;
    w.pp.colsum = c.take<double>((size_t)P * D.d);
    w.pp.vmin = c.take<float>((size_t)P * D.d);
    w.pp.vmax = c.take<float>((size_t)P * D.d);
    w.pp.rq2 = c.take<double>(P);
    w.pp.rk2 = c.take<double>(P);
    w.stats = c.take<double>(kStatsHead + D.d);
    w.nrm2 = c.take<double>(D.n);
    w.p = c.take<double>(D.n);
    w.F = c.take<double>((size_t)D.r * D.n);
    w.ctot = c.take<double>(nch);
    w.sendtot = c.take<double>(1);
    w.ranktot = c.take<double>(kMaxCpu);
    w.packet = c.take<double>(2 + D.d + D.r);
    w.packets = c.take<double>((size_t)kNsBMax * (2 + D.d + D.r));
    w.subtot = c.take<double>(ceil_div(D.n, 256));
    w.bs = c.take<BlkState>(1);
    w.sumbuf = c.take<double>(D.d);
    w.maxbuf = c.take<double>(1 + 2 * D.d);
    w.rkbuf = c.take<double>(1);
    w.L = c.take<double>((size_t)D.r * D.r);
    const int splits = weights_num_splits(D);
    w.Ypart = c.take<float>((size_t)splits * D.r * (D.d + 1) + 2);
    w.Yfull = c.take<double>((size_t)D.r * (D.d + 1));
    w.Dinv = c.take<double>(dinv_elems(D.r));
    w.X = c.take<float>((size_t)D.r * (D.d + 1));
    w.KS = c.take<char>((size_t)D.r * D.d * e);
    w.vmin = c.take<char>((size_t)D.d * e);
    w.vmax = c.take<char>((size_t)D.d * e);
    w.S = c.take<int32_t>(D.r);
    w.reff = c.take<int32_t>(1);
    w.ctl = c.take<Ctl>(1);
    w.aimg = c.take<char>(attend_ws_bytes(D));
    return ((c.off + 255) & ~size_t(255)) + 256;
}

int nccl_status(ncclResult_t r) { return r == ncclSuccess ? WC_OK : WC_ENCCL; }

template <typename T, int D>
int ns_forward_t(Comm *cm, const Dims &Dm, int64_t n_global, int64_t n_off, const wc_opts *o, double beta,
                 double rq, const void *Q, const void *K, const void *V, void *O, int32_t *S_out, int32_t *reff_out,
                 NsWs &w, cudaStream_t st, int *launches_out) {
    const NcclApi &api = nccl();
    const int64_t n = Dm.n;
    const int nch = (int)ceil_div(n, kNsChunk);
    const int r = Dm.r;
    const bool want_q = rq < 0.0 && Dm.m > 0 && Q != nullptr;
    int launches = 0;
    // one collective on either transport: op 0 = sum, 1 = max, 2 = allgather of `count` per rank
    auto coll = [&](const double *src, double *dst, size_t count, int op) -> int {
        if (!cm->p2p) {
            if (op == 2) return nccl_status(api.allGather(src, dst, count, ncclFloat64, cm->comm, st));
            return nccl_status(api.allReduce(src, dst, count, ncclFloat64, op == 0 ? ncclSum : ncclMax, cm->comm, st));
        }
        if (count > cm->cap) return WC_EUNSUPPORTED;
        const unsigned long long ep = ++cm->epoch;
        const int par = (int)(ep & 1);
        p2p_post<<<1, 256, 0, st>>>(cm->peers, cm->world, cm->rank, cm->cap, src, (int)count, par, ep);
        p2p_reduce<<<1, 256, 0, st>>>(cm->peers.mbox[cm->rank], cm->peers.flags[cm->rank], cm->world, cm->cap,
                                      (int)count, par, ep, op, dst);
        launches += 2;
        return cudaPeekAtLastError() == cudaSuccess ? WC_OK : WC_ECUDA;
    };
#define WC_NCCL(x)                                  \
    do {                                            \
        const int rc_ = (x);                        \
        if (rc_) return rc_;                        \
    } while (0)
    // ---- A0 prologue with cross-rank reductions
    if (cudaMemsetAsync(w.S, 0xff, sizeof(int32_t) * r, st) != cudaSuccess) return WC_ECUDA;
    if (cudaMemsetAsync(w.L, 0, sizeof(double) * r * r, st) != cudaSuccess) return WC_ECUDA;
    if (launch_prologue_pass1(Dm, Q, K, V, want_q, w.pp, st) < 0) return WC_ECUDA;
    ns_pro_reduce1<<<1, 128, 0, st>>>(D, w.pp.P, w.pp.colsum, w.pp.vmin, w.pp.vmax, w.pp.rq2, w.sumbuf, w.maxbuf);
    WC_NCCL(coll(w.sumbuf, w.sumbuf, D, 0));
    WC_NCCL(coll(w.maxbuf, w.maxbuf, 1 + 2 * D, 1));
    ns_pro_final1<T><<<1, 128, 0, st>>>(n_global, D, w.sumbuf, w.maxbuf, w.stats, static_cast<T *>(w.vmin),
                                        static_cast<T *>(w.vmax), (o->flags & WC_NO_RECENTER) ? 1 : 0);
    if (launch_prologue_pass2(Dm, K, w.pp, w.stats, w.nrm2, st) < 0) return WC_ECUDA;
    ns_pro_reduce2<<<1, 32, 0, st>>>(w.pp.P, w.pp.rk2, w.rkbuf);
    WC_NCCL(coll(w.rkbuf, w.rkbuf, 1, 1));
    ns_tau<<<1, 32, 0, st>>>(n_global, r, w.rkbuf, w.maxbuf, want_q ? -1.0 : (rq < 0.0 ? 0.0 : rq), beta, w.stats,
                             w.ctl, (o->flags & WC_TAU_ONE) ? 1 : 0);
    ns_init<<<nch, kNsT, 0, st>>>(n, w.nrm2, w.stats, w.p, w.ctot);
    launches += 8;
    // ---- A1 + A2
    P2PRound off{};
    if (o->block >= 2) {
        // blocked selection (reading Z22): per block one exchange of the rank totals and one of the
        // b candidate packets (coll: NCCL, or the p2p post/reduce kernels).  Every block accepts at
        // least its first candidate, so the loop is launched for an estimate of the block count
        // (>= 50 % acceptance), then -- one host synchronisation -- continued while pivots remain.
        const int b = (int)o->block;
        const int plen = 2 + D + r;
        if (cm->p2p && (size_t)b * plen > cm->cap) return WC_EUNSUPPORTED;
        const int nsub = (int)ceil_div(n, 256);
        auto run_blocks = [&](int nblk) -> int {
            for (int k = 0; k < nblk; ++k) {
                ns_local_total<<<1, 32, 0, st>>>(nch, w.ctot, w.ctl, w.sendtot, off);
                WC_NCCL(coll(w.sendtot, w.ranktot, 1, 2));
                ns_blk_pick<T, D><<<1, kNsT, 0, st>>>(r, b, cm->world, cm->rank, n, n_off, nch, o->seed,
                                                       o->unit_offset, w.ranktot, w.ctot, w.p,
                                                       static_cast<const T *>(K), w.F, w.packets, w.ctl);
                WC_NCCL(coll(w.packets, w.packets, (size_t)b * plen, 0));
                ns_blk_elim<T, D><<<1, kNsT, 0, st>>>(r, b, o->seed, o->unit_offset, w.stats, w.packets, w.bs, w.S,
                                                       w.L, static_cast<T *>(w.KS), w.ctl);
                ns_blk_update<T, D><<<nsub, 256, 0, st>>>(r, b, n, n_off, static_cast<const T *>(K), w.stats,
                                                          w.packets, w.bs, w.F, w.p, w.subtot, w.ctl);
                ns_blk_advance<<<(nch + 255) / 256, 256, 0, st>>>(nch, nsub, b, w.subtot, w.ctot, w.ctl, r);
                launches += 6;
            }
            return WC_OK;
        };
        int planned = (r + b - 1) / b + 3;  // acceptance is ~90 % on the configs measured
        WC_NCCL(run_blocks(planned));
        while (planned < r + 1) {
            Ctl h{};
            if (cudaMemcpyAsync(&h, w.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st) != cudaSuccess) return WC_ECUDA;
            if (cudaStreamSynchronize(st) != cudaSuccess) return WC_ECUDA;
            if (h.done || h.i >= r) break;
            const int more = std::max(1, (r - h.i + b - 1) / b + 1);
            WC_NCCL(run_blocks(more));
            planned += more;
        }
    } else {
    // sequential Alg 1: r rounds
    const size_t usm = (size_t)(2 * D + r + kNuW * kNuST + 2 * kNuST + 40) * sizeof(double);
    auto upd = ns_update<T, D>;
    cudaFuncSetAttribute(upd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm);
    // p2p: the two per-round exchanges are fused into the round kernels (no extra launches)
    if (cm->p2p && (size_t)(2 + D + r) > cm->cap) return WC_EUNSUPPORTED;
    for (int i = 0; i < r; ++i) {
        P2PRound ptot = off, ppk = off;
        if (cm->p2p) {
            ptot = P2PRound{1, cm->world, cm->rank, cm->cap, cm->peers, ++cm->epoch};
            ppk = P2PRound{1, cm->world, cm->rank, cm->cap, cm->peers, ++cm->epoch};
        }
        ns_local_total<<<1, 32, 0, st>>>(nch, w.ctot, w.ctl, w.sendtot, ptot);
        if (!cm->p2p) WC_NCCL(coll(w.sendtot, w.ranktot, 1, 2));
        ns_pick<T, D><<<1, kNsT, 0, st>>>(i, r, cm->world, cm->rank, n, n_off, nch, o->seed, o->unit_offset, w.ranktot, w.ctot, w.p,
                                           static_cast<const T *>(K), w.F, w.packet, w.ctl, ptot, ppk);
        if (!cm->p2p) WC_NCCL(coll(w.packet, w.packet, 2 + D + r, 0));
        upd<<<nch, kNuT, usm, st>>>(i, r, n, n_off, static_cast<const T *>(K), w.stats, w.packet, w.F, w.p, w.ctot,
                                    w.S, w.L, static_cast<T *>(w.KS), w.ctl, ppk);
        launches += 3;
    }
    }
    ns_finish<<<1, 32, 0, st>>>(w.ctl, w.reff, w.stats);
    // ---- A3 + A4: local partial Y~, allreduce, replicated solve
    if (launch_weights_partial_ks(Dm, K, V, w.KS, w.reff, w.stats, w.Ypart, w.Yfull, st) < 0) return WC_ECUDA;
    WC_NCCL(coll(w.Yfull, w.Yfull, (size_t)r * (D + 1), 0));
    if (launch_weights_solve(Dm, w.Yfull, w.L, w.reff, w.X, w.Dinv, st) < 0) return WC_ECUDA;
    // ---- A5: local queries
    const int clip = (o->flags & WC_NO_CLIP) ? 0 : 1;
    if (Dm.m > 0 && launch_attend(Dm, Q, w.KS, w.X, w.reff, w.vmin, w.vmax, beta, clip, O, w.aimg, st) < 0) return WC_ECUDA;
    if (S_out && cudaMemcpyAsync(S_out, w.S, sizeof(int32_t) * r, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return WC_ECUDA;
    if (reff_out && cudaMemcpyAsync(reff_out, w.reff, sizeof(int32_t), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return WC_ECUDA;
    launches += 5;
#undef WC_NCCL
    *launches_out = launches;
    return cudaPeekAtLastError() == cudaSuccess ? WC_OK : WC_ECUDA;
}

}  // namespace

size_t ns_workspace_bytes(const Dims &D) {
    NsWs w;
    return ns_carve(D, nullptr, w);
}

int ns_forward(void *comm, const Dims &D, int64_t n_global, int64_t n_off, const wc_opts *o, double beta, double rq,
               const void *Q, const void *K, const void *V, void *O, int32_t *S, int32_t *reff, void *ws,
               cudaStream_t st, int *launches) {
    NsWs w;
    ns_carve(D, ws, w);
    Comm *cm = static_cast<Comm *>(comm);
#define WC_NSF(TT, DD) return ns_forward_t<TT, DD>(cm, D, n_global, n_off, o, beta, rq, Q, K, V, O, S, reff, w, st, launches)
    if (D.dtype == 0) {
        switch (D.d) { case 16: WC_NSF(float, 16); case 32: WC_NSF(float, 32); case 64: WC_NSF(float, 64); case 128: WC_NSF(float, 128); }
    } else {
        switch (D.d) { case 16: WC_NSF(__nv_bfloat16, 16); case 32: WC_NSF(__nv_bfloat16, 32); case 64: WC_NSF(__nv_bfloat16, 64); case 128: WC_NSF(__nv_bfloat16, 128); }
    }
#undef WC_NSF
    return WC_EINVAL;
}

int ns_comm_unique_id(void *id128) {
    const NcclApi &api = nccl();
    if (!api.ok) return WC_EUNSUPPORTED;
    ncclUniqueId id;
    if (api.getUniqueId(&id) != ncclSuccess) return WC_ENCCL;
    std::memcpy(id128, &id, sizeof(id));
    return WC_OK;
}

int ns_comm_init(void **out, const void *id128, int world, int rank) {
    const NcclApi &api = nccl();
    if (!api.ok) return WC_EUNSUPPORTED;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    Comm *c = new Comm;
    c->world = world;
    c->rank = rank;
    if (api.commInitRank(&c->comm, world, id, rank) != ncclSuccess) {
        delete c;
        return WC_ENCCL;
    }
    *out = c;
    return WC_OK;
}

int ns_p2p_create(void **out, int world, int rank, size_t cap, void *handle64) {
    if (world < 1 || world > kP2PMaxWorld || rank < 0 || rank >= world || cap < 1) return WC_EINVAL;
    Comm *c = new Comm;
    c->world = world;
    c->rank = rank;
    c->p2p = 1;
    c->cap = cap;
    const size_t bytes = p2p_bytes(world, cap);
    if (cudaMalloc(&c->base, bytes) != cudaSuccess || cudaMemset(c->base, 0, bytes) != cudaSuccess) {
        delete c;
        return WC_ECUDA;
    }
    p2p_set_peer(c, rank, c->base);
    std::memset(handle64, 0, 64);
    if (world > 1) {
        cudaIpcMemHandle_t h;
        static_assert(sizeof(h) == 64, "IPC handle size");
        if (cudaIpcGetMemHandle(&h, c->base) != cudaSuccess) {
            cudaFree(c->base);
            delete c;
            return WC_ECUDA;
        }
        std::memcpy(handle64, &h, 64);
    }
    *out = c;
    return WC_OK;
}

int ns_p2p_connect(void *comm, const void *handles) {
    Comm *c = static_cast<Comm *>(comm);
    if (!c || !c->p2p || !handles) return WC_EINVAL;
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char *>(handles) + 64 * (size_t)q, 64);
        void *ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return WC_ECUDA;
        c->opened[q] = static_cast<char *>(ptr);
        p2p_set_peer(c, q, c->opened[q]);
    }
    return WC_OK;
}

int ns_comm_destroy(void *comm) {
    if (!comm) return WC_OK;
    Comm *c = static_cast<Comm *>(comm);
    if (c->p2p) {
        cudaDeviceSynchronize();
        for (int q = 0; q < kP2PMaxWorld; ++q)
            if (c->opened[q]) cudaIpcCloseMemHandle(c->opened[q]);
        if (c->base) cudaFree(c->base);
    } else {
        const NcclApi &api = nccl();
        if (api.ok && c->comm) api.commDestroy(c->comm);
    }
    delete c;
    return WC_OK;
}

int ns_comm_world(void *comm) { return comm ? static_cast<Comm *>(comm)->world : 0; }

}  // namespace wc
