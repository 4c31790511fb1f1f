// api.cu -- the C ABI of libwildcat.so (declared in include/wildcat.h).
// Argument validation, workspace carving and kernel sequencing only; every arithmetic step
// of the method runs in the sm_100a kernels of prologue.cu / select.cu / weights.cu / attend.cu.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/wildcat.h"
#include "kernels.h"

static_assert(WC_STATS_HEAD == wc::kStatsHead, "stats layout of include/wildcat.h and the kernels differ");

namespace {

thread_local int g_launches = 0;

// ---- stage timing instrumentation (wc_timing_enable / wc_timing_read)
constexpr int kMaxEv = 8;
thread_local bool g_timing = false;
thread_local cudaEvent_t g_ev[kMaxEv] = {};
thread_local int g_nev = 0;

// WC_DEBUG_SYNC=1: synchronise after every stage and report the first CUDA error (debug only).
void tmark(cudaStream_t st, bool first = false) {
    static const bool dbg = std::getenv("WC_DEBUG_SYNC") != nullptr;
    if (dbg) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) std::fprintf(stderr, "[wildcat] stage %d: %s\n", first ? 0 : g_nev, cudaGetErrorString(e));
    }
    if (!g_timing) return;
    if (first) g_nev = 0;
    if (g_nev >= kMaxEv) return;
    if (!g_ev[g_nev]) cudaEventCreate(&g_ev[g_nev]);
    cudaEventRecord(g_ev[g_nev], st);
    ++g_nev;
}

struct Carver {
    char *base;
    size_t off = 0;
    explicit Carver(void *b) : base(static_cast<char *>(b)) {}
    template <typename T> T *take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

int check_shape(const wc_shape *s) {
    if (!s) return WC_EINVAL;
    if (s->dtype != WC_F32 && s->dtype != WC_BF16) return WC_EDTYPE;
    if (s->batch < 1 || s->heads_q < 1 || s->heads_kv < 1 || s->heads_q % s->heads_kv) return WC_ESHAPE;
    if (!(s->d == 16 || s->d == 32 || s->d == 64 || s->d == 128)) return WC_ESHAPE;
    if (s->n < 1 || s->n > (int64_t)0x7fffffff || s->m < 0 || s->r < 1 || s->r > s->n) return WC_ESHAPE;
    if (s->bins != 1) return WC_EUNSUPPORTED;
    return WC_OK;
}

wc::Dims dims_of(const wc_shape *s) {
    wc::Dims D;
    D.batch = s->batch; D.hq = s->heads_q; D.hkv = s->heads_kv; D.d = s->d; D.r = s->r; D.dtype = s->dtype;
    D.m = s->m; D.n = s->n;
    return D;
}

size_t esize(const wc_shape *s) { return s->dtype == WC_F32 ? 4 : 2; }

double beta_of(const wc_shape *s, const wc_opts *o) {
    return (o && o->beta > 0.0) ? o->beta : 1.0 / std::sqrt((double)s->d);
}
double rq_of(const wc_opts *o) {
    if (!o || std::isnan(o->rq) || o->rq < 0.0) return -1.0;
    return o->rq;
}

// Selection dispatch: sequential Alg 1, or the blocked variant when opts->block >= 2.
int run_select(const wc::Dims &D, const wc_opts *o, const void *K, double *stats, wc::SelectBufs sb, int32_t *S,
               int32_t *r_eff, double *L, cudaStream_t st) {
    if (o->block >= 2) {
        const int k = wc::launch_select_blocked(D, K, stats, sb, o->seed, (int)o->block, S, r_eff, L, st);
        return k == -2 ? WC_EUNSUPPORTED : (k < 0 ? WC_ECUDA : k);
    }
    const int k = wc::launch_select(D, K, stats, sb, o->seed, S, r_eff, L, st);
    return k < 0 ? WC_ECUDA : k;
}

int check_opts(const wc_opts *o, const wc_shape *s) {
    if (!o) return WC_EINVAL;
    if (o->block > (uint32_t)WC_MAX_BLOCK) return WC_EINVAL;
    if (o->block >= 2 && s->r > 1024) return WC_EUNSUPPORTED;
    return WC_OK;
}

struct SelectWs {
    wc::ProloguePartials pp;
    wc::SelectBufs sb;
};

void carve_select(Carver &c, const wc_shape *s, SelectWs &w) {
    const wc::Dims D = dims_of(s);
    const size_t U = D.units();
    const int P = wc::prologue_num_splits(D);
    w.pp.P = P;
    w.pp.colsum = c.take<double>(U * P * D.d);
    w.pp.vmin = c.take<float>(U * P * D.d);
    w.pp.vmax = c.take<float>(U * P * D.d);
    w.pp.rq2 = c.take<double>(U * P);
    w.pp.rk2 = c.take<double>(U * P);
    w.sb.nrm2 = c.take<double>(U * D.n);
    w.sb.p = c.take<double>(2 * U * D.n);
    w.sb.F = c.take<double>(U * wc::f_elems_per_unit(D.n, D.r, wc::select_ctas_per_unit(D)));
    w.sb.part = c.take<double>(U * 2 * wc::kMaxCpu);
    w.sb.bar = c.take<unsigned>(U);
    w.sb.gsum = c.take<double>(U * 2 * (size_t)((D.n + 31) / 32));
    w.sb.FT = c.take<double>(U * (size_t)D.n * wc::ft_ld(D.r));
}

float *carve_weights(Carver &c, const wc_shape *s, wc::ProloguePartials *pp) {
    const wc::Dims D = dims_of(s);
    const size_t U = D.units();
    if (pp) {
        const int P = wc::prologue_num_splits(D);
        pp->P = P;
        pp->colsum = c.take<double>(U * P * D.d);
        pp->vmin = c.take<float>(U * P * D.d);
        pp->vmax = c.take<float>(U * P * D.d);
        pp->rq2 = c.take<double>(U * P);
        pp->rk2 = c.take<double>(U * P);
    }
    // fp32 split partials of Y~, followed by the fp64 reduced Y~ (8-byte aligned: the float count is even)
    const size_t parts = U * wc::weights_num_splits(D) * (size_t)D.r * (D.d + 1);
    // + the fp64 Y~, + the inverted diagonal blocks of L (solve scratch)
    return c.take<float>(((parts + 1) & ~size_t(1)) + 2 * U * (size_t)D.r * (D.d + 1) + 2 * U * wc::dinv_elems(D.r));
}

int finish(int launches) {
    if (launches < 0 || cudaPeekAtLastError() != cudaSuccess) return WC_ECUDA;
    g_launches = launches;
    return WC_OK;
}

int ws_ok(void *ws, size_t have, size_t need) {
    if (need && !ws) return WC_EWORKSPACE;
    if (have < need) return WC_EWORKSPACE;
    if (reinterpret_cast<uintptr_t>(ws) & 255) return WC_EWORKSPACE;
    return WC_OK;
}

}  // namespace

extern "C" {

size_t wc_workspace_bytes(const wc_shape *s, int op) {
    if (check_shape(s) != WC_OK) return 0;
    Carver c(nullptr);
    const wc::Dims D = dims_of(s);
    const size_t U = D.units();
    switch (op) {
        case WC_OP_SELECT: {
            SelectWs w;
            carve_select(c, s, w);
            break;
        }
        case WC_OP_WEIGHTS:
            carve_weights(c, s, nullptr);
            {
                wc::ProloguePartials pp;
                carve_weights(c, s, &pp);
            }
            break;
        case WC_OP_ATTEND: {
            const size_t a = wc::attend_ws_bytes(D);
            return a ? ((a + 255) & ~size_t(255)) + 256 : 0;
        }
        case WC_OP_FORWARD: {
            SelectWs w;
            carve_select(c, s, w);
            c.take<double>(U * WC_STATS_STRIDE(D.d));
            c.take<int32_t>(U * D.r);
            c.take<int32_t>(U);
            c.take<double>(U * (size_t)D.r * D.r);
            carve_weights(c, s, nullptr);
            c.take<char>(U * (size_t)D.r * D.d * esize(s));
            c.take<float>(U * (size_t)D.r * (D.d + 1));
            c.take<char>(2 * U * (size_t)D.d * esize(s));
            c.take<char>(wc::attend_ws_bytes(D));
            break;
        }
        case WC_OP_FORWARD_NSHARD:
            if (D.units() != 1) return 0;
            return wc::ns_workspace_bytes(D);
        default:
            return 0;
    }
    return ((c.off + 255) & ~size_t(255)) + 256;
}

int wildcat_select(const wc_shape *s, const wc_opts *o, const void *Q, const void *K, int32_t *S,
                   int32_t *r_eff, double *L, double *stats, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    if (!o || !K || !S || !r_eff || !L || !stats) return WC_EINVAL;
    if ((rc = check_opts(o, s))) return rc;
    const double rq = rq_of(o);
    if (rq < 0.0 && !Q && s->m > 0) return WC_EINVAL;  // m = 0: R_Q = max over no queries = 0
    if ((rc = ws_ok(ws, ws_bytes, wc_workspace_bytes(s, WC_OP_SELECT)))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const wc::Dims D = dims_of(s);
    Carver c(ws);
    SelectWs w;
    carve_select(c, s, w);
    const size_t U = D.units();
    if (cudaMemsetAsync(S, 0xff, U * D.r * sizeof(int32_t), st) != cudaSuccess) return WC_ECUDA;
    if (cudaMemsetAsync(L, 0, U * (size_t)D.r * D.r * sizeof(double), st) != cudaSuccess) return WC_ECUDA;
    tmark(st, true);
    int n1 = wc::launch_prologue(D, Q, K, nullptr, rq, beta_of(s, o), w.pp, stats, w.sb.nrm2, nullptr, nullptr, st);
    if (n1 < 0) return WC_ECUDA;
    tmark(st);
    int n2 = run_select(D, o, K, stats, w.sb, S, r_eff, L, st);
    if (n2 < 0) return n2;
    tmark(st);
    return finish(n1 + n2);
}

int wildcat_weights(const wc_shape *s, const wc_opts *o, const void *K, const void *V, const int32_t *S,
                    const int32_t *r_eff, const double *L, const double *stats, void *KS, float *X, void *vmin,
                    void *vmax, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    (void)o;
    if (!K || !V || !S || !r_eff || !L || !stats || !KS || !X || !vmin || !vmax) return WC_EINVAL;
    if ((rc = ws_ok(ws, ws_bytes, wc_workspace_bytes(s, WC_OP_WEIGHTS)))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const wc::Dims D = dims_of(s);
    Carver c(ws);
    float *Ypart = carve_weights(c, s, nullptr);
    wc::ProloguePartials pp;
    carve_weights(c, s, &pp);
    tmark(st, true);
    int n1 = wc::launch_vrange(D, V, pp, vmin, vmax, st);
    if (n1 < 0) return WC_ECUDA;
    tmark(st);
    int n2 = wc::launch_weights(D, K, V, S, r_eff, L, stats, Ypart, KS, X, st);
    if (n2 < 0) return WC_ECUDA;
    tmark(st);
    return finish(n1 + n2);
}

int wildcat_attend(const wc_shape *s, const wc_opts *o, const void *Q, const void *KS, const float *X,
                   const int32_t *r_eff, const void *vmin, const void *vmax, void *O, void *ws, size_t ws_bytes,
                   void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    if ((s->m > 0 && (!Q || !O)) || !KS || !X || !r_eff || !vmin || !vmax) return WC_EINVAL;
    if ((rc = ws_ok(ws, ws_bytes, wc_workspace_bytes(s, WC_OP_ATTEND)))) return rc;
    const int clip = (o && (o->flags & WC_NO_CLIP)) ? 0 : 1;
    tmark(static_cast<cudaStream_t>(stream), true);
    int n1 = wc::launch_attend(dims_of(s), Q, KS, X, r_eff, vmin, vmax, beta_of(s, o), clip, O, ws,
                               static_cast<cudaStream_t>(stream));
    if (n1 < 0) return WC_ECUDA;
    tmark(static_cast<cudaStream_t>(stream));
    return finish(n1);
}

int wildcat_forward(const wc_shape *s, const wc_opts *o, const void *Q, const void *K, const void *V, void *O,
                    int32_t *S_out, int32_t *reff_out, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    if (!o || !K || !V || (s->m > 0 && (!Q || !O))) return WC_EINVAL;
    if ((rc = check_opts(o, s))) return rc;
    const double rq = rq_of(o);
    if (rq < 0.0 && !Q && s->m > 0) return WC_EINVAL;  // m = 0: R_Q = max over no queries = 0
    if ((rc = ws_ok(ws, ws_bytes, wc_workspace_bytes(s, WC_OP_FORWARD)))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const wc::Dims D = dims_of(s);
    const size_t U = D.units();
    Carver c(ws);
    SelectWs w;
    carve_select(c, s, w);
    double *stats = c.take<double>(U * WC_STATS_STRIDE(D.d));
    int32_t *S = c.take<int32_t>(U * D.r);
    int32_t *reff = c.take<int32_t>(U);
    double *L = c.take<double>(U * (size_t)D.r * D.r);
    float *Ypart = carve_weights(c, s, nullptr);
    void *KS = c.take<char>(U * (size_t)D.r * D.d * esize(s));
    float *X = c.take<float>(U * (size_t)D.r * (D.d + 1));
    char *vr = c.take<char>(2 * U * (size_t)D.d * esize(s));
    void *vmin = vr, *vmax = vr + U * (size_t)D.d * esize(s);
    void *aimg = c.take<char>(wc::attend_ws_bytes(D));
    if (S_out) S = S_out;
    if (reff_out) reff = reff_out;
    if (cudaMemsetAsync(S, 0xff, U * D.r * sizeof(int32_t), st) != cudaSuccess) return WC_ECUDA;
    if (cudaMemsetAsync(L, 0, U * (size_t)D.r * D.r * sizeof(double), st) != cudaSuccess) return WC_ECUDA;
    const double beta = beta_of(s, o);
    int total = 0, k;
    tmark(st, true);
    if ((k = wc::launch_prologue(D, Q, K, V, rq, beta, w.pp, stats, w.sb.nrm2, vmin, vmax, st)) < 0) return WC_ECUDA;
    total += k;
    tmark(st);
    if ((k = run_select(D, o, K, stats, w.sb, S, reff, L, st)) < 0) return k;
    total += k;
    tmark(st);
    if ((k = wc::launch_weights(D, K, V, S, reff, L, stats, Ypart, KS, X, st)) < 0) return WC_ECUDA;
    total += k;
    tmark(st);
    const int clip = (o->flags & WC_NO_CLIP) ? 0 : 1;
    if ((k = wc::launch_attend(D, Q, KS, X, reff, vmin, vmax, beta, clip, O, aimg, st)) < 0) return WC_ECUDA;
    total += k;
    tmark(st);
    return finish(total);
}

int wc_comm_unique_id(void *id128) {
    if (!id128) return WC_EINVAL;
    return wc::ns_comm_unique_id(id128);
}

int wc_comm_init(void **comm, const void *id128, int world, int rank) {
    if (!comm || !id128 || world < 1 || world > wc::kMaxCpu || rank < 0 || rank >= world) return WC_EINVAL;
    return wc::ns_comm_init(comm, id128, world, rank);
}

int wc_comm_destroy(void *comm) { return wc::ns_comm_destroy(comm); }

int wildcat_forward_nshard(void *comm, const wc_shape *s, int64_t n_global, int64_t n_offset, const wc_opts *o,
                           const void *Q, const void *K, const void *V, void *O, int32_t *S, int32_t *r_eff,
                           void *ws, size_t ws_bytes, void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    if (!comm || !o || !K || !V || (s->m > 0 && (!Q || !O))) return WC_EINVAL;
    if (s->batch != 1 || s->heads_kv != 1) return WC_EUNSUPPORTED;
    if (o->block >= 2) return WC_EUNSUPPORTED;  // blocked selection is single-GPU in this build
    if (n_offset < 0 || n_global < s->n || n_offset + s->n > n_global || s->r > n_global) return WC_ESHAPE;
    if ((rc = ws_ok(ws, ws_bytes, wc_workspace_bytes(s, WC_OP_FORWARD_NSHARD)))) return rc;
    const double rq = rq_of(o);
    int launches = 0;
    rc = wc::ns_forward(comm, dims_of(s), n_global, n_offset, o, beta_of(s, o), rq, Q, K, V, O, S, r_eff, ws,
                        static_cast<cudaStream_t>(stream), &launches);
    if (rc) return rc;
    return finish(launches);
}

const char *wc_strerror(int st) {
    switch (st) {
        case WC_OK: return "ok";
        case WC_EINVAL: return "invalid argument (null pointer / bad option)";
        case WC_ESHAPE: return "invalid shape (r, n, m, d or head counts)";
        case WC_EDTYPE: return "unsupported dtype";
        case WC_EWORKSPACE: return "workspace too small or not 256-byte aligned";
        case WC_ECUDA: return "CUDA launch or runtime error";
        case WC_ENCCL: return "NCCL error";
        case WC_EUNSUPPORTED: return "unsupported configuration in this build (bins != 1)";
    }
    return "unknown status";
}

int wc_last_launch_count(void) { return g_launches; }

int wc_timing_enable(int on) {
    g_timing = on != 0;
    g_nev = 0;
    return WC_OK;
}

int wc_timing_read(float *ms, int cap) {
    if (!ms || cap < 0) return WC_EINVAL;
    if (g_nev < 2) return 0;
    if (cudaEventSynchronize(g_ev[g_nev - 1]) != cudaSuccess) return WC_ECUDA;
    int k = 0;
    for (; k < g_nev - 1 && k < cap; ++k)
        if (cudaEventElapsedTime(&ms[k], g_ev[k], g_ev[k + 1]) != cudaSuccess) return WC_ECUDA;
    return k;
}

int wc_version(void) { return 101; }

}  // extern "C"
