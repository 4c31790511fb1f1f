// api.cu -- the C ABI of libwildcat.so (declared in include/wildcat.h).
// Argument validation, workspace carving and kernel sequencing only; every arithmetic step
// of the method runs in the sm_100a kernels of prologue.cu / select.cu / weights.cu / attend.cu.
#include <algorithm>
#include <cmath>
#include <initializer_list>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/wildcat.h"
#include "kernels.h"

static_assert(WC_STATS_HEAD == wc::kStatsHead, "stats layout of include/wildcat.h and the kernels differ");
static_assert(WC_MAX_R == wc::kMaxR, "WC_MAX_R of include/wildcat.h and the kernels' plan differ");

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
    if (s->bins < 1 || s->bins > s->r) return WC_ESHAPE;  // (so bins <= r <= n: every bin has a key)
    return WC_OK;
}

wc::Dims dims_of(const wc_shape *s) {
    wc::Dims D;
    D.batch = s->batch; D.hq = s->heads_q; D.hkv = s->heads_kv; D.d = s->d; D.r = s->r; D.dtype = s->dtype;
    D.m = s->m; D.n = s->n;
    return D;
}

// Binning plan (Alg 2; readings Z12, Z13, Z23).  D: the unit-level problem (prologue,
// value range, attend with R coreset rows); Ds: the sub-unit problem of the selection and weights
// kernels -- unit u, bin b -> sub-unit u*B + b with nb = floor(n/B) keys (the last bin also holds the
// n - B nb remainder: Ds.n = nb + remainder is the per-sub-unit buffer size, Dims::sub_unit() the
// geometry) and rank rb = min(ceil(r/B), nb).  With B = 1, Ds = D and R = r.
struct Plan {
    wc::Dims D, Ds, Da;  // unit level, sub-unit level, attend (unit level with r = R)
    int B, rb, R;
};
Plan plan_of(const wc_shape *s) {
    Plan p;
    p.D = dims_of(s);
    p.B = s->bins;
    const int64_t nb = s->n / p.B;
    p.rb = (int)std::min<int64_t>((s->r + p.B - 1) / p.B, nb);
    p.R = p.B * p.rb;
    p.Ds = p.D;
    p.Ds.hkv = p.D.hkv * p.B;
    p.Ds.hq = p.D.hq * p.B;  // keeps group() = hq/hkv; the sub-unit dims never touch Q
    p.Ds.n = nb + (s->n - (int64_t)p.B * nb);
    p.Ds.r = p.rb;
    p.Ds.bins = p.B;
    p.Ds.nb = nb;
    p.Ds.unit_n = s->n;
    p.Da = p.D;
    p.Da.r = p.R;
    return p;
}

size_t esize(const wc_shape *s) { return s->dtype == WC_F32 ? 4 : 2; }

double beta_of(const wc_shape *s, const wc_opts *o) {
    return (o && o->beta > 0.0) ? o->beta : 1.0 / std::sqrt((double)s->d);
}
double rq_of(const wc_opts *o) {
    if (!o || std::isnan(o->rq) || o->rq < 0.0) return -1.0;
    return o->rq;
}

// Selection dispatch: sequential Alg 1, or the blocked variant when opts->block >= 2.  unit0 = the
// Philox id of the call's first sub-unit: opts->unit_offset * B (PAR2; readings Z2, Z23).
int run_select(const wc::Dims &D, const wc_opts *o, uint64_t unit0, const void *K, double *stats, wc::SelectBufs sb,
               int32_t *S, int32_t *r_eff, double *L, cudaStream_t st) {
    if (o->block >= 2) {
        const int k = wc::launch_select_blocked(D, K, stats, sb, o->seed, unit0, (int)o->block, S, r_eff, L, st);
        return k == -2 ? WC_EUNSUPPORTED : (k < 0 ? WC_ECUDA : k);
    }
    const int k = wc::launch_select(D, K, stats, sb, o->seed, unit0, S, r_eff, L, st);
    return k < 0 ? WC_ECUDA : k;
}

int pflags_of(const wc_opts *o) {
    int f = 0;
    if (o && (o->flags & WC_TAU_ONE)) f |= wc::kPfTauOne;
    if (o && (o->flags & WC_NO_RECENTER)) f |= wc::kPfNoRecenter;
    return f;
}

// WC_CHECK_FINITE (debug): scan the inputs before anything else is launched, synchronise the stream
// once, and report WC_ENONFINITE if one holds a NaN / Inf.  `scratch` (4 device bytes the call may
// overwrite: its workspace or an output) receives the flag.
struct Arr {
    const void *p;
    int64_t count;
};
int check_finite(const wc_opts *o, int dtype, void *scratch, std::initializer_list<Arr> arrs, cudaStream_t st,
                 int *launches) {
    if (!o || !(o->flags & WC_CHECK_FINITE)) return WC_OK;
    if (!scratch) return WC_OK;  // nothing to scan (no inputs with elements)
    int *flag = static_cast<int *>(scratch);
    if (cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess) return WC_ECUDA;
    for (const Arr &a : arrs) {
        const int k = wc::launch_check_finite(a.p, a.count, dtype, flag, st);
        if (k < 0) return WC_ECUDA;
        *launches += k;
    }
    int h = 0;
    if (cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) return WC_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return WC_ECUDA;
    return h ? WC_ENONFINITE : WC_OK;
}

int64_t q_elems(const wc_shape *s) { return (int64_t)s->batch * s->heads_q * s->m * s->d; }
int64_t kv_elems(const wc_shape *s) { return (int64_t)s->batch * s->heads_kv * s->n * s->d; }

int check_opts(const wc_opts *o, const wc_shape *s) {
    if (!o) return WC_EINVAL;
    if (o->flags & ~WC_FLAGS_ALL) return WC_EINVAL;
    if (o->block > (uint32_t)WC_MAX_BLOCK) return WC_EINVAL;
    const Plan p = plan_of(s);
    if (p.rb > WC_MAX_R) return WC_EUNSUPPORTED;  // solve / blocked plan (every selection path)
    if (o->block >= 2 && !wc::select_blocked_plan_ok(p.Ds, (int)o->block)) return WC_EUNSUPPORTED;
    return WC_OK;
}

void carve_prologue(Carver &c, const wc::Dims &D, wc::ProloguePartials &pp) {
    const size_t U = D.units();
    const int P = wc::prologue_num_splits(D);
    pp.P = P;
    pp.colsum = c.take<double>(U * P * D.d);
    pp.vmin = c.take<float>(U * P * D.d);
    pp.vmax = c.take<float>(U * P * D.d);
    pp.rq2 = c.take<double>(U * P);
    pp.rk2 = c.take<double>(U * P);
}

// Selection workspace: unit-level prologue partials and nrm2 ([units][n] == [units*B][nb]), the
// selection state at the sub-unit level, and (B > 1) the unit-level stats and sub-unit S / r_eff.
struct SelectWs {
    wc::ProloguePartials pp;
    wc::SelectBufs sb;
    double *stats_u = nullptr;
    int32_t *Ssub = nullptr, *reff_sub = nullptr;
};
void carve_select(Carver &c, const Plan &p, SelectWs &w) {
    carve_prologue(c, p.D, w.pp);
    const wc::Dims &D = p.Ds;
    const size_t U = D.units();
    w.sb.nrm2 = c.take<double>(U * D.n);
    w.sb.p = c.take<double>(2 * U * D.n);
    w.sb.F = c.take<double>(U * wc::f_elems_per_unit(D.n, D.r, wc::select_ctas_per_unit(D)));
    w.sb.part = c.take<double>(U * 2 * wc::kMaxCpu);
    w.sb.bar = c.take<unsigned>(U);
    w.sb.gsum = c.take<double>(U * 2 * (size_t)((D.n + 31) / 32));
    if (wc::select_ctas_per_unit(D) >= wc::kRejMinCpu) w.sb.rej = c.take<double>(U * wc::kRejStride);
    if (p.B > 1) {
        w.stats_u = c.take<double>((size_t)p.D.units() * WC_STATS_STRIDE(D.d));
        w.Ssub = c.take<int32_t>(U * D.r);
        w.reff_sub = c.take<int32_t>(U);
    }
}

// Weights workspace at the sub-unit level: fp32 split partials of Y~, the fp64 Y~, the inverted
// diagonal blocks of L; (B > 1) sub-unit S / r_eff and the unpacked KS / X.
struct WeightsWs {
    float *Ypart = nullptr;
    int32_t *Ssub = nullptr, *reff_sub = nullptr;
    void *KSsub = nullptr;
    float *Xsub = nullptr;
};
void carve_weights(Carver &c, const wc_shape *s, const Plan &p, WeightsWs &w) {
    const wc::Dims &D = p.Ds;
    const size_t U = D.units();
    const size_t parts = U * wc::weights_num_splits(D) * (size_t)D.r * (D.d + 1);
    w.Ypart = c.take<float>(((parts + 1) & ~size_t(1)) + 2 * U * (size_t)D.r * (D.d + 1) + 2 * U * wc::dinv_elems(D.r) +
                            2 * U * wc::solve_scratch_elems(D.r, D.d));
    if (p.B > 1) {
        w.Ssub = c.take<int32_t>(U * D.r);
        w.reff_sub = c.take<int32_t>(U);
        w.KSsub = c.take<char>(U * (size_t)D.r * D.d * esize(s));
        w.Xsub = c.take<float>(U * (size_t)D.r * (D.d + 1));
    }
}

// wildcat_forward workspace: selection + weights + the forward's own buffers.
struct ForwardWs {
    SelectWs sel;
    WeightsWs wts;
    double *stats = nullptr;  // [units*B][stride] (sub-unit stats; == unit stats when B = 1)
    int32_t *S = nullptr, *reff = nullptr;
    double *L = nullptr;
    void *KS = nullptr, *vmin = nullptr, *vmax = nullptr, *aimg = nullptr;
    float *X = nullptr;
};
void carve_forward(Carver &c, const wc_shape *s, const Plan &p, ForwardWs &w) {
    carve_select(c, p, w.sel);
    const size_t U = p.D.units(), Us = p.Ds.units();
    w.stats = c.take<double>(Us * WC_STATS_STRIDE(p.D.d));
    w.S = c.take<int32_t>(U * p.R);
    w.reff = c.take<int32_t>(U);
    w.L = c.take<double>(Us * (size_t)p.rb * p.rb);
    carve_weights(c, s, p, w.wts);
    w.KS = c.take<char>(U * (size_t)p.R * p.D.d * esize(s));
    w.X = c.take<float>(U * (size_t)p.R * (p.D.d + 1));
    char *vr = c.take<char>(2 * U * (size_t)p.D.d * esize(s));
    w.vmin = vr;
    w.vmax = vr ? vr + U * (size_t)p.D.d * esize(s) : nullptr;
    w.aimg = c.take<char>(wc::attend_ws_bytes(p.Da));
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

size_t rounded(const Carver &c) { return ((c.off + 255) & ~size_t(255)) + 256; }

// A0 + A1/A2 for a plan.  B = 1: prologue into `stats`, selection into S / r_eff / L.
// B > 1: unit prologue into w.stats_u, per-bin stats into `stats` ([units*B]), selection at the
// sub-unit level into w.Ssub / w.reff_sub and L ([units][B][rb][rb]); then S / r_eff packed.
int select_stage(const Plan &p, const wc_opts *o, double beta, double rq, const void *Q, const void *K, const void *V,
                 SelectWs &w, double *stats, int32_t *S, int32_t *r_eff, double *L, void *vmin, void *vmax,
                 cudaStream_t st, int *launches) {
    const size_t Us = p.Ds.units();
    int32_t *Ssel = p.B > 1 ? w.Ssub : S;
    int32_t *Rsel = p.B > 1 ? w.reff_sub : r_eff;
    wc::ProloguePartials pp = w.pp;  // pass 1 also initialises S (-1) and L (0)
    pp.fill_S = Ssel;
    pp.nS = (int64_t)Us * p.rb;
    pp.zero_L = L;
    pp.nL = (int64_t)Us * p.rb * p.rb;
    const int pf = pflags_of(o);
    int k = wc::launch_prologue(p.D, Q, K, V, rq, beta, pp, p.B > 1 ? w.stats_u : stats, w.sb.nrm2, vmin, vmax, pf,
                                st);
    if (k < 0) return WC_ECUDA;
    *launches += k;
    if (p.B > 1) {
        if ((k = wc::launch_bins_stats(p.D, p.B, beta, w.stats_u, w.sb.nrm2, stats, pf, st)) < 0) return WC_ECUDA;
        *launches += k;
    }
    tmark(st);
    if ((k = run_select(p.Ds, o, o->unit_offset * (uint64_t)p.B, K, stats, w.sb, Ssel, Rsel, L, st)) < 0) return k;
    *launches += k;
    if (p.B > 1) {
        if ((k = wc::launch_bins_pack(p.D, p.B, p.rb, w.Ssub, w.reff_sub, nullptr, nullptr, S, r_eff, nullptr, nullptr,
                                      st)) < 0)
            return WC_ECUDA;
        *launches += k;
    }
    return WC_OK;
}

// A3 + A4 for a plan (S / r_eff packed at the unit level when B > 1; unpacked here).
int weights_stage(const Plan &p, const void *K, const void *V, const int32_t *S, const int32_t *r_eff, const double *L,
                  const double *stats, WeightsWs &w, bool have_sub, void *KS, float *X, cudaStream_t st, int *launches) {
    int k;
    if (p.B == 1) {
        if ((k = wc::launch_weights(p.D, K, V, S, r_eff, L, stats, w.Ypart, KS, X, st)) < 0) return WC_ECUDA;
        *launches += k;
        return WC_OK;
    }
    if (!have_sub) {
        if ((k = wc::launch_bins_unpack(p.D, p.B, p.rb, S, w.Ssub, w.reff_sub, st)) < 0) return WC_ECUDA;
        *launches += k;
    }
    if ((k = wc::launch_weights(p.Ds, K, V, w.Ssub, w.reff_sub, L, stats, w.Ypart, w.KSsub, w.Xsub, st)) < 0)
        return WC_ECUDA;
    *launches += k;
    if ((k = wc::launch_bins_pack(p.D, p.B, p.rb, w.Ssub, w.reff_sub, w.KSsub, w.Xsub, nullptr, nullptr, KS, X, st)) < 0)
        return WC_ECUDA;
    *launches += k;
    return WC_OK;
}

// ---- KV-cache compression (reading Z24): full-context shape -> the middle's shape.
struct KvPlan {
    wc_shape full, mid;
    int64_t nmid = 0;
    int kf = 0, kl = 0, R = 0;
    bool has_mid = false;
};
int kv_plan(const wc_shape *s, int32_t kf, int32_t kl, KvPlan &kp) {
    if (!s) return WC_EINVAL;
    if (kf < 0 || kl < 0) return WC_ESHAPE;
    kp.full = *s;
    kp.full.r = 1;
    kp.full.bins = 1;
    int rc = check_shape(&kp.full);
    if (rc) return rc;
    kp.kf = kf;
    kp.kl = kl;
    kp.nmid = s->n - (int64_t)kf - (int64_t)kl;
    if (kp.nmid < 0) return WC_ESHAPE;
    kp.has_mid = kp.nmid > 0;
    if (kp.has_mid) {
        kp.mid = *s;
        kp.mid.n = kp.nmid;
        if ((rc = check_shape(&kp.mid))) return rc;
        kp.R = plan_of(&kp.mid).R;
    }
    return WC_OK;
}

struct KvWs {
    wc::ProloguePartials ppf;  // value range over the full V
    void *Kmid = nullptr, *Vmid = nullptr;
    SelectWs sel;
    WeightsWs wts;
    double *stats = nullptr, *L = nullptr;
    int32_t *S = nullptr, *reff = nullptr;
    void *KS = nullptr;
    float *X = nullptr;
};
void carve_kv(Carver &c, const KvPlan &kp, KvWs &w) {
    carve_prologue(c, dims_of(&kp.full), w.ppf);
    if (!kp.has_mid) return;
    const Plan p = plan_of(&kp.mid);
    const size_t U = p.D.units(), Us = p.Ds.units(), e = esize(&kp.mid);
    w.Kmid = c.take<char>(U * (size_t)kp.nmid * p.D.d * e);
    w.Vmid = c.take<char>(U * (size_t)kp.nmid * p.D.d * e);
    carve_select(c, p, w.sel);
    carve_weights(c, &kp.mid, p, w.wts);
    w.stats = c.take<double>(Us * WC_STATS_STRIDE(p.D.d));
    w.S = c.take<int32_t>(U * p.R);
    w.reff = c.take<int32_t>(U);
    w.L = c.take<double>(Us * (size_t)p.rb * p.rb);
    w.KS = c.take<char>(U * (size_t)p.R * p.D.d * e);
    w.X = c.take<float>(U * (size_t)p.R * (p.D.d + 1));
}

}  // namespace

extern "C" {

size_t wc_workspace_bytes(const wc_shape *s, int op) {
    if (check_shape(s) != WC_OK) return 0;
    Carver c(nullptr);
    const Plan p = plan_of(s);
    switch (op) {
        case WC_OP_SELECT: {
            SelectWs w;
            carve_select(c, p, w);
            break;
        }
        case WC_OP_WEIGHTS: {
            WeightsWs w;
            carve_weights(c, s, p, w);
            wc::ProloguePartials pp;
            carve_prologue(c, p.D, pp);
            break;
        }
        case WC_OP_ATTEND: {
            const size_t a = wc::attend_ws_bytes(p.Da);
            return a ? ((a + 255) & ~size_t(255)) + 256 : 0;
        }
        case WC_OP_FORWARD: {
            ForwardWs w;
            carve_forward(c, s, p, w);
            break;
        }
        case WC_OP_FORWARD_NSHARD:
            if (p.D.units() != 1 || p.B != 1) return 0;
            return wc::ns_workspace_bytes(p.D);
        default:
            return 0;
    }
    return rounded(c);
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
    const Plan p = plan_of(s);
    int launches = 0;
    if ((rc = check_finite(o, s->dtype, ws, {{Q, rq < 0.0 ? q_elems(s) : 0}, {K, kv_elems(s)}}, st, &launches)))
        return rc;
    Carver c(ws);
    SelectWs w;
    carve_select(c, p, w);
    tmark(st, true);
    if ((rc = select_stage(p, o, beta_of(s, o), rq, Q, K, nullptr, w, stats, S, r_eff, L, nullptr, nullptr, st,
                           &launches)))
        return rc;
    tmark(st);
    return finish(launches);
}

int wildcat_weights(const wc_shape *s, const wc_opts *o, const void *K, const void *V, const int32_t *S,
                    const int32_t *r_eff, const double *L, const double *stats, void *KS, float *X, void *vmin,
                    void *vmax, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    if (!K || !V || !S || !r_eff || !L || !stats || !KS || !X || !vmin || !vmax) return WC_EINVAL;
    if (o && (o->flags & ~WC_FLAGS_ALL)) return WC_EINVAL;
    if (plan_of(s).rb > WC_MAX_R) return WC_EUNSUPPORTED;  // the solve's plan
    if ((rc = ws_ok(ws, ws_bytes, wc_workspace_bytes(s, WC_OP_WEIGHTS)))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Plan p = plan_of(s);
    Carver c(ws);
    WeightsWs w;
    carve_weights(c, s, p, w);
    wc::ProloguePartials pp;
    carve_prologue(c, p.D, pp);
    int launches = 0;
    if ((rc = check_finite(o, s->dtype, ws, {{K, kv_elems(s)}, {V, kv_elems(s)}}, st, &launches))) return rc;
    tmark(st, true);
    const int kv = wc::launch_vrange(p.D, V, pp, vmin, vmax, st);
    if (kv < 0) return WC_ECUDA;
    launches += kv;
    tmark(st);
    if ((rc = weights_stage(p, K, V, S, r_eff, L, stats, w, false, KS, X, st, &launches))) return rc;
    tmark(st);
    return finish(launches);
}

int wildcat_attend(const wc_shape *s, const wc_opts *o, const void *Q, const void *KS, const float *X,
                   const int32_t *r_eff, const void *vmin, const void *vmax, void *O, void *ws, size_t ws_bytes,
                   void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    if ((s->m > 0 && (!Q || !O)) || !KS || !X || !r_eff || !vmin || !vmax) return WC_EINVAL;
    if ((rc = ws_ok(ws, ws_bytes, wc_workspace_bytes(s, WC_OP_ATTEND)))) return rc;
    if (o && (o->flags & ~WC_FLAGS_ALL)) return WC_EINVAL;
    const int clip = (o && (o->flags & WC_NO_CLIP)) ? 0 : 1;
    int nf = 0;  // the queries are the attend's only caller-provided input (O is scratch for the flag)
    if ((rc = check_finite(o, s->dtype, s->m > 0 ? O : nullptr, {{Q, q_elems(s)}}, static_cast<cudaStream_t>(stream),
                           &nf)))
        return rc;
    tmark(static_cast<cudaStream_t>(stream), true);
    int n1 = wc::launch_attend(plan_of(s).Da, Q, KS, X, r_eff, vmin, vmax, beta_of(s, o), clip, O, ws,
                               static_cast<cudaStream_t>(stream));
    if (n1 < 0) return WC_ECUDA;
    tmark(static_cast<cudaStream_t>(stream));
    return finish(n1 + nf);
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
    const Plan p = plan_of(s);
    Carver c(ws);
    ForwardWs w;
    carve_forward(c, s, p, w);
    int32_t *S = S_out ? S_out : w.S;
    int32_t *reff = reff_out ? reff_out : w.reff;
    const double beta = beta_of(s, o);
    int launches = 0;
    if ((rc = check_finite(o, s->dtype, ws, {{Q, q_elems(s)}, {K, kv_elems(s)}, {V, kv_elems(s)}}, st, &launches)))
        return rc;
    tmark(st, true);
    if ((rc = select_stage(p, o, beta, rq, Q, K, V, w.sel, w.stats, S, reff, w.L, w.vmin, w.vmax, st, &launches)))
        return rc;
    tmark(st);
    // B > 1: the sub-unit S / r_eff of the selection are still in w.sel
    if (p.B > 1) {
        w.wts.Ssub = w.sel.Ssub;
        w.wts.reff_sub = w.sel.reff_sub;
    }
    if ((rc = weights_stage(p, K, V, S, reff, w.L, w.stats, w.wts, true, w.KS, w.X, st, &launches))) return rc;
    tmark(st);
    const int clip = (o->flags & WC_NO_CLIP) ? 0 : 1;
    int k;
    if ((k = wc::launch_attend(p.Da, Q, w.KS, w.X, reff, w.vmin, w.vmax, beta, clip, O, w.aimg, st)) < 0)
        return WC_ECUDA;
    launches += k;
    tmark(st);
    return finish(launches);
}

size_t wc_kv_capacity(const wc_shape *s, int32_t keep_first, int32_t keep_last) {
    KvPlan kp;
    if (kv_plan(s, keep_first, keep_last, kp) != WC_OK) return 0;
    return (size_t)keep_first + (size_t)keep_last + (size_t)kp.R;
}

size_t wc_kv_workspace_bytes(const wc_shape *s, int32_t keep_first, int32_t keep_last) {
    KvPlan kp;
    if (kv_plan(s, keep_first, keep_last, kp) != WC_OK) return 0;
    Carver c(nullptr);
    KvWs w;
    carve_kv(c, kp, w);
    return rounded(c);
}

int wildcat_compress_kv(const wc_shape *s, const wc_opts *o, int32_t keep_first, int32_t keep_last, const void *Q,
                        const void *K, const void *V, void *KC, void *VC, float *WC, int32_t *c_eff, void *vmin,
                        void *vmax, int32_t *S_out, void *ws, size_t ws_bytes, void *stream) {
    KvPlan kp;
    int rc = kv_plan(s, keep_first, keep_last, kp);
    if (rc) return rc;
    if (!o || !K || !V || !KC || !VC || !WC || !c_eff || !vmin || !vmax) return WC_EINVAL;
    if (kp.has_mid && (rc = check_opts(o, &kp.mid))) return rc;
    const double rq = rq_of(o);
    if (kp.has_mid && rq < 0.0 && !Q && s->m > 0) return WC_EINVAL;
    if ((rc = ws_ok(ws, ws_bytes, wc_kv_workspace_bytes(s, keep_first, keep_last)))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver c(ws);
    KvWs w;
    carve_kv(c, kp, w);
    const wc::Dims Df = dims_of(&kp.full);
    int launches = 0, k;
    if ((rc = check_finite(o, s->dtype, ws, {{Q, rq < 0.0 ? q_elems(s) : 0}, {K, kv_elems(s)}, {V, kv_elems(s)}}, st,
                           &launches)))
        return rc;
    tmark(st, true);
    if ((k = wc::launch_vrange(Df, V, w.ppf, vmin, vmax, st)) < 0) return WC_ECUDA;  // full V
    launches += k;
    if (kp.has_mid) {
        const Plan p = plan_of(&kp.mid);
        const size_t e = esize(s), row = (size_t)s->d * e;
        // the middle tokens of every unit, packed [units][nmid][d] for the per-unit kernels
        for (int t = 0; t < 2; ++t) {
            if (cudaMemcpy2DAsync(t ? w.Vmid : w.Kmid, kp.nmid * row,
                                  static_cast<const char *>(t ? V : K) + (size_t)keep_first * row, s->n * row,
                                  kp.nmid * row, Df.units(), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return WC_ECUDA;
        }
        tmark(st);
        if ((rc = select_stage(p, o, beta_of(s, o), rq, Q, w.Kmid, nullptr, w.sel, w.stats, w.S, w.reff, w.L, nullptr,
                               nullptr, st, &launches)))
            return rc;
        tmark(st);
        if (p.B > 1) {
            w.wts.Ssub = w.sel.Ssub;
            w.wts.reff_sub = w.sel.reff_sub;
        }
        if ((rc = weights_stage(p, w.Kmid, w.Vmid, w.S, w.reff, w.L, w.stats, w.wts, true, w.KS, w.X, st, &launches)))
            return rc;
    }
    tmark(st);
    if ((k = wc::launch_kv_assemble(Df, K, V, keep_first, keep_last, kp.R, w.KS, w.X, w.S, w.reff, KC, VC, WC, c_eff,
                                    S_out, st)) < 0)
        return WC_ECUDA;
    launches += k;
    tmark(st);
    return finish(launches);
}

// ---- decode over a compact KV cache (WtdAttn, Alg 3): shape.r = C rows, bins = 1
static wc::Dims decode_dims(const wc_shape *s) {
    wc::Dims D = dims_of(s);
    D.r = s->r;
    return D;
}

size_t wc_decode_workspace_bytes(const wc_shape *s) {
    if (check_shape(s) != WC_OK || s->bins != 1) return 0;
    const wc::Dims D = decode_dims(s);
    if (D.m <= wc::kDecodeMaxM) return ((wc::attend_decode_ws_bytes(D) + 255) & ~size_t(255)) + 256;
    const size_t x = (size_t)D.units() * D.r * (D.d + 1) * sizeof(float);
    return ((x + 255) & ~size_t(255)) + ((wc::attend_ws_bytes(D) + 255) & ~size_t(255)) + 256;
}

int wildcat_decode(const wc_shape *s, const wc_opts *o, const void *Q, const void *KC, const void *VC, const float *WC,
                   const int32_t *c_eff, const void *vmin, const void *vmax, void *O, void *ws, size_t ws_bytes,
                   void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    if (s->bins != 1) return WC_ESHAPE;
    if ((s->m > 0 && (!Q || !O)) || !KC || !VC || !WC || !c_eff || !vmin || !vmax) return WC_EINVAL;
    if (o && (o->flags & ~WC_FLAGS_ALL)) return WC_EINVAL;
    if ((rc = ws_ok(ws, ws_bytes, wc_decode_workspace_bytes(s)))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int clip = (o && (o->flags & WC_NO_CLIP)) ? 0 : 1;
    int nf = 0;
    if ((rc = check_finite(o, s->dtype, s->m > 0 ? O : nullptr, {{Q, q_elems(s)}}, st, &nf))) return rc;
    const wc::Dims D = decode_dims(s);
    tmark(st, true);
    int k;
    if (D.m <= wc::kDecodeMaxM) {
        k = wc::launch_attend_decode_vw(D, Q, KC, VC, WC, c_eff, vmin, vmax, beta_of(s, o), clip, O, ws, st);
    } else {  // many queries: expand the cache rows to [V_S, w] and run the general attend
        float *X = static_cast<float *>(ws);
        const size_t x = (size_t)D.units() * D.r * (D.d + 1) * sizeof(float);
        void *aws = static_cast<char *>(ws) + ((x + 255) & ~size_t(255));
        k = wc::launch_vw_to_x(D, VC, WC, X, st);
        if (k >= 0) {
            const int k2 = wc::launch_attend(D, Q, KC, X, c_eff, vmin, vmax, beta_of(s, o), clip, O, aws, st);
            k = k2 < 0 ? -1 : k + k2;
        }
    }
    if (k < 0) return WC_ECUDA;
    tmark(st);
    return finish(k + nf);
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

int wc_p2p_comm_create(void **comm, int world, int rank, size_t capacity, void *handle64) {
    if (!comm || !handle64) return WC_EINVAL;
    return wc::ns_p2p_create(comm, world, rank, capacity, handle64);
}

int wc_p2p_comm_connect(void *comm, const void *handles) { return wc::ns_p2p_connect(comm, handles); }

int wildcat_forward_nshard(void *comm, const wc_shape *s, int64_t n_global, int64_t n_offset, const wc_opts *o,
                           const void *Q, const void *K, const void *V, void *O, int32_t *S, int32_t *r_eff,
                           void *ws, size_t ws_bytes, void *stream) {
    int rc = check_shape(s);
    if (rc) return rc;
    if (!comm || !o || !K || !V || (s->m > 0 && (!Q || !O))) return WC_EINVAL;
    if (s->batch != 1 || s->heads_kv != 1) return WC_EUNSUPPORTED;
    if (s->bins != 1) return WC_EUNSUPPORTED;               // binned selection is single-GPU
    if (o->block > 16) return WC_EUNSUPPORTED;              // the n-sharded blocked plan: b <= 16
    if (s->r > WC_MAX_R) return WC_EUNSUPPORTED;                  // the solve's plan
    if (n_offset < 0 || n_global < s->n || n_offset + s->n > n_global || s->r > n_global) return WC_ESHAPE;
    if ((rc = ws_ok(ws, ws_bytes, wc_workspace_bytes(s, WC_OP_FORWARD_NSHARD)))) return rc;
    if (o->flags & ~WC_FLAGS_ALL) return WC_EINVAL;
    const double rq = rq_of(o);
    int launches = 0;
    if ((rc = check_finite(o, s->dtype, ws, {{Q, q_elems(s)}, {K, kv_elems(s)}, {V, kv_elems(s)}},
                           static_cast<cudaStream_t>(stream), &launches)))
        return rc;
    int nf = launches;
    rc = wc::ns_forward(comm, dims_of(s), n_global, n_offset, o, beta_of(s, o), rq, Q, K, V, O, S, r_eff, ws,
                        static_cast<cudaStream_t>(stream), &launches);
    if (rc) return rc;
    return finish(launches + nf);
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
        case WC_EUNSUPPORTED: return "unsupported configuration in this build (n-sharded bins/blocks, r too large for the selection plan)";
        case WC_ENONFINITE: return "non-finite input (NaN or Inf) found by WC_CHECK_FINITE";
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

int wc_version(void) { return 201; }

}  // extern "C"
