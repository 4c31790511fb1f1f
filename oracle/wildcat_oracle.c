/*
 * wildcat_oracle.c -- plain, slow, fp64 CPU oracle for WildCat (arxiv 2602.10056).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (libwildcat.so + its Python binding) never calls it and
 * shares no code, header, table or helper with it.
 *
 * Every function follows PAPER.md (cited as P:<line>) step by step in fp64,
 * with no blocking, fusion or reordering beyond what the paper states.
 * Where the paper is silent the reading taken is the one listed in
 * DESIGN.md "Readings" (Z-numbers follow SURVEY.md section 8(c)).
 *
 * Floating point: compiled with -O2 -ffp-contract=off (no FMA contraction),
 * round-to-nearest; OpenMP only across independent keys or queries (each
 * output entry is still summed in its own fixed sequential order).
 *
 * Parity pins: every function here is pinned by a -m "not gpu" test in
 * tests/test_oracle_*.py against something other than itself (published
 * known-answer vectors, closed forms, the paper's ODE, brute-force
 * enumeration, an independent library solve).  See DESIGN.md "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11 "Random123").  Not from the paper: the
 * paper does not name its random number generator (reading Z2).  Pinned by
 * the Random123 known-answer vectors in tests/test_oracle_rng.py.          */
/* ------------------------------------------------------------------------ */
void wco_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The pivot uniform of round i for unit `unit` (reading Z2):
 *   (x0,x1,x2,x3) = Philox4x32-10(key=(seed_lo,seed_hi), ctr=(i, unit_lo, unit_hi, 'PIVT'))
 *   u = ((x0>>5)*2^26 + (x1>>6)) * 2^-53  in [0,1).                          */
double wco_pivot_uniform(uint64_t seed, uint32_t round_i, uint64_t unit)
{
    uint32_t ctr[4] = {round_i, (uint32_t)unit, (uint32_t)(unit >> 32), 0x50495654u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    wco_philox4x32_10(ctr, key, x);
    double a = (double)(x[0] >> 5);
    double b = (double)(x[1] >> 6);
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------------------ */
/* Lambert W0 by the Loczi iteration, P:1877-1890 (Appendix "Properties of the
 * Lambert W Function", theorem "Fast Lambert W calculation"):
 *   beta_0 = log z - log log z   (z > e);   exp(log z - 1)  (z < e)
 *   beta_{k+1} = beta_k/(1+beta_k) * (1 + log z - log beta_k)
 * 6 iterations (reading Z17: error < max(0.32^64, 0.633^64/3)).  At z = e
 * both seeds equal 1, which is W0(e), so the first branch is used for z >= e.
 * z = 0 returns 0 (W0(0) = 0).  z < 0 is not needed (returns NaN). */
/* ------------------------------------------------------------------------ */
double wco_lambert_w0(double z)
{
    if (z == 0.0) return 0.0;
    if (!(z > 0.0)) return NAN;
    double lz = log(z);
    double b;
    if (z >= M_E) b = lz - log(lz);
    else          b = exp(lz - 1.0);
    for (int k = 0; k < 6; ++k)
        b = b / (1.0 + b) * (1.0 + lz - log(b));
    return b;
}

/* rho_0 = sqrt(1 + e^{W0(2/e^2) + 2}) ~= 3.19, P:282 (below Eq. 7). */
double wco_rho0(void)
{
    double w = wco_lambert_w0(2.0 / (M_E * M_E));
    return sqrt(1.0 + exp(w + 2.0));
}

/* Temperature, Eq. 7:
 *   tau = sqrt( (R_K/R_Q) * b0 / (2 W0(b0/(2 rho0))) ),  b0 = log(n)/(beta R_Q R_K) + 2.
 * Fallback tau = 1 when R_Q * R_K = 0 (b0 undefined; reading S:192).       */
double wco_temperature(double beta, double rq, double rk, int64_t n)
{
    if (!(rq * rk > 0.0)) return 1.0;
    double rho0 = wco_rho0();
    double b0 = log((double)n) / (beta * rq * rk) + 2.0;
    double w = wco_lambert_w0(b0 / (2.0 * rho0));
    return sqrt((rk / rq) * b0 / (2.0 * w));
}

/* ------------------------------------------------------------------------ */
/* Prologue of one unit: Alg 4 P:352-354 and Alg 2 P:300-305.
 *   kbar = row mean of K ("Recenter keys");  R_K = max_l ||k_l - kbar||;
 *   R_Q = max_i ||q_i|| over the unit's query rows, unless rq_given >= 0
 *   (Alg 2 takes R_Q as an input; reading Z11);
 *   tau (Eq. 7), g = beta/tau^2, mstar = g R_K^2 (reading Z10: the kernel used for
 *   selection and weights is h~(a,b) = exp(g<a-kbar,b-kbar> - mstar), which is
 *   h_tau of P:306 on centred keys times the global constant e^{-mstar}).
 * stats out: [tau, g, mstar, R_K, R_Q].
 * Options (flags; the switches of SURVEY 8(b)): WCO_NO_RECENTER skips "Recenter keys"
 * (P:300-301): kbar = 0, so R_K = max ||k_l|| and the kernel is on uncentred keys;
 * WCO_TAU_ONE skips Eq. 7: tau = 1, i.e. h_tau = exp(beta <.,.>) (P:306 at tau = 1).        */
/* ------------------------------------------------------------------------ */
#define WCO_TAU_ONE 2
#define WCO_NO_RECENTER 4
void wco_prologue(int64_t n, int32_t d, const double *K, int64_t mq, const double *Qrows,
                  double rq_given, double beta, double *kbar, double *stats, int32_t flags)
{
    for (int j = 0; j < d; ++j) {
        double s = 0.0;
        for (int64_t l = 0; l < n; ++l) s += K[l * d + j];
        kbar[j] = (flags & WCO_NO_RECENTER) ? 0.0 : s / (double)n;
    }
    double rk2 = 0.0;
    for (int64_t l = 0; l < n; ++l) {
        double s = 0.0;
        for (int j = 0; j < d; ++j) {
            double c = K[l * d + j] - kbar[j];
            s += c * c;
        }
        if (s > rk2) rk2 = s;
    }
    double rk = sqrt(rk2);
    double rq;
    if (rq_given >= 0.0) {
        rq = rq_given;
    } else {
        double rq2 = 0.0;
        for (int64_t i = 0; i < mq; ++i) {
            double s = 0.0;
            for (int j = 0; j < d; ++j) s += Qrows[i * d + j] * Qrows[i * d + j];
            if (s > rq2) rq2 = s;
        }
        rq = sqrt(rq2);
    }
    double tau = (flags & WCO_TAU_ONE) ? 1.0 : wco_temperature(beta, rq, rk, n);
    double g = beta / (tau * tau);
    stats[0] = tau;
    stats[1] = g;
    stats[2] = g * rk * rk;
    stats[3] = rk;
    stats[4] = rq;
}

/* h~(a, b) = exp(g <a - kbar, b - kbar> - mstar)  (P:306 kernel h_tau on
 * centred keys, scaled by e^{-mstar}; reading Z9/Z10).                     */
static double hker(int32_t d, const double *a, const double *b, const double *kbar,
                   double g, double mstar)
{
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += (a[j] - kbar[j]) * (b[j] - kbar[j]);
    return exp(g * s - mstar);
}

/* Pivot draw of Eq. 4, reading Z2: inverse CDF with strict '>':
 *   t = u * T,  s = min{ l : sum_{l'<=l} p_l' > t };  if rounding leaves no such l,
 *   s = the last l with p_l > 0.  The prefix is the plain sequential sum. */
static int64_t draw_pivot(int64_t n, const double *p, double T, double u)
{
    double t = u * T;
    double c = 0.0;
    for (int64_t l = 0; l < n; ++l) {
        c += p[l];
        if (c > t) return l;
    }
    for (int64_t l = n - 1; l >= 0; --l)
        if (p[l] > 0.0) return l;
    return -1;
}

/* One F-form round (see wco_select below) with pivot s at 0-based round i:
 * writes F[i,:], downdates p and zeroes p_s.                                */
static void fform_round(int64_t n, int32_t d, int32_t i, const double *K, const double *kbar,
                        double g, double mstar, double *F, double *p, int64_t s)
{
    double ps = p[s];
    double rs = sqrt(ps);
    const double *ks = K + s * d;
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < n; ++l) {
        double c = hker(d, K + l * d, ks, kbar, g, mstar);
        double acc = 0.0;
        for (int32_t j = 0; j < i; ++j) acc += F[(size_t)j * n + l] * F[(size_t)j * n + s];
        c = c - acc;
        double f = c / rs;
        F[(size_t)i * n + l] = f;
        double q = p[l] - f * f;
        p[l] = q > 0.0 ? q : 0.0;
    }
    p[s] = 0.0;
}

/* ------------------------------------------------------------------------ */
/* RPNys selection in the Cholesky-factor ("F") form, per unit.
 * Alg 1 maintains M = h(K_S,K_S)^{-1} and R = h(K_S,K); its
 * downdate delta = g^T R equals -F[i,:] where F is the partial Cholesky
 * factor of RP-Cholesky ("the two estimates are identical").
 * Round i (0-based), pivot s:
 *   c_l     = h~(k_l, k_s) - sum_{j<i} F[j,l] F[j,s]
 *   F[i,l]  = c_l / sqrt(p_s)                       (reading Z5: divide by the drawn p_s)
 *   p_l     = max(p_l - F[i,l]^2, 0)                (clamp, reading Z4)
 *   p_s     = 0
 * Exhaustion (reading Z3): stop with r_eff = i when T = sum p <= theta,
 *   theta = 1000 * r * 2^-52 * T0.
 * Outputs: S[r] (-1 past r_eff), *r_eff, F[r*n] (rows past r_eff zero) may be
 * NULL, p_out[n] final residual diagonal (may be NULL), trace[r+1] the value of
 * T at the start of each round (trace[r_eff] is the final T; may be NULL),
 * L[r*r] lower-triangular L[a][b] = F[b, s_a] for b <= a (reading Z6; may be NULL).
 * Returns 0, or -1 on allocation failure.                                   */
/* ------------------------------------------------------------------------ */
int wco_select(int64_t n, int32_t d, int32_t r, const double *K, const double *kbar,
               double g, double mstar, uint64_t seed, uint64_t unit,
               int32_t *S, int32_t *r_eff, double *F_out, double *p_out,
               double *trace, double *L)
{
    double *p = (double *)malloc(sizeof(double) * (size_t)n);
    double *F = (double *)calloc((size_t)r * (size_t)n, sizeof(double));
    if (!p || !F) { free(p); free(F); return -1; }

    /* p <- (h(k_l,k_l))_l   (Alg 1 "Compute kernel diagonal") */
    for (int64_t l = 0; l < n; ++l) p[l] = hker(d, K + l * d, K + l * d, kbar, g, mstar);
    double T0 = 0.0;
    for (int64_t l = 0; l < n; ++l) T0 += p[l];
    double theta = 1000.0 * (double)r * ldexp(1.0, -52) * T0;

    for (int i = 0; i < r; ++i) S[i] = -1;
    int32_t re = r;
    for (int32_t i = 0; i < r; ++i) {
        double T = 0.0;
        for (int64_t l = 0; l < n; ++l) T += p[l];
        if (trace) trace[i] = T;
        if (T <= theta) { re = i; break; }
        double u = wco_pivot_uniform(seed, (uint32_t)i, unit);
        int64_t s = draw_pivot(n, p, T, u);
        fform_round(n, d, i, K, kbar, g, mstar, F, p, s);
        S[i] = (int32_t)s;
    }
    if (re == r && trace) {
        double T = 0.0;
        for (int64_t l = 0; l < n; ++l) T += p[l];
        trace[r] = T;
    }
    *r_eff = re;
    if (L) {
        memset(L, 0, sizeof(double) * (size_t)r * (size_t)r);
        for (int a = 0; a < re; ++a)
            for (int b = 0; b <= a; ++b) L[a * r + b] = F[(size_t)b * n + S[a]];
    }
    if (F_out) memcpy(F_out, F, sizeof(double) * (size_t)r * (size_t)n);
    if (p_out) memcpy(p_out, p, sizeof(double) * (size_t)n);
    free(p);
    free(F);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Blocked ("accelerated") RPCholesky -- the oversampling mechanism the paper
 * names for future work (citing accelerated RPCholesky [epperly2024embrace]);
 * the algorithm is that cited work's block rejection sampler, reading Z22.
 * Per block, with i pivots accepted so far and residual diagonal p (T = sum p):
 *   1. draw b candidates s_0..s_{b-1} i.i.d. from p / T (Eq. 4 rule, draw_pivot),
 *      candidate c = (global candidate count) uses the pivot uniform of counter c,
 *      so b = 1 reproduces wco_select exactly;
 *   2. H = residual kernel on the candidates at the block start:
 *      H[a][a] = p[s_a];  H[a][c] = h~(k_sa, k_sc) - sum_{q<i} F[q,s_a] F[q,s_c];
 *   3. rejection, in candidate order j = 0..b-1 (stop once i + accepted = r):
 *      accept s_j iff  v_j * p[s_j] < H[j][j]   (v_j = accept uniform of counter c),
 *      where H[j][j] is the Schur complement after the candidates accepted before
 *      it in this block (so P(accept) = current residual / block-start residual;
 *      the first candidate is always accepted, a repeated candidate never);
 *      on acceptance H[a][c] -= H[a][j] H[j][c] / H[j][j] for a, c > j;
 *   4. the accepted pivots, in order, each run one F-form round (fform_round).
 * The accepted sequence has the law of sequential RPCholesky (rejection sampling
 * from the proposal p >= current residual); pivots for a given seed differ from
 * wco_select's unless b = 1.  Exhaustion (Z3) is tested at block starts.
 * Extra outputs: nblocks[1], ncand[1] (candidates drawn) -- may be NULL.      */
/* ------------------------------------------------------------------------ */
double wco_accept_uniform(uint64_t seed, uint32_t cand, uint64_t unit)
{
    uint32_t ctr[4] = {cand, (uint32_t)unit, (uint32_t)(unit >> 32), 0x41435054u};  /* 'ACPT' */
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    wco_philox4x32_10(ctr, key, x);
    double a = (double)(x[0] >> 5);
    double b = (double)(x[1] >> 6);
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}

int wco_select_blocked(int64_t n, int32_t d, int32_t r, int32_t b, const double *K, const double *kbar,
                       double g, double mstar, uint64_t seed, uint64_t unit,
                       int32_t *S, int32_t *r_eff, double *F_out, double *p_out, double *L,
                       int32_t *nblocks, int32_t *ncand)
{
    if (b < 1) return -1;
    double *p = (double *)malloc(sizeof(double) * (size_t)n);
    double *F = (double *)calloc((size_t)r * (size_t)n, sizeof(double));
    double *H = (double *)malloc(sizeof(double) * (size_t)b * (size_t)b);
    int64_t *cs = (int64_t *)malloc(sizeof(int64_t) * (size_t)b);
    int64_t *acc = (int64_t *)malloc(sizeof(int64_t) * (size_t)b);
    if (!p || !F || !H || !cs || !acc) { free(p); free(F); free(H); free(cs); free(acc); return -1; }

    for (int64_t l = 0; l < n; ++l) p[l] = hker(d, K + l * d, K + l * d, kbar, g, mstar);
    double T0 = 0.0;
    for (int64_t l = 0; l < n; ++l) T0 += p[l];
    double theta = 1000.0 * (double)r * ldexp(1.0, -52) * T0;

    for (int a = 0; a < r; ++a) S[a] = -1;
    int32_t i = 0, nb = 0;
    uint32_t c = 0;
    while (i < r) {
        double T = 0.0;
        for (int64_t l = 0; l < n; ++l) T += p[l];
        if (T <= theta) break;
        /* 1. candidates */
        for (int j = 0; j < b; ++j) cs[j] = draw_pivot(n, p, T, wco_pivot_uniform(seed, c + (uint32_t)j, unit));
        /* 2. block-start residual kernel on the candidates */
        for (int a = 0; a < b; ++a)
            for (int e = 0; e < b; ++e) {
                if (a == e) { H[a * b + a] = p[cs[a]]; continue; }
                double v = hker(d, K + cs[a] * d, K + cs[e] * d, kbar, g, mstar);
                double f = 0.0;
                for (int32_t q = 0; q < i; ++q) f += F[(size_t)q * n + cs[a]] * F[(size_t)q * n + cs[e]];
                H[a * b + e] = v - f;
            }
        /* 3. rejection */
        int na = 0;
        for (int j = 0; j < b && i + na < r; ++j) {
            int dup = 0;
            for (int a = 0; a < na; ++a) dup |= (acc[a] == cs[j]);
            double v = wco_accept_uniform(seed, c + (uint32_t)j, unit);
            if (dup || !(v * p[cs[j]] < H[j * b + j])) continue;
            acc[na++] = cs[j];
            double hjj = H[j * b + j];
            for (int a = j + 1; a < b; ++a)
                for (int e = j + 1; e < b; ++e) H[a * b + e] -= H[a * b + j] * H[j * b + e] / hjj;
        }
        c += (uint32_t)b;
        ++nb;
        /* 4. F-form rounds for the accepted pivots */
        for (int a = 0; a < na; ++a) {
            fform_round(n, d, i, K, kbar, g, mstar, F, p, acc[a]);
            S[i++] = (int32_t)acc[a];
        }
    }
    *r_eff = i;
    if (nblocks) *nblocks = nb;
    if (ncand) *ncand = (int32_t)c;
    if (L) {
        memset(L, 0, sizeof(double) * (size_t)r * (size_t)r);
        for (int a = 0; a < i; ++a)
            for (int e = 0; e <= a; ++e) L[a * r + e] = F[(size_t)e * n + S[a]];
    }
    if (F_out) memcpy(F_out, F, sizeof(double) * (size_t)r * (size_t)n);
    if (p_out) memcpy(p_out, p, sizeof(double) * (size_t)n);
    free(p); free(F); free(H); free(cs); free(acc);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Literal Algorithm 1, M/R form, same pivot stream and draw rule,
 * same exhaustion and clamp readings.  Cross-check of wco_select.
 * Reading Z1: the printed "if i > 0" means "if S is non-empty": in the first
 * round g = (-1)/sqrt(p_s).
 *   g_[i-1] <- M_[i-1],[i-1] R_[i-1],s ;  g_i <- -1 ;  g_[i] <- g_[i]/sqrt(p_s)
 *   M <- M + g g^T ;  R_i <- h(k_s, K) ;  delta <- g^T R ;  p <- p - delta^2 ; p_s <- 0
 * Returns W = M R (r x n).  M[r*r], R[r*n], W[r*n], p_out[n] may be NULL.  */
/* ------------------------------------------------------------------------ */
int wco_select_mr(int64_t n, int32_t d, int32_t r, const double *K, const double *kbar,
                  double g, double mstar, uint64_t seed, uint64_t unit,
                  int32_t *S, int32_t *r_eff, double *M_out, double *R_out, double *W_out,
                  double *p_out)
{
    double *p = (double *)malloc(sizeof(double) * (size_t)n);
    double *M = (double *)calloc((size_t)r * r, sizeof(double));
    double *R = (double *)calloc((size_t)r * (size_t)n, sizeof(double));
    double *gv = (double *)calloc((size_t)r, sizeof(double));
    if (!p || !M || !R || !gv) { free(p); free(M); free(R); free(gv); return -1; }

    for (int64_t l = 0; l < n; ++l) p[l] = hker(d, K + l * d, K + l * d, kbar, g, mstar);
    double T0 = 0.0;
    for (int64_t l = 0; l < n; ++l) T0 += p[l];
    double theta = 1000.0 * (double)r * ldexp(1.0, -52) * T0;

    for (int i = 0; i < r; ++i) S[i] = -1;
    int32_t re = r;
    for (int32_t i = 0; i < r; ++i) {
        double T = 0.0;
        for (int64_t l = 0; l < n; ++l) T += p[l];
        if (T <= theta) { re = i; break; }
        double u = wco_pivot_uniform(seed, (uint32_t)i, unit);
        int64_t s = draw_pivot(n, p, T, u);
        double ps = p[s];
        /* g_[i-1] <- M_[i-1],[i-1] R_[i-1],s */
        for (int a = 0; a < i; ++a) {
            double acc = 0.0;
            for (int b = 0; b < i; ++b) acc += M[a * r + b] * R[(size_t)b * n + s];
            gv[a] = acc;
        }
        gv[i] = -1.0;
        double rs = sqrt(ps);
        for (int a = 0; a <= i; ++a) gv[a] = gv[a] / rs;
        /* M <- M + g g^T */
        for (int a = 0; a <= i; ++a)
            for (int b = 0; b <= i; ++b) M[a * r + b] += gv[a] * gv[b];
        /* R_i <- h(k_s, K) */
        const double *ks = K + s * d;
        for (int64_t l = 0; l < n; ++l) R[(size_t)i * n + l] = hker(d, ks, K + l * d, kbar, g, mstar);
        /* delta <- g^T R ; p <- p - delta^2 (clamped) ; p_s <- 0 */
        for (int64_t l = 0; l < n; ++l) {
            double delta = 0.0;
            for (int a = 0; a <= i; ++a) delta += gv[a] * R[(size_t)a * n + l];
            double q = p[l] - delta * delta;
            p[l] = q > 0.0 ? q : 0.0;
        }
        p[s] = 0.0;
        S[i] = (int32_t)s;
    }
    *r_eff = re;
    if (W_out) {
        for (int a = 0; a < r; ++a)
            for (int64_t l = 0; l < n; ++l) {
                double acc = 0.0;
                for (int b = 0; b < re; ++b) acc += M[a * r + b] * R[(size_t)b * n + l];
                W_out[(size_t)a * n + l] = acc;
            }
    }
    if (M_out) memcpy(M_out, M, sizeof(double) * (size_t)r * r);
    if (R_out) memcpy(R_out, R, sizeof(double) * (size_t)r * (size_t)n);
    if (p_out) memcpy(p_out, p, sizeof(double) * (size_t)n);
    free(p); free(M); free(R); free(gv);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Nystrom weights applied to [V, 1_n] (P:156-158 weights W = h(K_S,K_S)^+ h(K_S,K);
 * Alg 2 "Compress values" V_S <- W V, w <- W 1_n).  Reading Z8: with the
 * exhaustion rule H~_SS is positive definite, so the inverse is taken by a
 * textbook Cholesky factorisation; failure returns -2 (never pseudo-inverted).
 * The kernel is h~ (the e^{-mstar} factor cancels in W).
 *   Y[a][c] = sum_l h~(k_{s_a}, k_l) [V,1][l][c]
 *   X = H~_SS^{-1} Y                      X: [r][d+1], rows >= r_eff zero. */
/* ------------------------------------------------------------------------ */
int wco_weights(int64_t n, int32_t d, int32_t r, const double *K, const double *V,
                const int32_t *S, int32_t r_eff, const double *kbar, double g, double mstar,
                double *X)
{
    int32_t q = r_eff;
    int32_t dc = d + 1;
    memset(X, 0, sizeof(double) * (size_t)r * dc);
    if (q <= 0) return 0;
    double *H = (double *)malloc(sizeof(double) * (size_t)q * q);
    double *Lc = (double *)calloc((size_t)q * q, sizeof(double));
    double *Y = (double *)calloc((size_t)q * dc, sizeof(double));
    if (!H || !Lc || !Y) { free(H); free(Lc); free(Y); return -1; }
    for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b)
            H[a * q + b] = hker(d, K + (int64_t)S[a] * d, K + (int64_t)S[b] * d, kbar, g, mstar);
#pragma omp parallel for schedule(static)
    for (int a = 0; a < q; ++a) {
        const double *ks = K + (int64_t)S[a] * d;
        for (int64_t l = 0; l < n; ++l) {
            double h = hker(d, ks, K + l * d, kbar, g, mstar);
            for (int c = 0; c < d; ++c) Y[a * dc + c] += h * V[l * d + c];
            Y[a * dc + d] += h;
        }
    }
    /* textbook Cholesky H = Lc Lc^T */
    for (int j = 0; j < q; ++j) {
        double s = H[j * q + j];
        for (int k = 0; k < j; ++k) s -= Lc[j * q + k] * Lc[j * q + k];
        if (!(s > 0.0)) { free(H); free(Lc); free(Y); return -2; }
        double ljj = sqrt(s);
        Lc[j * q + j] = ljj;
        for (int i = j + 1; i < q; ++i) {
            double t = H[i * q + j];
            for (int k = 0; k < j; ++k) t -= Lc[i * q + k] * Lc[j * q + k];
            Lc[i * q + j] = t / ljj;
        }
    }
    /* forward substitution Lc Z = Y, then back substitution Lc^T X = Z */
    for (int c = 0; c < dc; ++c) {
        for (int a = 0; a < q; ++a) {
            double t = Y[a * dc + c];
            for (int b = 0; b < a; ++b) t -= Lc[a * q + b] * Y[b * dc + c];
            Y[a * dc + c] = t / Lc[a * q + a];
        }
        for (int a = q - 1; a >= 0; --a) {
            double t = Y[a * dc + c];
            for (int b = a + 1; b < q; ++b) t -= Lc[b * q + a] * X[b * dc + c];
            X[a * dc + c] = t / Lc[a * q + a];
        }
    }
    free(H); free(Lc); free(Y);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Weighted coreset attention, Alg 3 with X = [V_S, w]:
 *   a_is = beta <q_i, k_s>   (K_S uncentred, Alg 2 "K_S <- K_S + kbar")
 *   P_is = exp(a_is - max_s a_is)          (row shift cancels in the ratio)
 *   num = sum_s P_is V_S[s],  den = sum_s P_is w_s
 *   o = num/den where den > 0 else 0;  O = clip(o, vmin, vmax)  (reading Z14/Z15)
 * KS [r][d], X [r][d+1], only the first r_eff rows are used.               */
/* ------------------------------------------------------------------------ */
void wco_attend(int64_t m, int32_t d, int32_t r, const double *Q, const double *KS,
                const double *X, int32_t r_eff, double beta, const double *vmin,
                const double *vmax, int32_t clip, double *O)
{
    int32_t dc = d + 1;
#pragma omp parallel
    {
        double *a = (double *)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            const double *q = Q + i * d;
            double mu = -INFINITY;
            for (int s = 0; s < r_eff; ++s) {
                double t = 0.0;
                for (int j = 0; j < d; ++j) t += q[j] * KS[s * d + j];
                a[s] = beta * t;
                if (a[s] > mu) mu = a[s];
            }
            double den = 0.0;
            for (int s = 0; s < r_eff; ++s) den += exp(a[s] - mu) * X[s * dc + d];
            for (int c = 0; c < d; ++c) {
                double num = 0.0;
                for (int s = 0; s < r_eff; ++s) num += exp(a[s] - mu) * X[s * dc + c];
                double o = den > 0.0 ? num / den : 0.0;
                if (clip) {
                    if (o < vmin[c]) o = vmin[c];
                    if (o > vmax[c]) o = vmax[c];
                }
                O[i * d + c] = o;
            }
        }
        free(a);
    }
}

/* ------------------------------------------------------------------------ */
/* Exact softmax attention, Eq. 1, row max shifted (exact by the
 * per-row cancellation of P:264-271).                                        */
/* ------------------------------------------------------------------------ */
void wco_exact_attention(int64_t m, int64_t n, int32_t d, const double *Q, const double *K,
                         const double *V, double beta, double *O)
{
#pragma omp parallel
    {
        double *a = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            const double *q = Q + i * d;
            double mu = -INFINITY;
            for (int64_t l = 0; l < n; ++l) {
                double t = 0.0;
                for (int j = 0; j < d; ++j) t += q[j] * K[l * d + j];
                a[l] = beta * t;
                if (a[l] > mu) mu = a[l];
            }
            double den = 0.0;
            for (int64_t l = 0; l < n; ++l) den += exp(a[l] - mu);
            for (int c = 0; c < d; ++c) {
                double num = 0.0;
                for (int64_t l = 0; l < n; ++l) num += exp(a[l] - mu) * V[l * d + c];
                O[i * d + c] = num / den;
            }
        }
        free(a);
    }
}

/* ------------------------------------------------------------------------ */
/* Algorithm 4 WildCat over a batch of units, B = 1 bin.
 * Layouts: Q,O [batch][hq][m][d];  K,V [batch][hkv][n][d];  unit u = b*hkv + h.
 * Query head h uses unit (b, h / (hq/hkv)) (reading Z11, GQA).
 * rq < 0 -> R_Q from the unit's query group (Alg 4).
 * Optional outputs (may be NULL): S [units][r], r_eff [units],
 * stats [units][5] = tau,g,mstar,R_K,R_Q, X [units][r][d+1].
 * block > 1 selects with the blocked variant (wco_select_blocked, reading Z22).
 * unit0: these units are units [unit0, unit0 + batch*hkv) of a larger batch -- unit u draws
 * the Philox stream of unit id unit0 + u (reading Z2; PAR2 of SURVEY 8(e)).
 * flags: WCO_TAU_ONE / WCO_NO_RECENTER (see wco_prologue).
 * Returns 0, or the first nonzero sub-status.                               */
/* ------------------------------------------------------------------------ */
int wco_forward(int32_t batch, int32_t hq, int32_t hkv, int64_t m, int64_t n, int32_t d,
                int32_t r, double beta, double rq, uint64_t seed, int32_t clip, int32_t block,
                const double *Q, const double *K, const double *V, double *O,
                int32_t *S_out, int32_t *reff_out, double *stats_out, double *X_out,
                uint64_t unit0, int32_t flags)
{
    int32_t group = hq / hkv;
    int32_t dc = d + 1;
    double *kbar = (double *)malloc(sizeof(double) * d);
    double *X = (double *)malloc(sizeof(double) * (size_t)r * dc);
    double *KS = (double *)malloc(sizeof(double) * (size_t)r * d);
    double *vmin = (double *)malloc(sizeof(double) * d);
    double *vmax = (double *)malloc(sizeof(double) * d);
    int32_t *S = (int32_t *)malloc(sizeof(int32_t) * r);
    if (!kbar || !X || !KS || !vmin || !vmax || !S) return -1;
    int status = 0;
    for (int32_t b = 0; b < batch && status == 0; ++b) {
        for (int32_t h = 0; h < hkv && status == 0; ++h) {
            uint64_t u = (uint64_t)b * hkv + h;
            const double *Ku = K + (size_t)u * n * d;
            const double *Vu = V + (size_t)u * n * d;
            const double *Qg = Q + ((size_t)b * hq + (size_t)h * group) * m * d;
            /* (vmin, vmax): columnwise range of V, Alg 4 */
            for (int c = 0; c < d; ++c) {
                double lo = Vu[c], hi = Vu[c];
                for (int64_t l = 1; l < n; ++l) {
                    double v = Vu[l * d + c];
                    if (v < lo) lo = v;
                    if (v > hi) hi = v;
                }
                vmin[c] = lo;
                vmax[c] = hi;
            }
            double st[5];
            wco_prologue(n, d, Ku, (int64_t)group * m, Qg, rq, beta, kbar, st, flags);
            int32_t re = 0;
            const uint64_t uid = unit0 + u;  /* global unit id of the Philox stream */
            if (block > 1)
                status = wco_select_blocked(n, d, r, block, Ku, kbar, st[1], st[2], seed, uid, S, &re, NULL, NULL,
                                            NULL, NULL, NULL);
            else
                status = wco_select(n, d, r, Ku, kbar, st[1], st[2], seed, uid, S, &re, NULL, NULL, NULL, NULL);
            if (status) break;
            status = wco_weights(n, d, r, Ku, Vu, S, re, kbar, st[1], st[2], X);
            if (status) break;
            for (int a = 0; a < r; ++a)
                for (int j = 0; j < d; ++j) KS[a * d + j] = a < re ? Ku[(int64_t)S[a] * d + j] : 0.0;
            for (int32_t hh = 0; hh < group; ++hh) {
                size_t qoff = ((size_t)b * hq + (size_t)h * group + hh) * m * d;
                wco_attend(m, d, r, Q + qoff, KS, X, re, beta, vmin, vmax, clip, O + qoff);
            }
            if (S_out) memcpy(S_out + (size_t)u * r, S, sizeof(int32_t) * r);
            if (reff_out) reff_out[u] = re;
            if (stats_out) memcpy(stats_out + (size_t)u * 5, st, sizeof(st));
            if (X_out) memcpy(X_out + (size_t)u * r * dc, X, sizeof(double) * (size_t)r * dc);
        }
    }
    free(kbar); free(X); free(KS); free(vmin); free(vmax); free(S);
    return status;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 4 WildCat with B > 1 bins (Alg 2 CompressKV).
 * Readings (Z12, Z13, Z23):
 *   - kbar is the row mean over ALL n keys of the unit and the recentring is global;
 *     R_Q and the value range are over the unit's full query group / full V;
 *   - bins are contiguous: bin b = rows [b nb, (b+1) nb) with nb = floor(n / B), and the last bin
 *     also takes the n - B nb remainder rows (the paper's "evenly divide (or reshape)"; Z13);
 *   - per bin: R_K^b = max ||k_l - kbar|| over the bin, tau_b = Eq. 7 with n_b the bin's
 *     size (Z12), RPNys on the bin's centred keys at rank rb = min(ceil(r/B), nb) (Z13), with the
 *     Philox stream of unit id u*B + b (Z23), sequential or blocked (block > 1);
 *   - the bin coresets are concatenated in bin order with their valid rows only, so
 *     the unit's coreset is r_eff = sum_b r_eff_b rows; V_S, w from each bin's own Nystrom
 *     weights over its own keys (W block diagonal); then Alg 3 over the whole coreset.
 * Outputs (may be NULL): S [units][B*rb] unit-level key indices, -1 past r_eff;
 * r_eff [units]; binstats [units][B][5] = tau_b, g_b, mstar_b, R_K^b, R_Q;
 * X [units][B*rb][d+1] (rows past r_eff zero).  Returns -2 unless 1 <= B <= min(r, n).   */
/* ------------------------------------------------------------------------ */
/* CompressKV (Alg 2) of ONE unit with B >= 1 contiguous bins: the per-unit body of
 * wco_forward_binned, shared with wco_compress_kv.  Ku, Vu [n][d]; Qg [mq][d] the unit's query rows
 * (for R_Q; unused when rq >= 0).  Outputs: S [B*rb] unit-level key indices (-1 past tot),
 * KS [B*rb][d], X [B*rb][d+1] (rows past tot zero), *tot = r_eff, binstats [B][5] (may be NULL).
 * Requires 1 <= B <= n (checked by the callers).                                                */
static int compress_unit(int64_t n, int32_t d, int32_t r, int32_t bins, int32_t block, double beta,
                         double rq, uint64_t seed, uint64_t u, const double *Ku, const double *Vu,
                         int64_t mq, const double *Qg, int32_t *S, double *KS, double *X,
                         int32_t *tot_out, double *binstats, int32_t flags)
{
    const int64_t nb = n / bins;
    int32_t rb = (r + bins - 1) / bins;
    if (rb > nb) rb = (int32_t)nb;
    const int32_t R = bins * rb, dc = d + 1;
    double *kbar = (double *)malloc(sizeof(double) * d);
    double *Xb = (double *)malloc(sizeof(double) * (size_t)rb * dc);
    int32_t *Sb = (int32_t *)malloc(sizeof(int32_t) * rb);
    if (!kbar || !Xb || !Sb) {
        free(kbar); free(Xb); free(Sb);
        return -1;
    }
    int status = 0;
    double st[5];
    wco_prologue(n, d, Ku, mq, Qg, rq, beta, kbar, st, flags);  /* global kbar, R_Q */
    const double rqu = st[4];
    memset(X, 0, sizeof(double) * (size_t)R * dc);
    memset(KS, 0, sizeof(double) * (size_t)R * d);
    for (int a = 0; a < R; ++a) S[a] = -1;
    int32_t tot = 0;
    for (int32_t b = 0; b < bins && status == 0; ++b) {
        const double *Kb = Ku + (size_t)b * nb * d;
        const double *Vb = Vu + (size_t)b * nb * d;
        const int64_t nbb = (b == bins - 1) ? n - (int64_t)(bins - 1) * nb : nb;  /* last bin: + remainder (Z13) */
        double rk2 = 0.0;  /* R_K^b over the bin's centred keys */
        for (int64_t l = 0; l < nbb; ++l) {
            double s2 = 0.0;
            for (int j = 0; j < d; ++j) {
                double c = Kb[l * d + j] - kbar[j];
                s2 += c * c;
            }
            if (s2 > rk2) rk2 = s2;
        }
        const double rk = sqrt(rk2);
        const double tau = (flags & WCO_TAU_ONE) ? 1.0 : wco_temperature(beta, rqu, rk, nbb);  /* Z12: n_b */
        const double g = beta / (tau * tau), mstar = g * rk * rk;
        int32_t re = 0;
        const uint64_t ub = u * (uint64_t)bins + (uint64_t)b;  /* Z23 */
        if (block > 1)
            status = wco_select_blocked(nbb, d, rb, block, Kb, kbar, g, mstar, seed, ub, Sb, &re, NULL, NULL,
                                        NULL, NULL, NULL);
        else
            status = wco_select(nbb, d, rb, Kb, kbar, g, mstar, seed, ub, Sb, &re, NULL, NULL, NULL, NULL);
        if (status) break;
        status = wco_weights(nbb, d, rb, Kb, Vb, Sb, re, kbar, g, mstar, Xb);
        if (status) break;
        for (int a = 0; a < re; ++a) {  /* concatenate the bin's valid rows */
            S[tot + a] = (int32_t)(b * nb + Sb[a]);
            memcpy(KS + (size_t)(tot + a) * d, Kb + (size_t)Sb[a] * d, sizeof(double) * d);
            memcpy(X + (size_t)(tot + a) * dc, Xb + (size_t)a * dc, sizeof(double) * dc);
        }
        tot += re;
        if (binstats) {
            double *bs = binstats + (size_t)b * 5;
            bs[0] = tau; bs[1] = g; bs[2] = mstar; bs[3] = rk; bs[4] = rqu;
        }
    }
    *tot_out = tot;
    free(kbar); free(Xb); free(Sb);
    return status;
}

/* Columnwise range of V over rows [0, n) (Alg 4). */
static void value_range(int64_t n, int32_t d, const double *Vu, double *vmin, double *vmax)
{
    for (int c = 0; c < d; ++c) {
        double lo = Vu[c], hi = Vu[c];
        for (int64_t l = 1; l < n; ++l) {
            double v = Vu[l * d + c];
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
        vmin[c] = lo;
        vmax[c] = hi;
    }
}

int wco_forward_binned(int32_t batch, int32_t hq, int32_t hkv, int64_t m, int64_t n, int32_t d,
                       int32_t r, int32_t bins, double beta, double rq, uint64_t seed, int32_t clip,
                       int32_t block, const double *Q, const double *K, const double *V, double *O,
                       int32_t *S_out, int32_t *reff_out, double *binstats_out, double *X_out,
                       uint64_t unit0, int32_t flags)
{
    if (bins < 1 || bins > n || bins > r) return -2;
    const int64_t nb = n / bins;
    int32_t rb = (r + bins - 1) / bins;
    if (rb > nb) rb = (int32_t)nb;
    const int32_t R = bins * rb, dc = d + 1, group = hq / hkv;
    double *X = (double *)malloc(sizeof(double) * (size_t)R * dc);
    double *KS = (double *)malloc(sizeof(double) * (size_t)R * d);
    double *vmin = (double *)malloc(sizeof(double) * d);
    double *vmax = (double *)malloc(sizeof(double) * d);
    int32_t *S = (int32_t *)malloc(sizeof(int32_t) * R);
    if (!X || !KS || !vmin || !vmax || !S) return -1;
    int status = 0;
    for (int32_t bt = 0; bt < batch && status == 0; ++bt) {
        for (int32_t h = 0; h < hkv && status == 0; ++h) {
            uint64_t u = (uint64_t)bt * hkv + h;
            const double *Ku = K + (size_t)u * n * d;
            const double *Vu = V + (size_t)u * n * d;
            const double *Qg = Q + ((size_t)bt * hq + (size_t)h * group) * m * d;
            value_range(n, d, Vu, vmin, vmax);  /* value range over the full V */
            int32_t tot = 0;
            status = compress_unit(n, d, r, bins, block, beta, rq, seed, unit0 + u, Ku, Vu, (int64_t)group * m, Qg,
                                   S, KS, X, &tot, binstats_out ? binstats_out + (size_t)u * bins * 5 : NULL, flags);
            if (status) break;
            for (int32_t hh = 0; hh < group; ++hh) {
                size_t qoff = ((size_t)bt * hq + (size_t)h * group + hh) * m * d;
                wco_attend(m, d, R, Q + qoff, KS, X, tot, beta, vmin, vmax, clip, O + qoff);
            }
            if (S_out) memcpy(S_out + (size_t)u * R, S, sizeof(int32_t) * R);
            if (reff_out) reff_out[u] = tot;
            if (X_out) memcpy(X_out + (size_t)u * R * dc, X, sizeof(double) * (size_t)R * dc);
        }
    }
    free(X); free(KS); free(vmin); free(vmax); free(S);
    return status;
}

/* ------------------------------------------------------------------------ */
/* KV-cache compression ("prefill phase"; E3 protocol P:667-669).
 * Per unit u = b*hkv + h with keys/values K, V [n][d]:
 *   - the first keep_first and the last keep_last tokens are retained exactly ("retain the first
 *     and last 32 context tokens and compress the remaining tokens");
 *   - the middle n_mid = n - keep_first - keep_last tokens are compressed by CompressKV (Alg 2,
 *     P:297-313) with rank r and B <= n_mid bins, exactly as wco_forward_binned does for a
 *     unit whose keys are the middle slice (its own kbar and R_K; R_Q from the unit's query rows
 *     Q [m per q-head] of the prompt, or rq >= 0; Philox unit id u, sub-unit u*B + b);
 *   - reading Z24: the cache is the union of exact and compressed entries, each entry a key row
 *     and an [value | weight] row: a retained token l contributes (k_l, [v_l, 1]), a coreset key
 *     s contributes (k_s, [V_S, w]_s) -- so WtdAttn (Alg 3) over the cache sums the
 *     exact terms of the retained tokens and the Nystrom estimate of the middle's terms under one
 *     softmax shift (the estimate is of the unnormalised sums, so the two add);
 *   - the clip range (vmin, vmax) is over all n values ("full V").
 * Cache rows per unit, capacity C = keep_first + keep_last + R (R = B*rb, rb = min(ceil(r/B),
 * n_mid/B); R = 0 when n_mid = 0): [first keep_first tokens | last keep_last tokens | r_eff
 * coreset rows in the order of Alg 2], zero rows after; c_eff = keep_first + keep_last + r_eff.
 * Outputs: KC [units][C][d], XC [units][C][d+1], c_eff [units], vmin/vmax [units][d],
 * S [units][R] (global token indices of the coreset, -1 past r_eff; may be NULL).
 * Returns -2 on an invalid split (keep_* < 0, n_mid < 0, n_mid > 0 with B > n_mid or B > r).   */
/* ------------------------------------------------------------------------ */
int wco_compress_kv(int32_t batch, int32_t hq, int32_t hkv, int64_t m, int64_t n, int32_t d, int32_t r,
                    int32_t bins, int32_t block, int32_t keep_first, int32_t keep_last, double beta, double rq,
                    uint64_t seed, const double *Q, const double *K, const double *V, double *KC, double *XC,
                    int32_t *c_eff, double *vmin_out, double *vmax_out, int32_t *S_out, uint64_t unit0,
                    int32_t flags)
{
    const int64_t nmid = n - keep_first - keep_last;
    if (keep_first < 0 || keep_last < 0 || nmid < 0) return -2;
    if (nmid > 0 && (bins < 1 || bins > nmid || bins > r || r < 1)) return -2;
    int32_t R = 0;
    if (nmid > 0) {
        int32_t rb = (r + bins - 1) / bins;
        if (rb > nmid / bins) rb = (int32_t)(nmid / bins);
        R = bins * rb;
    }
    const int32_t kept = keep_first + keep_last, C = kept + R, dc = d + 1, group = hq / hkv;
    double *X = (double *)malloc(sizeof(double) * (size_t)(R > 0 ? R : 1) * dc);
    double *KS = (double *)malloc(sizeof(double) * (size_t)(R > 0 ? R : 1) * d);
    int32_t *S = (int32_t *)malloc(sizeof(int32_t) * (size_t)(R > 0 ? R : 1));
    if (!X || !KS || !S) return -1;
    int status = 0;
    for (int32_t bt = 0; bt < batch && status == 0; ++bt) {
        for (int32_t h = 0; h < hkv && status == 0; ++h) {
            const uint64_t u = (uint64_t)bt * hkv + h;
            const double *Ku = K + (size_t)u * n * d;
            const double *Vu = V + (size_t)u * n * d;
            const double *Qg = Q + ((size_t)bt * hq + (size_t)h * group) * m * d;
            double *KCu = KC + (size_t)u * C * d;
            double *XCu = XC + (size_t)u * C * dc;
            value_range(n, d, Vu, vmin_out + (size_t)u * d, vmax_out + (size_t)u * d);
            memset(KCu, 0, sizeof(double) * (size_t)C * d);
            memset(XCu, 0, sizeof(double) * (size_t)C * dc);
            for (int32_t a = 0; a < kept; ++a) {  /* retained tokens: (k_l, [v_l, 1]) */
                const int64_t l = a < keep_first ? a : n - keep_last + (a - keep_first);
                memcpy(KCu + (size_t)a * d, Ku + (size_t)l * d, sizeof(double) * d);
                memcpy(XCu + (size_t)a * dc, Vu + (size_t)l * d, sizeof(double) * d);
                XCu[(size_t)a * dc + d] = 1.0;
            }
            int32_t tot = 0;
            if (nmid > 0) {
                status = compress_unit(nmid, d, r, bins, block, beta, rq, seed, unit0 + u,
                                       Ku + (size_t)keep_first * d, Vu + (size_t)keep_first * d, (int64_t)group * m,
                                       Qg, S, KS, X, &tot, NULL, flags);
                if (status) break;
                memcpy(KCu + (size_t)kept * d, KS, sizeof(double) * (size_t)tot * d);
                memcpy(XCu + (size_t)kept * dc, X, sizeof(double) * (size_t)tot * dc);
            }
            c_eff[u] = kept + tot;
            if (S_out)
                for (int32_t a = 0; a < R; ++a) S_out[(size_t)u * R + a] = a < tot ? S[a] + keep_first : -1;
        }
    }
    free(X); free(KS); free(S);
    return status;
}

int wco_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void wco_set_num_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
