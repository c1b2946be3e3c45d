/*
 * oracle/pcdn_oracle.c -- plain, slow, single-threaded fp64 CPU oracle of PCDN
 * (Bian, Li, Liu, Yang, arXiv:1306.4080; "PAPER.md" below is /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_1306_4080_b200/),
 * and neither side includes or imports the other.
 *
 * It follows the paper's algorithm step by step, in the paper's order and notation:
 *   Eq.1  F_c(w) = c sum_i phi(w; x_i, y_i) + ||w||_1
 *   Eq.2  phi_log = log(1 + e^{-y w'x})
 *   Eq.3  phi_svm = max(0, 1 - y w'x)^2
 *   Eq.5  closed-form 1-D Newton direction
 *   Eq.6/7 Armijo rule and Delta
 *   Eq.8  random disjoint partition into b = ceil(n/P) bundles
 *   Eq.9/10 P-dim direction = sum_j d(w;j) e_j
 *   Alg.3 PCDN outer/inner loop
 *   Alg.4 + Eq.12 line search from retained w'x_i and d'x_i
 *   Eq.13 logistic gradient / Hessian diagonal
 *   App.A.2 L2-SVM generalized Hessian, nu = 1e-12
 *   Eq.14 relative function value difference
 *   Alg.1 CDN (separately coded, for the P=1 reduction)
 *   Alg.2 SCDN (Shotgun CDN, NEXT #3; synchronous reading Z27)
 *   Lasso (NEXT #4; "easily extended to ... Lasso"): the squared loss
 *   phi = (t_i - w'x_i)^2 with real targets t (reading Z26): G = 2(z - t), H = 2, the line-search
 *   summand (t - z - a dx)^2 - (t - z)^2 = a dx (a dx + 2(z - t)).
 *   Elastic net (NEXT #4; "easily extended to ... elastic net"): the separable
 *   term ||w||_1 + (mu/2)||w||_2^2, mu >= 0 (mu = 0: the paper's problem).  Reading Z25: the
 *   smooth part becomes L(w) + (mu/2)||w||^2, so g_j, h_j gain mu w_j, mu (Eq.5 unchanged in form),
 *   Delta (Eq.7) uses them, and the line search's L1 term gains (mu/2)((w_j+a d_j)^2 - w_j^2).
 * Readings where the paper is silent/ambiguous are DESIGN.md Z1..Z24 (cited inline).
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py against
 * closed forms, brute force, finite differences, an independent scipy solver and the
 * paper's invariants, except the exact multi-step iterate trajectory on general data,
 * which is "parity unpinned" beyond those invariants (Oracle pins).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no FMA contraction, no OpenMP, no SIMD
 * intrinsics).
 */
#include <math.h>
#include <time.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_OK 0
#define ORA_ERR_INVALID 1
#define ORA_BUDGET 2
#define ORA_ERR_NUMERIC 3

#define ORA_LOSS_LOGISTIC 0
#define ORA_LOSS_L2SVM 1
#define ORA_LOSS_SQUARED 2   /* Lasso / elastic-net regression (reading Z26) */

typedef struct {
    int64_t s, n;
    const int64_t *col_ptr;   /* CSC, n+1 */
    const int32_t *row_idx;   /* nnz, ascending per column */
    const float *val;         /* nnz */
    const int8_t *y;          /* s, +-1 */
    double c;                 /* regularization weight, Eq.1 */
    int32_t loss;             /* ORA_LOSS_* */
    int32_t qmax;             /* line-search cap (Z10) */
    double sigma, beta, gamma, nu;   /* Armijo constants, nu */
    double mu;                /* elastic-net weight (reading Z25; 0 = the paper's problem) */
    const double *t;          /* s real targets of the squared loss (Z26); NULL otherwise */
} ora_prob;

/* ------------------------------------------------------------------------------ */
/* Z2: random disjoint partition.  pi_k is a keyed pseudo-random permutation of    */
/* {0..n-1}: an 8-round balanced Feistel network on 2*hb bits with cycle walking.   */
/* Bundle t of outer iteration k is pi_k[tP : min((t+1)P, n)] (Eq.8).              */
/* ------------------------------------------------------------------------------ */
uint64_t ora_mix64(uint64_t x)
{
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

static int ora_half_bits(int64_t n)
{
    int bits = 0;                     /* ceil(log2(n)) */
    while (bits < 63 && ((int64_t)1 << bits) < n) bits++;
    int hb = (bits + 1) / 2;
    return hb < 1 ? 1 : hb;
}

int64_t ora_perm_at(uint64_t seed, int64_t k, int64_t n, int64_t t)
{
    int hb = ora_half_bits(n);
    uint64_t mask = ((uint64_t)1 << hb) - 1;
    uint64_t base = ora_mix64(seed ^ 0x6A09E667F3BCC909ULL);
    uint64_t kk = ora_mix64(base ^ (uint64_t)k);
    uint64_t key[8];
    for (int r = 0; r < 8; r++) key[r] = ora_mix64(kk + (uint64_t)(r + 1) * 0x9E3779B97F4A7C15ULL);
    uint64_t x = (uint64_t)t;
    do {
        uint64_t L = x >> hb, R = x & mask;
        for (int r = 0; r < 8; r++) {
            uint64_t nl = R;
            uint64_t nr = L ^ (ora_mix64(key[r] ^ R) & mask);
            L = nl;
            R = nr;
        }
        x = (L << hb) | R;
    } while (x >= (uint64_t)n);
    return (int64_t)x;
}

void ora_permutation(uint64_t seed, int64_t k, int64_t n, int32_t *out)
{
    for (int64_t t = 0; t < n; t++) out[t] = (int32_t)ora_perm_at(seed, k, n, t);
}

/* ------------------------------------------------------------------------------ */
/* Losses (Eq.2, Eq.3) and their per-sample derivative factors (Eq.13, App. A.2).  */
/* ------------------------------------------------------------------------------ */
static double softplus(double t)  /* log(1+e^t), overflow-safe (Z19) */
{
    return (t > 0 ? t : 0.0) + log1p(exp(-fabs(t)));
}

/* phi as a function of the margin m = y w'x */
double ora_phi(int loss, double m)
{
    if (loss == ORA_LOSS_LOGISTIC) return softplus(-m);           /* Eq.2 */
    double b = 1.0 - m;                                            /* Eq.3 */
    return b > 0 ? b * b : 0.0;
}

/* sigma(t) = 1/(1+e^-t) evaluated without overflow; returns sigma(m) and sigma(-m) */
static void sig_pair(double m, double *sm, double *snm)
{
    if (m >= 0) {
        double e = exp(-m);
        *sm = 1.0 / (1.0 + e);
        *snm = e / (1.0 + e);
    } else {
        double e = exp(m);
        *sm = e / (1.0 + e);
        *snm = 1.0 / (1.0 + e);
    }
}

/* Per-sample factors so that grad_j L = c sum_i x_ij G_i and hess_jj L = c sum_i x_ij^2 H_i.
 *  LR  (Eq.13): G = (tau(m)-1) y = -sigma(-m) y,  H = tau(1-tau) = sigma(m) sigma(-m)
 *  SVM (App.A.2; gradient derived from Eq.3, reading Z5):
 *       b = 1 - y z; i in I(w) iff b > 0 (strict): G = -2 y b, H = 2; else 0, 0 */
void ora_GH(int loss, double z, int y, double *G, double *H)
{
    double yd = (double)y;
    if (loss == ORA_LOSS_LOGISTIC) {
        double m = yd * z, sm, snm;
        sig_pair(m, &sm, &snm);
        *G = -snm * yd;
        *H = sm * snm;
    } else {
        double b = 1.0 - yd * z;
        if (b > 0) {
            *G = -2.0 * yd * b;
            *H = 2.0;
        } else {
            *G = 0.0;
            *H = 0.0;
        }
    }
}

/* Per-sample forms with the sample's target available (the squared loss needs t_i, Z26). */
static double phi_i(const ora_prob *pb, int64_t i, double z)
{
    if (pb->loss == ORA_LOSS_SQUARED) {
        double r = pb->t[i] - z;
        return r * r;
    }
    return ora_phi(pb->loss, (double)pb->y[i] * z);
}

static void GH_i(const ora_prob *pb, int64_t i, double z, double *G, double *H)
{
    if (pb->loss == ORA_LOSS_SQUARED) {   /* d/dz (t - z)^2 = 2(z - t), d2/dz2 = 2 */
        *G = 2.0 * (z - pb->t[i]);
        *H = 2.0;
        return;
    }
    ora_GH(pb->loss, z, pb->y[i], G, H);
}

/* Eq.1 evaluated from scratch from (z = Xw, w) (a6, Z19, Z23). */
double ora_objective(const ora_prob *pb, const double *z, const double *w)
{
    double loss = 0.0, l1 = 0.0, l2 = 0.0;
    for (int64_t i = 0; i < pb->s; i++) loss += phi_i(pb, i, z[i]);
    for (int64_t j = 0; j < pb->n; j++) {
        l1 += fabs(w[j]);
        l2 += w[j] * w[j];
    }
    return pb->c * loss + l1 + 0.5 * pb->mu * l2;   /* Eq.1 (+ the elastic-net term, Z25) */
}

/* z = X w, column by column in ascending j (each z_i accumulates in ascending j). */
void ora_compute_z(const ora_prob *pb, const double *w, double *z)
{
    for (int64_t i = 0; i < pb->s; i++) z[i] = 0.0;
    for (int64_t j = 0; j < pb->n; j++)
        for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++)
            z[pb->row_idx[p]] += w[j] * (double)pb->val[p];
}

/* g_j, h_j for one feature (Eq.13 / App.A.2), with the nu floor of reading Z4:
 * h <- max(h, nu) after the factor c (and the elastic-net terms mu w_j, mu of Z25), for both
 * losses.  Also returns sum |terms|.  w may be NULL when mu == 0. */
static void gh_one(const ora_prob *pb, const double *z, const double *w, int64_t j,
                   double *g, double *h, double *gabs, double *habs)
{
    double gs = 0.0, hs = 0.0, ga = 0.0, ha = 0.0;
    for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++) {
        int64_t i = pb->row_idx[p];
        double x = (double)pb->val[p], G, H;
        GH_i(pb, i, z[i], &G, &H);
        gs += x * G;
        hs += (x * x) * H;
        ga += fabs(x * G);
        ha += fabs((x * x) * H);
    }
    const double wj = w ? w[j] : 0.0;
    *g = pb->c * gs + pb->mu * wj;
    *h = pb->c * hs + pb->mu;
    if (!(*h > pb->nu)) *h = pb->nu;
    if (gabs) *gabs = pb->c * ga + fabs(pb->mu * wj);
    if (habs) *habs = pb->c * ha + pb->mu;
}

void ora_gh_all(const ora_prob *pb, const double *z, const double *w, double *g, double *h)
{
    for (int64_t j = 0; j < pb->n; j++) gh_one(pb, z, w, j, &g[j], &h[j], NULL, NULL);
}

/* Eq.5; branches tested in printed order (reading Z17). */
double ora_newton_dir(double g, double h, double wj)
{
    double hw = h * wj;
    if (g + 1.0 <= hw) return -(g + 1.0) / h;
    if (g - 1.0 >= hw) return -(g - 1.0) / h;
    return -wj;
}

/* Per-sample change of phi along the bundle direction at step alpha (reading Z7):
 *  LR : l = log((1+e^{-(m+u)})/(1+e^{-m})) = log1p(expm1(-u) sigma(-m)),   m = y z, u = alpha y dx
 *       (if |u| > 1: softplus(-(m+u)) - softplus(-m))  -- algebraically Eq.12's summand
 *  SVM: l = max(0, 1 - y(z + alpha dx))^2 - max(0, 1 - y z)^2                     (reading Z6) */
static double loss_change(int loss, double z, int y, double dx, double alpha)
{
    double yd = (double)y;
    if (loss == ORA_LOSS_LOGISTIC) {
        double m = yd * z;
        double u = alpha * (yd * dx);
        if (fabs(u) <= 1.0) {
            double sm, snm;
            sig_pair(m, &sm, &snm);
            return log1p(expm1(-u) * snm);
        }
        return softplus(-(m + u)) - softplus(-m);
    }
    double b1 = 1.0 - yd * (z + alpha * dx);
    double b0 = 1.0 - yd * z;
    double p1 = b1 > 0 ? b1 * b1 : 0.0;
    double p0 = b0 > 0 ? b0 * b0 : 0.0;
    return p1 - p0;
}

/* ------------------------------------------------------------------------------ */
/* One PCDN inner iteration (Alg.3 lines 6-10 with Alg.4), a1..a5 of SURVEY §8(a). */
/* ------------------------------------------------------------------------------ */
typedef struct {
    double *g, *h, *d, *g_abs, *h_abs;   /* [P], bundle order (nullable) */
    int32_t *T;                          /* [s] capacity (nullable) */
    double *dx, *dx_abs;                 /* [s] capacity, aligned with T (nullable) */
    int64_t nT;
    int32_t q;
    int32_t pad;
    double alpha, Delta, Delta_abs, lhs, lhs_abs, rhs, F_before, F_after;
    double margin_accept;   /* RHS - LHS at accepted q, relative to max(|LHS|,|RHS|,lhs_abs) */
    double margin_prev;     /* LHS - RHS at q-1 (relative), +inf if q == 0 */
    double margin_d;        /* min over bundle of |Eq.5 branch test| / (|g|+1+|h w|) */
    int64_t bundle_nnz;
} ora_step_out;

typedef struct {
    double *w;      /* [n] */
    double *z;      /* [s] = X w, maintained (retained w'x_i) */
    double F;       /* maintained objective (Z23) */
    double *dx;     /* [s] scratch, zero outside the touched set */
    double *dxa;    /* [s] scratch */
    uint8_t *mark;  /* [s] scratch */
    int32_t *list;  /* [s] scratch */
} ora_state;

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* mode 0: incremental line search from retained quantities (Alg.4, Eq.12).
 * mode 1: direct line search, F(w + alpha d) recomputed from scratch (tiny inputs). */
int ora_bundle_step(const ora_prob *pb, ora_state *st, const int32_t *bundle, int64_t P,
                    int mode, ora_step_out *out)
{
    const int64_t s = pb->s;
    double *g = (double *)malloc(sizeof(double) * (size_t)(P > 0 ? P : 1));
    double *h = (double *)malloc(sizeof(double) * (size_t)(P > 0 ? P : 1));
    double *d = (double *)malloc(sizeof(double) * (size_t)(P > 0 ? P : 1));
    double Delta = 0.0, Delta_abs = 0.0, margin_d = INFINITY;
    int64_t bnnz = 0;

    /* a1, a2: per-feature g_j, h_j and d_j (Alg.3 l.7-9 "in parallel"), Delta (Eq.7 on B) */
    for (int64_t kk = 0; kk < P; kk++) {
        int64_t j = bundle[kk];
        double ga, ha;
        gh_one(pb, st->z, st->w, j, &g[kk], &h[kk], &ga, &ha);
        double wj = st->w[j];
        d[kk] = ora_newton_dir(g[kk], h[kk], wj);
        double hw = h[kk] * wj;
        double sc = fabs(g[kk]) + 1.0 + fabs(hw);
        double m1 = fabs((g[kk] + 1.0) - hw) / sc, m2 = fabs((g[kk] - 1.0) - hw) / sc;
        if (m1 < margin_d) margin_d = m1;
        if (m2 < margin_d) margin_d = m2;
        double dj = d[kk];
        double delta_j = g[kk] * dj + pb->gamma * h[kk] * dj * dj + fabs(wj + dj) - fabs(wj);
        Delta += delta_j;
        Delta_abs += fabs(g[kk] * dj) + fabs(pb->gamma * h[kk] * dj * dj) + fabs(wj + dj) + fabs(wj);
        if (out) {
            if (out->g) out->g[kk] = g[kk];
            if (out->h) out->h[kk] = h[kk];
            if (out->d) out->d[kk] = dj;
            if (out->g_abs) out->g_abs[kk] = ga;
            if (out->h_abs) out->h_abs[kk] = ha;
        }
        bnnz += pb->col_ptr[j + 1] - pb->col_ptr[j];
    }

    /* a3: d'x_i over the touched samples T (Alg.4 l.1; reading Z8), bundle order */
    int64_t nl = 0;
    for (int64_t kk = 0; kk < P; kk++) {
        if (d[kk] == 0.0) continue;
        int64_t j = bundle[kk];
        for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++) {
            int32_t i = pb->row_idx[p];
            if (!st->mark[i]) {
                st->mark[i] = 1;
                st->dx[i] = 0.0;
                st->dxa[i] = 0.0;
                st->list[nl++] = i;
            }
            double t = d[kk] * (double)pb->val[p];
            st->dx[i] += t;
            st->dxa[i] += fabs(t);
        }
    }
    qsort(st->list, (size_t)nl, sizeof(int32_t), cmp_i32);   /* T ascending */

    /* a4: Armijo over alpha = beta^q (Eq.6), LHS from retained quantities (Eq.12) */
    double F0 = st->F;
    double *wnew = NULL, *znew = NULL;
    if (mode == 1) {
        wnew = (double *)malloc(sizeof(double) * (size_t)pb->n);
        znew = (double *)malloc(sizeof(double) * (size_t)s);
        F0 = ora_objective(pb, st->z, st->w);
    }
    double alpha = 1.0, lhs = 0.0, lhs_abs = 0.0, rhs = 0.0, prev_margin = INFINITY;
    int32_t q = -1;
    for (int32_t qq = 0; qq <= pb->qmax; qq++) {
        if (mode == 0) {
            double L1 = 0.0, Ls = 0.0, L1a = 0.0, Lsa = 0.0;
            for (int64_t kk = 0; kk < P; kk++) {
                double wj = st->w[bundle[kk]];
                /* separable term change: |w+ad| - |w| + (mu/2)((w+ad)^2 - w^2), the latter as
                 * mu a d (w + a d / 2) (reading Z25) */
                double t = fabs(wj + alpha * d[kk]) - fabs(wj) + pb->mu * alpha * d[kk] * (wj + 0.5 * alpha * d[kk]);
                L1 += t;
                L1a += fabs(t);
            }
            for (int64_t a = 0; a < nl; a++) {
                int32_t i = st->list[a];
                double t = pb->loss == ORA_LOSS_SQUARED
                               ? alpha * st->dx[i] * (alpha * st->dx[i] + 2.0 * (st->z[i] - pb->t[i]))   /* Z26 */
                               : loss_change(pb->loss, st->z[i], pb->y[i], st->dx[i], alpha);
                Ls += t;
                Lsa += fabs(t);
            }
            lhs = L1 + pb->c * Ls;
            lhs_abs = L1a + pb->c * Lsa;
        } else {
            memcpy(wnew, st->w, sizeof(double) * (size_t)pb->n);
            for (int64_t kk = 0; kk < P; kk++) wnew[bundle[kk]] = st->w[bundle[kk]] + alpha * d[kk];
            ora_compute_z(pb, wnew, znew);
            lhs = ora_objective(pb, znew, wnew) - F0;
            lhs_abs = fabs(lhs);
        }
        rhs = pb->sigma * alpha * Delta;
        double scale = fmax(fmax(fabs(lhs), fabs(rhs)), lhs_abs);
        if (scale == 0.0) scale = 1.0;
        if (lhs <= rhs) {
            q = qq;
            if (out) out->margin_accept = (rhs - lhs) / scale;
            break;
        }
        prev_margin = (lhs - rhs) / scale;
        alpha *= pb->beta;   /* reading Z11: alpha_q by repeated multiplication */
    }

    int rc = ORA_OK;
    if (q < 0) {
        /* reading Z10: no q <= q_max passes.  Theorem 1 rules this out in exact arithmetic;
         * in fp64 it happens only when d is at rounding level (near the optimum), so the
         * step is a null step: alpha = 0, state unchanged.  Non-finite values are errors. */
        alpha = 0.0;
        if (!isfinite(lhs) || !isfinite(Delta)) rc = ORA_ERR_NUMERIC;
    } else {
        /* a5: commit (Alg.3 l.10; Alg.4 l.4-5 with additive retained z) */
        for (int64_t kk = 0; kk < P; kk++) st->w[bundle[kk]] += alpha * d[kk];
        if (mode == 0) {
            for (int64_t a = 0; a < nl; a++) {
                int32_t i = st->list[a];
                st->z[i] += alpha * st->dx[i];
            }
            st->F += lhs;
        } else {
            ora_compute_z(pb, st->w, st->z);
            st->F = ora_objective(pb, st->z, st->w);
        }
    }
    if (out) {
        out->nT = nl;
        for (int64_t a = 0; a < nl; a++) {
            int32_t i = st->list[a];
            if (out->T) out->T[a] = i;
            if (out->dx) out->dx[a] = st->dx[i];
            if (out->dx_abs) out->dx_abs[a] = st->dxa[i];
        }
        out->q = q;
        out->alpha = alpha;
        out->Delta = Delta;
        out->Delta_abs = Delta_abs;
        out->lhs = lhs;
        out->lhs_abs = lhs_abs;
        out->rhs = rhs;
        out->F_before = F0;
        out->F_after = st->F;
        out->margin_prev = prev_margin;
        out->margin_d = margin_d;
        out->bundle_nnz = bnnz;
    }
    for (int64_t a = 0; a < nl; a++) {
        int32_t i = st->list[a];
        st->mark[i] = 0;
        st->dx[i] = 0.0;
        st->dxa[i] = 0.0;
    }
    free(g);
    free(h);
    free(d);
    free(wnew);
    free(znew);
    return rc;
}

/* ------------------------------------------------------------------------------ */
/* Alg.3 driver with the Eq.14 outer stop test (readings Z12, Z23).                */
/* ------------------------------------------------------------------------------ */
typedef struct {
    int32_t outer_iters;
    int32_t status;
    int64_t steps;
    int64_t nnz_processed;
    int64_t touched_total;
    int64_t null_steps;
    double F;
    double gap;
    double t_steps;   /* wall seconds inside the bundle steps (timing only; the CPU baseline's rate) */
} ora_solve_info;

/* margin_trace (nullable): per step, the smallest relative margin of its decisions -- the Eq.5
 * branch tests, the accepted Armijo test and the rejected one before it (reading Z22).  A GPU
 * decision may differ from the oracle's only where this is below the tie threshold.
 * max_steps > 0: stop after that many bundle steps (a bounded timing sample of the CPU baseline;
 * the outer iteration in progress is not finished, no outer refresh, rc = ORA_BUDGET). */
int ora_solve(const ora_prob *pb, double *w, double *z, int64_t P, double eps, double fstar,
              uint64_t seed, int32_t max_outer, int32_t *q_trace, double *F_trace,
              double *outer_F, int64_t trace_cap, ora_solve_info *info, double *margin_trace,
              int64_t max_steps)
{
    const int64_t s = pb->s, n = pb->n;
    if (P < 1 || P > n) return ORA_ERR_INVALID;
    ora_state st;
    st.w = w;
    st.z = z;
    st.dx = (double *)calloc((size_t)s, sizeof(double));
    st.dxa = (double *)calloc((size_t)s, sizeof(double));
    st.mark = (uint8_t *)calloc((size_t)s, 1);
    st.list = (int32_t *)malloc(sizeof(int32_t) * (size_t)s);
    int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    ora_compute_z(pb, w, z);
    st.F = ora_objective(pb, z, w);
    int64_t steps = 0, nnzp = 0, touched = 0, nulls = 0;
    double t_steps = 0.0;
    int rc = ORA_BUDGET;
    int32_t k;
    double gap = INFINITY;
    ora_step_out o;
    memset(&o, 0, sizeof(o));
    for (k = 0; k < max_outer; k++) {
        ora_permutation(seed, k, n, perm);                        /* Alg.3 l.4, Eq.8 */
        for (int64_t t0 = 0; t0 < n; t0 += P) {                   /* Alg.3 l.5 */
            if (max_steps > 0 && steps >= max_steps) goto done;
            int64_t Pt = (n - t0) < P ? (n - t0) : P;
            struct timespec ta, tb;
            clock_gettime(CLOCK_MONOTONIC, &ta);
            int r = ora_bundle_step(pb, &st, perm + t0, Pt, 0, &o);
            clock_gettime(CLOCK_MONOTONIC, &tb);
            t_steps += (double)(tb.tv_sec - ta.tv_sec) + 1e-9 * (double)(tb.tv_nsec - ta.tv_nsec);
            if (r != ORA_OK) {
                rc = r;
                goto done;
            }
            if (steps < trace_cap) {
                if (q_trace) q_trace[steps] = o.q;
                if (F_trace) F_trace[steps] = st.F;
                if (margin_trace) {
                    double m = o.margin_d;
                    if (o.q >= 0 && o.margin_accept < m) m = o.margin_accept;
                    if (o.margin_prev < m) m = o.margin_prev;
                    margin_trace[steps] = m;
                }
            }
            steps++;
            if (o.q < 0) nulls++;
            nnzp += o.bundle_nnz;
            touched += o.nT;
        }
        st.F = ora_objective(pb, z, w);                           /* a6: refresh (Z23) */
        if (outer_F) outer_F[k] = st.F;
        if (!isfinite(st.F)) {
            rc = ORA_ERR_NUMERIC;
            k++;
            goto done;
        }
        if (eps > 0.0) {
            gap = (st.F - fstar) / fstar;                         /* Eq.14 */
            if (gap <= eps) {
                rc = ORA_OK;
                k++;
                goto done;
            }
        }
    }
done:
    if (info) {
        info->outer_iters = k;
        info->status = rc;
        info->steps = steps;
        info->nnz_processed = nnzp;
        info->touched_total = touched;
        info->null_steps = nulls;
        info->F = st.F;
        info->gap = eps > 0.0 ? (st.F - fstar) / fstar : NAN;
        info->t_steps = t_steps;
    }
    free(st.dx);
    free(st.dxa);
    free(st.mark);
    free(st.list);
    free(perm);
    return rc;
}

/* ------------------------------------------------------------------------------ */
/* CDN, Alg.1, coded separately from the PCDN path above: its own */
/* derivative forms (Eq.13 literally, tau(y w'x)), its own 1-D Armijo with direct  */
/* phi differences over the column's samples (Eq.6 with d = d_j e_j).  Features in */
/* outer pass k are visited in the order pi_k (reading Z3), so that PCDN(P=1) and  */
/* CDN walk the same coordinates ("CDN is a special case ... P=1").  */
/* ------------------------------------------------------------------------------ */
static double tau(double t)   /* tau(t) = 1/(1+e^{-t}) */
{
    if (t >= 0) return 1.0 / (1.0 + exp(-t));
    double e = exp(t);
    return e / (1.0 + e);
}

int ora_cdn(const ora_prob *pb, double *w, double *z, uint64_t seed, int32_t max_outer,
            double *F_trace, int64_t trace_cap, double *F_out)
{
    const int64_t n = pb->n;
    int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    ora_compute_z(pb, w, z);
    int64_t steps = 0;
    int rc = ORA_OK;
    for (int32_t k = 0; k < max_outer && rc == ORA_OK; k++) {
        ora_permutation(seed, k, n, perm);
        for (int64_t t = 0; t < n; t++) {
            int64_t j = perm[t];
            double gl = 0.0, hl = 0.0;
            for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++) {
                int64_t i = pb->row_idx[p];
                double x = (double)pb->val[p], yd = (double)pb->y[i];
                if (pb->loss == ORA_LOSS_SQUARED) {            /* d/dw_j sum (t - x'w)^2 */
                    gl += -2.0 * (pb->t[i] - z[i]) * x;
                    hl += 2.0 * x * x;
                } else if (pb->loss == ORA_LOSS_LOGISTIC) {
                    double ta = tau(yd * z[i]);
                    gl += (ta - 1.0) * yd * x;                 /* Eq.13 */
                    hl += ta * (1.0 - ta) * x * x;
                } else if (yd * z[i] < 1.0) {                  /* I(w) */
                    gl += -2.0 * yd * x * (1.0 - yd * z[i]);
                    hl += 2.0 * x * x;
                }
            }
            double wj = w[j], dj;
            gl = gl * pb->c + pb->mu * wj;                     /* Z25 */
            hl = hl * pb->c + pb->mu;
            if (!(hl > pb->nu)) hl = pb->nu;
            if (gl + 1.0 <= hl * wj) dj = -(gl + 1.0) / hl;    /* Eq.5 */
            else if (gl - 1.0 >= hl * wj) dj = -(gl - 1.0) / hl;
            else dj = -wj;
            double Delta = gl * dj + pb->gamma * hl * dj * dj + fabs(wj + dj) - fabs(wj);
            double alpha = 1.0;
            int ok = 0;
            for (int32_t q = 0; q <= pb->qmax; q++) {
                double chg = 0.0;
                for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++) {
                    int64_t i = pb->row_idx[p];
                    double yd = (double)pb->y[i];
                    double znew = z[i] + alpha * dj * (double)pb->val[p];
                    chg += pb->loss == ORA_LOSS_SQUARED
                               ? (pb->t[i] - znew) * (pb->t[i] - znew) - (pb->t[i] - z[i]) * (pb->t[i] - z[i])
                               : ora_phi(pb->loss, yd * znew) - ora_phi(pb->loss, yd * z[i]);
                }
                double wn = wj + alpha * dj;
                double lhs = pb->c * chg + fabs(wn) - fabs(wj) + 0.5 * pb->mu * (wn * wn - wj * wj);
                if (lhs <= pb->sigma * alpha * Delta) {
                    ok = 1;
                    break;
                }
                alpha *= pb->beta;
            }
            if (!ok) continue;   /* null step (reading Z10) */
            w[j] = wj + alpha * dj;
            for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++)
                z[pb->row_idx[p]] += alpha * dj * (double)pb->val[p];
            if (F_trace && steps < trace_cap) F_trace[steps] = ora_objective(pb, z, w);
            steps++;
        }
    }
    if (F_out) *F_out = ora_objective(pb, z, w);
    free(perm);
    return rc;
}

/* ------------------------------------------------------------------------------ */
/* SCDN, Alg.2, synchronous reading Z27: each iteration takes the */
/* next P-bar features of the partition stream pi_k (the same bundles PCDN visits);   */
/* every feature computes d_j (Eq.5) and its own 1-D Armijo step alpha_j (Eq.6 with   */
/* d = d_j e_j, direct phi differences over its column) at the iteration's start      */
/* state, then ALL updates w_j += alpha_j d_j are applied together (the deterministic */
/* limit of Shotgun's concurrent updates).  No P-dimensional line search: F may rise  */
/* when correlated features move together.  P-bar = 1 is CDN.          */
/* ------------------------------------------------------------------------------ */
int ora_scdn(const ora_prob *pb, double *w, double *z, int64_t Pbar, uint64_t seed, int32_t max_outer,
             double *F_trace, int64_t trace_cap, int64_t *steps_out, double *F_out)
{
    const int64_t n = pb->n;
    if (Pbar < 1 || Pbar > n) return ORA_ERR_INVALID;
    int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    double *step = (double *)malloc(sizeof(double) * (size_t)Pbar);
    ora_compute_z(pb, w, z);
    int64_t steps = 0;
    int rc = ORA_OK;
    for (int32_t k = 0; k < max_outer && rc == ORA_OK; k++) {
        ora_permutation(seed, k, n, perm);
        for (int64_t t0 = 0; t0 < n; t0 += Pbar) {
            const int64_t Pt = (n - t0) < Pbar ? (n - t0) : Pbar;
            for (int64_t kk = 0; kk < Pt; kk++) {          /* "in parallel": all from the same state */
                const int64_t j = perm[t0 + kk];
                double g, h;
                gh_one(pb, z, w, j, &g, &h, NULL, NULL);
                const double wj = w[j];
                const double dj = ora_newton_dir(g, h, wj);
                const double Delta = g * dj + pb->gamma * h * dj * dj + fabs(wj + dj) - fabs(wj);
                double alpha = 1.0, take = 0.0;
                for (int32_t q = 0; q <= pb->qmax; q++) {
                    double chg = 0.0;
                    for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++) {
                        const int64_t i = pb->row_idx[p];
                        const double znew = z[i] + alpha * dj * (double)pb->val[p];
                        chg += phi_i(pb, i, znew) - phi_i(pb, i, z[i]);
                    }
                    const double wn = wj + alpha * dj;
                    const double lhs = pb->c * chg + fabs(wn) - fabs(wj) + 0.5 * pb->mu * (wn * wn - wj * wj);
                    if (lhs <= pb->sigma * alpha * Delta) {
                        take = alpha;
                        break;
                    }
                    alpha *= pb->beta;
                }
                step[kk] = take * dj;                       /* null step (Z10): 0 */
            }
            for (int64_t kk = 0; kk < Pt; kk++) {          /* apply all updates together */
                const int64_t j = perm[t0 + kk];
                if (step[kk] == 0.0) continue;
                w[j] += step[kk];
                for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++)
                    z[pb->row_idx[p]] += step[kk] * (double)pb->val[p];
            }
            if (F_trace && steps < trace_cap) F_trace[steps] = ora_objective(pb, z, w);
            steps++;
            if (!isfinite(ora_objective(pb, z, w))) {
                rc = ORA_ERR_NUMERIC;
                break;
            }
        }
    }
    if (steps_out) *steps_out = steps;
    if (F_out) *F_out = ora_objective(pb, z, w);
    free(perm);
    free(step);
    return rc;
}

/* Minimum-norm subgradient of F at w (KKT residual): returns its
 * 1-norm and fills out[n] (nullable). */
double ora_min_norm_subgrad(const ora_prob *pb, const double *w, const double *z, double *out)
{
    double tot = 0.0;
    for (int64_t j = 0; j < pb->n; j++) {
        double gs = 0.0;
        for (int64_t p = pb->col_ptr[j]; p < pb->col_ptr[j + 1]; p++) {
            int64_t i = pb->row_idx[p];
            double G, H;
            GH_i(pb, i, z[i], &G, &H);
            gs += (double)pb->val[p] * G;
        }
        double gj = pb->c * gs + pb->mu * w[j], v;
        if (w[j] > 0) v = gj + 1.0;
        else if (w[j] < 0) v = gj - 1.0;
        else v = (gj > 1.0) ? gj - 1.0 : (gj < -1.0 ? gj + 1.0 : 0.0);
        if (out) out[j] = v;
        tot += fabs(v);
    }
    return tot;
}

/* Per-sample loss change exposed for pins (same function the line search uses). */
double ora_loss_change(int loss, double z, int y, double dx, double alpha)
{
    return loss_change(loss, z, y, dx, alpha);
}

int ora_state_size(void) { return (int)sizeof(ora_state); }
int ora_step_out_size(void) { return (int)sizeof(ora_step_out); }
int ora_prob_size(void) { return (int)sizeof(ora_prob); }
int ora_solve_info_size(void) { return (int)sizeof(ora_solve_info); }
