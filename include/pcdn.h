/*
 * pcdn.h -- C-ABI of the B200 (sm_100a) PCDN hot path.
 *
 * PCDN = Parallel Coordinate Descent Newton (Bian, Li, Liu, Yang, arXiv:1306.4080).
 * Citations "PAPER.md:L" are lines of the paper's LaTeX source; "Zk" are the readings
 * listed in DESIGN.md.  The problem solved is Eq.1:
 *
 *      min_w  F_c(w) = c * sum_{i<s} phi(y_i w'x_i) + ||w||_1
 *      phi_log(m) = log(1 + e^{-m})      (Eq.2)       loss = PCDN_LOSS_LOGISTIC
 *      phi_svm(m) = max(0, 1 - m)^2      (Eq.3)       loss = PCDN_LOSS_L2SVM
 *
 * Letters follow the paper: s samples, n features, P bundle size.
 *
 * Conventions for every call:
 *  - Array arguments are DEVICE pointers unless marked (host).  They are borrowed: the caller
 *    (e.g. torch) owns them and keeps them alive and unmodified while the context exists.
 *  - The library allocates no device memory except in pcdn_train_host(); state and scratch
 *    live in the caller's workspace (pcdn_workspace_bytes).
 *  - Every call is stream-ordered on the context's CUDA stream.  Calls that return host
 *    values (info structs, F_out, status after device checks) synchronize that stream.
 *  - Return value: a PCDN_* status code.  On failure pcdn_last_error() describes the cause;
 *    the context stays usable after PCDN_ERR_INVALID, not after PCDN_ERR_CUDA.
 *  - A context is not thread-safe; use one per stream.
 */
#ifndef PCDN_H
#define PCDN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (mirroring SPEC.md:473, 503 exit codes 0/1/2/3). */
#define PCDN_OK 0            /* success; for pcdn_solve: stop test met (Eq.14 gap <= eps)   */
#define PCDN_ERR_INVALID 1   /* argument or data-invariant violation                         */
#define PCDN_BUDGET 2        /* pcdn_solve: max_outer outer iterations done, gap > eps       */
#define PCDN_ERR_NUMERIC 3   /* non-finite objective / direction (reading Z10)               */
#define PCDN_ERR_CUDA 4      /* CUDA runtime error (the context must be destroyed)           */
#define PCDN_ERR_NOMEM 5     /* workspace too small / host allocation failed                 */

#define PCDN_LOSS_LOGISTIC 0 /* Eq.2 */
#define PCDN_LOSS_L2SVM 1    /* Eq.3, generalized Hessian App. A.2        */
#define PCDN_LOSS_SQUARED 2  /* (t_i - w'x_i)^2 with real targets: Lasso / elastic net
                                (reading Z26); pcdn_set_targets */

typedef struct pcdn_ctx pcdn_ctx;

/* Result of one bundle step (Alg.3 lines 6-10). */
typedef struct {
    int32_t q;           /* accepted Armijo index, alpha = beta^q (Eq.6); -1 = null step (Z10) */
    int32_t reserved;
    double alpha;        /* accepted step size (0 for a null step)                            */
    double Delta;        /* Eq.7 restricted to the bundle             */
    double lhs;          /* F(w + alpha d) - F(w) from retained quantities (Eq.12)            */
    double rhs;          /* sigma * alpha * Delta                                              */
    double F;            /* maintained objective after the step (reading Z23)                 */
    int64_t bundle_nnz;  /* sum over the bundle's columns of their nonzero counts             */
    int64_t n_touched;   /* |T|: samples with a nonzero in a column with d_j != 0 (Z8)        */
} pcdn_step_info;

/* Result of pcdn_solve (Alg.3 outer loop + Eq.14 stop test). */
typedef struct {
    int32_t status;           /* PCDN_OK / PCDN_BUDGET / error code                           */
    int32_t outer_iters;      /* outer iterations k completed                                 */
    int64_t steps;            /* bundle steps (inner iterations t) completed                  */
    int64_t null_steps;       /* steps whose line search was exhausted (Z10)                  */
    int64_t nnz_processed;    /* sum over steps of bundle_nnz                                 */
    int64_t touched_total;    /* sum over steps of |T|                                        */
    int64_t positions;        /* sum over steps of the bundle size                           */
    int64_t kernel_launches;  /* CUDA kernels launched by this call                           */
    double F;                 /* F_c(w) recomputed from (z, w) at the last outer boundary     */
    double gap;               /* (F - F*)/F* (Eq.14), NaN without a reference                 */
    double t_wall_ms;         /* host wall time of the call                                   */
    double t_step_kernel_ms;  /* CUDA-event time of the bundle-step kernels (sum)             */
    double t_gpu_ms;          /* CUDA-event time from first to last kernel of the call        */
    double alg_bytes;         /* algorithmic bytes of the bundle steps  */
} pcdn_solve_info;

/* Bytes of device workspace a context for an s x n matrix with nnz nonzeros needs
 * (alignment included).  Pure host function. */
size_t pcdn_workspace_bytes(int64_t s, int64_t n, int64_t nnz);

/* Create a context.  Inputs (all device, borrowed):
 *   csc_col_ptr[n+1] (int64, col_ptr[0]=0, col_ptr[n]=nnz, nondecreasing),
 *   csc_row_idx[nnz] (int32, strictly increasing inside each column, < s),
 *   csc_val[nnz] (fp32, finite) -- column x^j of X;
 *   csr_row_ptr[s+1], csr_col_idx[nnz], csr_val[nnz] -- the same nonzeros by row;
 *   y[s] (int8 in {-1,+1}; ignored, and may be NULL, for PCDN_LOSS_SQUARED, whose
 *   real targets come from pcdn_set_targets); c > 0 (Eq.1); loss = PCDN_LOSS_*.
 *   workspace: device buffer of >= pcdn_workspace_bytes(s,n,nnz) bytes, 256-byte aligned.
 *   cuda_stream: cudaStream_t (NULL = legacy default stream).
 * Validates every invariant above on the device (PCDN_ERR_INVALID names the first offending
 * index), then sets w = 0, z = Xw = 0, F = F_c(0).  Synchronizes. */
int pcdn_create(int64_t s, int64_t n, int64_t nnz,
                const int64_t *csc_col_ptr, const int32_t *csc_row_idx, const float *csc_val,
                const int64_t *csr_row_ptr, const int32_t *csr_col_idx, const float *csr_val,
                const int8_t *y, double c, int loss,
                void *workspace, size_t workspace_bytes, void *cuda_stream, pcdn_ctx **out);

/* Armijo constants (Eq.6-7).  Defaults sigma=0.01, beta=0.5, gamma=0,
 * q_max=50 (Z10).  Requires 0<sigma<1, 0<beta<1, 0<=gamma<1, 0<=q_max<=200. */
int pcdn_set_armijo(pcdn_ctx *ctx, double sigma, double beta, double gamma, int q_max);

/* F* for the Eq.14 stop test (reading Z12).  Must be finite and > 0. */
int pcdn_set_reference(pcdn_ctx *ctx, double f_star);

/* One PCDN inner iteration on the given bundle (Alg.3 l.6-10): a1 g/h (Eq.13, App.A.2),
 * a2 d (Eq.5) and Delta (Eq.7), a3 d'x_i over T (Alg.4 l.1), a4 P-dim Armijo (Eq.6, Eq.12),
 * a5 commit to w and the retained z (Alg.4 l.4-5).
 *   bundle[P]: device, P distinct feature ids in [0,n) (checked on device -> PCDN_ERR_INVALID),
 *              processed in this order (bundle position k = index in this array).
 *   info: host, nullable.  g_out/h_out/d_out: device [P], nullable (g, h after the nu floor, d).
 * Synchronizes when info != NULL. */
int pcdn_bundle_step(pcdn_ctx *ctx, const int32_t *bundle, int64_t P, pcdn_step_info *info,
                     double *g_out, double *h_out, double *d_out);

/* Touched set and d'x of the last pcdn_bundle_step taken with debug on (pcdn_set_debug).
 * T_out (host, ascending sample ids) and dx_out (host) get min(|T|, capacity) entries;
 * *nT (host) gets |T|.  Synchronizes. */
int pcdn_last_touched(pcdn_ctx *ctx, int32_t *T_out, double *dx_out, int64_t capacity, int64_t *nT);

/* Alg.3: from the current w, run outer iterations k = 0..max_outer-1.  Outer k draws the
 * partition pi_k(seed, k) (Eq.8, reading Z2) and runs b = ceil(n/P) bundle steps on the
 * device without host round trips; then F is recomputed from (z, w) (Z23) and, if eps > 0,
 * the Eq.14 gap is tested (needs pcdn_set_reference).  eps <= 0 runs exactly max_outer.
 * Returns PCDN_OK when the gap <= eps, PCDN_BUDGET after max_outer.  info: host, nullable. */
int pcdn_solve(pcdn_ctx *ctx, int64_t P, double eps, uint64_t seed, int32_t max_outer,
               pcdn_solve_info *info);

/* F_c(w) (Eq.1) into *F_out (host).  recompute_from_w != 0: recompute z = Xw (CSR, ascending
 * column order) first; otherwise evaluate from the retained z.  Synchronizes. */
int pcdn_objective(pcdn_ctx *ctx, int recompute_from_w, double *F_out);

/* Copy w (device fp64[n]) out / in.  pcdn_set_w recomputes z = Xw and F (state injection). */
int pcdn_get_w(pcdn_ctx *ctx, double *w_out);
int pcdn_set_w(pcdn_ctx *ctx, const double *w);
/* Copy the retained z = Xw (device fp64[s]). */
int pcdn_get_z(pcdn_ctx *ctx, double *z_out);
/* Back to w = 0, z = 0, F = F_c(0). */
int pcdn_reset(pcdn_ctx *ctx);

/* Device copy of the partition permutation pi_k (reading Z2) for outer iteration k:
 * out[n] (device int32); bundle t = out[tP : min((t+1)P, n)]. */
int pcdn_permutation(pcdn_ctx *ctx, uint64_t seed, int64_t k, int32_t *out);

/* Optional per-step trace during pcdn_solve: q_trace[t], F_trace[t] (device, nullable) for the
 * first `capacity` steps of each call. */
int pcdn_set_trace(pcdn_ctx *ctx, int32_t *q_trace, double *F_trace, int64_t capacity);

/* Debug flags.  on & 1: record T and d'x of each step (for pcdn_last_touched).  on & 2: build
 * each outer iteration's lists with the reference sequence of launches (k_perm, device-wide
 * scans, compactions) instead of the single-pass k_prep_lists -- a test knob; the lists are
 * identical.  on & 4: the dense kernel as one launch per outer iteration (test knob; results
 * bit-identical). */
int pcdn_set_debug(pcdn_ctx *ctx, int on);

/* Launch knobs (results stay within fp64 rounding-order differences; for a fixed setting they
 * are bit-reproducible).  mode: 0 auto (cluster-resident when the mean bundle holds <= 64K
 * nonzeros and the samples fit the cluster's shared memory, else cluster / grid as below),
 * 1 one thread-block cluster of `ctas` <= 16 CTAs with hardware cluster barriers, per-sample
 *   state in HBM/L2,
 * 2 cooperative grid of `ctas` CTAs with a software grid barrier (0 = all co-resident),
 * 3 cluster-resident: one cluster of `ctas` CTAs (power of two <= 16; 0 = largest that fits)
 *   holding the per-sample state and the step's d'x records in distributed shared memory
 *   (DESIGN.md 7); PCDN_ERR_INVALID if the samples do not fit.
 * 4 dense row-block kernel (every column full).
 * heavy_len: column length above which a column leaves the one-warp path (0 = the library's
 * choice per mode and bundle size).  Modes 1-2 (the sparse kernel): longer columns are reduced by
 * whole CTAs in chunks of 12 * heavy_len nonzeros; default 256, and in mode 2 64 / 128 when a
 * step brings a CTA at most 256 / 640 bundle nonzeros (nnz * P / n / CTAs).  Mode 3:
 * split over the cluster's warps above 96.  Mode 5 (the round-1 grid kernel): 2048, columns of
 * 129..2048 nonzeros reduced inside one CTA, longer ones nnz-balanced over the launch's warps. */
int pcdn_set_launch(pcdn_ctx *ctx, int mode, int ctas, int heavy_len);

/* Sample-sharded step: data larger than one
 * GPU.  Each rank creates a context over ITS rows (their CSC/CSR, labels / targets); w and the
 * partition stream are replicated.  One PCDN bundle step (Alg.3 l.6-10 with Alg.4) is then, on
 * every rank, for the same device bundle[P] (distinct feature indices; not validated here):
 *   pcdn_shard_gh          -> gh_out (DEVICE fp64[2P]): sum_i x_ij G_i, sum_i x_ij^2 H_i over the
 *                             local samples (Eq.13 / App. A.2 factors, before the factor c);
 *   caller: sum gh over the ranks (in rank order, for bit-identical results on every rank);
 *   pcdn_shard_direction   d_j (Eq.5), the Delta terms (Eq.7) from the GLOBAL sums, and the d'x
 *                             records of the local samples;
 *   pcdn_shard_line_search -> out (DEVICE fp64[13]) for candidates alpha = beta^(q0+q), q < 6:
 *                             out[q] = local sum_i phi change (Eq.12 summand, before c);
 *                             out[6+q] = the bundle's separable-term change, out[12] = Delta --
 *                             both only if with_l1 (exactly one rank), else 0.  first = 1 for the
 *                             step's first window (folds d'x_i), 0 for later windows;
 *   caller: sum out over the ranks (rank order);
 *   pcdn_shard_decide      the Eq.6 decision of the window from the rank-summed totals tot (DEVICE
 *                             fp64[13]), on the device with the context's sigma, beta, q_max
 *                             (pcdn_set_armijo): the first q with out[6+q] + c out[q] <= sigma
 *                             alpha out[12]; recorded in the context and copied to *out (host):
 *                             q (-1: none in this window), next (1: run the window at q0 + 6; 0
 *                             with q = -1: q_max passed, a null step, reading Z10), alpha, LHS,
 *                             RHS, Delta, and the maintained objective F after the step.
 *                             PCDN_ERR_NUMERIC for non-finite totals.  Synchronizes;
 *   pcdn_shard_commit      with the recorded decision: w_B += alpha d_B (every rank), z and the
 *                             factors of the local touched samples, F += LHS (q = -1: a null
 *                             step, records cleared).  Synchronizes.
 * At an outer boundary (reading Z23):
 *   pcdn_shard_loss        -> loss_out (DEVICE fp64[1]): c sum_i phi_i over the local samples;
 *   caller: sum loss_out over the ranks (rank order);
 *   pcdn_shard_objective   F = the summed loss (DEVICE fp64[1]) + ||w||_1 + mu/2 ||w||^2 on the
 *                             device; becomes the maintained F and is copied to *F_out (host).
 * The kernels never wait on another rank (the caller's collectives sit between the calls).
 * Returns PCDN_ERR_INVALID for null pointers, P outside [1, n], q0 < 0. */
typedef struct {
    int32_t q;      /* accepted Armijo index, -1 if none in the window */
    int32_t next;   /* 1: no candidate passed and q0 + 6 <= q_max -- run the next window */
    double alpha, lhs, rhs, Delta;
    double F;       /* maintained objective after the step (before it, for q = -1) */
} pcdn_shard_decision;

int pcdn_shard_gh(pcdn_ctx *ctx, const int32_t *bundle, int64_t P, double *gh_out);
int pcdn_shard_direction(pcdn_ctx *ctx, const int32_t *bundle, int64_t P, const double *gh);
int pcdn_shard_line_search(pcdn_ctx *ctx, const int32_t *bundle, int64_t P, int q0, int first, int with_l1,
                           double *out);
int pcdn_shard_decide(pcdn_ctx *ctx, const double *tot, int q0, pcdn_shard_decision *out);
int pcdn_shard_commit(pcdn_ctx *ctx, const int32_t *bundle, int64_t P);
int pcdn_shard_loss(pcdn_ctx *ctx, double *loss_out);
int pcdn_shard_objective(pcdn_ctx *ctx, const double *loss_sum, double *F_out);

/* SCDN baseline (Alg.2 Shotgun CDN; reading Z27): with
 * on != 0, pcdn_bundle_step / pcdn_solve run SCDN instead of PCDN -- each feature of a bundle (of
 * size P-bar = P) takes its own 1-D Armijo step from the bundle's start state and all updates are
 * applied together, with no P-dimensional line search (the accepted q is reported as 0).  The
 * paper's setting is P-bar = 8.  Runs on the cluster-resident kernel only: a
 * solve/step returns PCDN_ERR_INVALID in another launch mode, or when a bundle column is longer
 * than the warp split length (pcdn_set_launch's heavy_len).  PCDN_ERR_INVALID: null context. */
int pcdn_set_scdn(pcdn_ctx *ctx, int on);

/* Squared loss (PCDN_LOSS_SQUARED, reading Z26): borrow the real targets t (DEVICE fp64[s], kept
 * alive and unmodified by the caller) -- F = c sum_i (t_i - w'x_i)^2 + ||w||_1 (+ elastic net).
 * Required before any state-dependent call on a squared-loss context (those return
 * PCDN_ERR_INVALID until then; pcdn_create accepts y = NULL for this loss and ignores y).
 * Validates that every target is finite, then resets the state (w = 0, z, factors, F).
 * PCDN_ERR_INVALID: null context/pointer, another loss, or a non-finite target.
 * pcdn_train_host does not take targets and rejects this loss. */
int pcdn_set_targets(pcdn_ctx *ctx, const double *t);

/* Elastic net ("easily extended to ... elastic net";
 * reading Z25 of DESIGN.md): minimise  c sum_i phi_i + ||w||_1 + (mu/2)||w||_2^2.  mu >= 0 enters
 * g_j (+ mu w_j), h_j (+ mu), the objective and the line search's separable term
 * (+ mu a d_j (w_j + a d_j / 2)); mu = 0 (the default) is the paper's problem, bit for bit.
 * Recomputes the maintained objective on the context's stream.  PCDN_ERR_INVALID for a null
 * context or mu < 0 / not finite. */
int pcdn_set_elastic(pcdn_ctx *ctx, double mu);

/* HBM-state kernels (modes 1, 2): keep the per-sample state (z, coef, record counts, touched
 * bitmap, d'x; one contiguous workspace window) L2-resident with a persisting access-policy window
 * on the step-kernel launches of SMALL steps (estimated bundle nonzeros <= 65536; default OFF).
 * The first such launch sets the device's persisting-L2 limit (cudaLimitPersistingL2CacheSize) to
 * min(device maximum, window bytes) -- a device-wide carve-out that then also shrinks the L2
 * available to large steps and to other work (config 5: -4% step time at P = 4096, but +50% at
 * P = 10^5..10^6 once the carve-out exists), hence opt-in; if the device refuses, the knob turns
 * itself off.  Results are unchanged (a cache policy only).
 * Returns PCDN_ERR_INVALID for a null context. */
int pcdn_set_l2_persist(pcdn_ctx *ctx, int on);

/* Testing knob of mode 3: cap the records a CTA keeps in shared memory per step (0 = as many as
 * fit); the rest spill to the CTA's HBM overflow region.  Results are unchanged. */
int pcdn_set_resident_cap(pcdn_ctx *ctx, int cap);

/* Profiling mode: CTA 0 of the step kernel accumulates clock64() cycles per phase
 * (0 g/h/d + scatter, 1 barrier after it, 2 touched set, 3 d'x fold, 4 line-search partials,
 * 5 barrier + decision, 6 commit, 7 end-of-step barrier).  pcdn_set_profile(ctx, 1) zeroes the
 * counters; pcdn_phase_cycles copies the 16 counters to out (host) and the launch mode used by
 * the last step launch (1 cluster, 2 grid) to *mode (host, nullable).  Synchronizes. */
int pcdn_set_profile(pcdn_ctx *ctx, int on);   /* on: 0 off, 1 phase counters, 2 warp timeline */
int pcdn_phase_cycles(pcdn_ctx *ctx, int64_t *out, int32_t *mode);

/* Profiling mode 2 (pcdn_set_profile(ctx, 2)) records instead (the phase counters stay off, so
 * that thread 0 of CTA 0 runs unmarked), for CTA 0 of the cluster-resident
 * step kernel, clock64() of every warp at 16 points of each of the first 16 steps of a launch.
 * out (host) gets int64[16 steps][16 warps][16 points] (0 = point not reached).  Synchronizes. */
int pcdn_warp_timeline(pcdn_ctx *ctx, int64_t *out);

/* Human-readable description of the last error (never NULL). */
const char *pcdn_last_error(const pcdn_ctx *ctx);

/* Destroy the context (does not free caller memory). */
void pcdn_destroy(pcdn_ctx *ctx);

/* One-call host API: copies HOST arrays (pinned recommended) to the device, trains with
 * pcdn_solve and copies w back to w_out (host fp64[n]).  Allocates and frees its own device
 * memory (stream-ordered).  f_star <= 0 with eps > 0 is invalid.  info: host, nullable.
 * csr_row_ptr, csr_col_idx, csr_val may all be NULL: the CSR is then built on the device from
 * the CSC (a stable radix sort of the nonzeros by row: every row lists its columns ascending),
 * which halves the bytes copied over PCIe.  Passing some but not all of them is invalid. */
int pcdn_train_host(int64_t s, int64_t n, int64_t nnz,
                    const int64_t *csc_col_ptr, const int32_t *csc_row_idx, const float *csc_val,
                    const int64_t *csr_row_ptr, const int32_t *csr_col_idx, const float *csr_val,
                    const int8_t *y, double c, int loss, int64_t P, double eps, double f_star,
                    uint64_t seed, int32_t max_outer, void *cuda_stream, double *w_out,
                    pcdn_solve_info *info);

/* Library version string. */
const char *pcdn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PCDN_H */
