// pcdn_kernels.cuh -- sm_100a kernels of the PCDN hot path.
//
// Citations "PAPER.md:L" point into the paper (arXiv:1306.4080 LaTeX source); "Zk" are the
// readings of DESIGN.md.  This file shares nothing with oracle/ (the CPU oracle).
//
// Design summary:
//   a0  k_perm           keyed Feistel permutation pi_k, one thread per position (Z2)
//       k_scan_*         device-wide exclusive scans building the per-step heavy-column lists
//   a1..a5 k_step        ONE persistent cooperative kernel runs all b bundle steps of an outer
//                        iteration; phases are separated by a software grid barrier:
//        A  g_j,h_j -> d_j -> scatter of (k, d_j x_ij) records into per-row segments
//           (light columns: one warp per column; heavy columns: nnz-balanced split over all
//           warps with a deterministic warp -> CTA -> grid combine)          [grid barrier]
//        C  row-block owners: touched set T from a bitmap, d'x_i by an in-order fold of the
//           row's records sorted by bundle position (no float atomics), line-search partial
//           sums for a window of candidates q                                  [grid barrier]
//        D  every CTA reduces the partials in the same order, picks the first passing q
//           (Eq.6), commits w_B, z_T and the cached per-sample factors           [grid barrier]
//   a6  k_obj_*          F_c(w) from (z, w) with a fixed-order two-level reduction (Eq.1)
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace pcdn {

// Checked build (-DPCDN_CHECKS=1, libpcdn_checked.so): device-side bounds and protocol checks that
// trap with the failing condition.  compute-sanitizer is closed on this pool; the GPU test suite
// runs against this build instead (scripts/checked_run.sh).  The product build compiles them out.
// Profiling instrumentation (pcdn_set_profile phase cycles, pcdn_warp_timeline) is compiled into
// the step kernels only with -DPCDN_PROFILE=1 (libpcdn_prof.so, loaded through PCDN_LIB by the
// profiling scripts): even as untaken branches it costs the product kernels registers and time.
#ifndef PCDN_PROFILE
#define PCDN_PROFILE 0
#endif
#ifndef PCDN_CHECKS
#define PCDN_CHECKS 0
#endif
#if PCDN_CHECKS
#define PCDN_CHECK(cond)                                                                          \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("PCDN_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                            \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define PCDN_CHECK(cond) \
    do {                 \
    } while (0)
#endif

constexpr int NT = 512;            // threads per CTA of the step kernel
constexpr int NW = NT / 32;        // warps per CTA
constexpr int QW = 6;              // Armijo candidates of a wide line-search window
constexpr int NPART = 32;          // per-CTA partial slots (packed: Ls[nq], L1[nq], Delta, |T|)
constexpr int WREG = 4;            // bitmap words per thread kept in registers in phase C1
constexpr int NE_MAX = 64;         // heavy entries handled per round inside one CTA
constexpr int NREG = 8;            // rows with <= NREG records are folded by one thread
constexpr int SHORT = 8;           // columns with <= SHORT nonzeros are reduced by one thread
constexpr int MED_LEN = 128;       // ... with <= MED_LEN by one warp
constexpr int CTA_LEN = 2048;      // ... with <= CTA_LEN by one CTA in the HBM-state kernels (default)
constexpr int MIDQ = 256;          // per-CTA queue of such columns in one step
constexpr int NHW = 4;             // warps that fold rows with > NREG records
constexpr int HB = 1024;           // per-warp sort buffer for such rows
constexpr int TSM = 4096;          // touched samples of a row block kept in shared memory
constexpr int SCAN_TILE = 2048;    // items per CTA of the device-wide scans
constexpr int FMAX = 256;          // full columns of a step staged in shared memory
constexpr int TL_STEPS = 16;       // per-warp timeline (profiling mode 2): first steps of a launch
constexpr int TL_PTS = 16;         //   and points per step
constexpr int SCAN_NT = 256;

constexpr int LOSS_LOGISTIC = 0;
constexpr int LOSS_L2SVM = 1;
constexpr int LOSS_SQ = 2;         // squared loss (t_i - w'x_i)^2, Lasso / elastic net (reading Z26)

struct __align__(16) Rec {   // one contribution d_k x_ik to sample i, k = bundle position
    int32_t k;
    int32_t pad;
    double v;
};

struct __align__(16) HPart {  // CTA partial of a heavy column crossing CTA boundaries
    int64_t e;
    double g, h;
    double pad;
};

struct DFlag {   // a finished heavy column's direction d_j, published with the step's stamp
    unsigned long long stamp;
    double d;
};

struct StepArgs {
    // problem (immutable during the kernel)
    int64_t s, n;
    const int64_t *__restrict__ col_ptr;
    const int32_t *__restrict__ row_idx;
    const float *__restrict__ val;
    const int64_t *__restrict__ row_ptr;  // CSR offsets: capacity of each sample's record segment
    const int8_t *__restrict__ y;
    double c, sigma, beta, gamma, nu;
    double mu;   // elastic-net weight of (mu/2)||w||^2 (reading Z25; 0 = the paper's problem)
    const double *t;   // real targets of the squared loss (reading Z26), else unused
    int scdn;          // 1: SCDN (Alg.2, reading Z27) -- per-feature 1-D steps, no P-dim line search
    int loss, qmax;
    int heavy_len;
    const int *stop;   // nullable: set by an earlier outer boundary's stop test -> the launch exits at once
    // state
    double *w;
    double *z;
    double2 *coef;   // cached per-sample (G_i, H_i): grad_j = c sum x G, hess_jj = c sum x^2 H
    double *F;       // maintained objective (device scalar)
    int32_t *cnt;    // per-sample record count (zero between steps)
    uint32_t *bits;  // touched-sample bitmap (zero between steps)
    Rec *rec;        // per-sample record segments at row_ptr[i]
    double *dxg;     // d'x_i for i in T (valid only on T)
    int32_t *tlist;  // T, per row block, ascending
    // bundles of this launch
    const int32_t *__restrict__ order;  // feature id per position
    const int4 *__restrict__ colinfo;   // packed (j, length, col_ptr[j]) per position
    const int64_t *__restrict__ hpos;   // heavy positions before each position [ntot+1]
    const int32_t *__restrict__ hlist;  // heavy entry -> position
    const int4 *__restrict__ hdesc;     // heavy entry -> (position, j, col_ptr[j] lo, hi)
    const int64_t *__restrict__ hstart; // heavy entry -> global heavy-nnz offset [nheavy+1]
    const int64_t *__restrict__ fpos;   // full columns before each position [ntot+1]
    const int32_t *__restrict__ flist;  // full-column entry -> position
    int64_t ntot, P, nsteps;
    // per-step scratch
    double *dk, *deltak;  // [P] direction and Delta term per bundle position
    double *part;         // [2][G][NPART]
    HPart *hpart;         // [G][2]
    // outputs
    double *g_out, *h_out, *d_out;  // nullable [P] (single-step launches)
    int32_t *q_trace;
    double *F_trace;
    int64_t trace_off, trace_cap;
    int64_t *counters;   // [0]=steps [1]=null [2]=nnz [3]=touched [4]=positions
    double *info;        // last step: q, alpha, Delta, lhs, rhs, F, nnz, nT
    int debug;
    long long *prof;     // nullable: per-phase clock64 cycles of CTA 0 (profiling mode)
    long long *tl;       // nullable: per-warp timeline of CTA 0, [TL_STEPS][NW][TL_PTS] (profile 2)
    double *dbg_dx;
    uint8_t *dbg_mark;
    // cluster-resident variant (pcdn_resident.cuh): cluster of 2^res_lg CTAs, res_Bs samples
    // per CTA, res_cap records per CTA in shared memory; rec (as the overflow of received
    // records), rec2 (overflow segments) and rslot (overflow slots) are global spill regions
    int res_lg, res_Bs, res_cap;
    int res_off[8];   // byte offsets of the dynamic shared-memory arrays (ResLayout)
    Rec *rec2;
    uint32_t *rslot;
    int *ovf_cnt;   // [16] overflow records received per CTA in the current step
    double *part_gh;  // dense kernel: per-CTA partial (g, h) of every bundle column [G][P][2]
    int dense_tcap;   // dense kernel: floats per shared-memory tile buffer (two buffers)
    // dense kernel, whole solve in one launch (n_outer > 1): outer iteration oi uses positions
    // [oi&1]*n of order/colinfo (2n each); at every outer boundary the kernel recomputes F from
    // (z, w) exactly as k_obj, takes the Eq.14 stop test and builds the next partition itself
    int n_outer;
    int64_t outer0;   // outer iteration index of the launch's first (the partition stream's k)
    uint64_t seed;
    double eps_stop, fstar;
    double *objp;                 // [3 * OBJ_NB] objective partials
    int32_t *pflag, *pfflag;      // scratch for perm_positions
    int64_t *outers_done;
    // sparse kernel (pcdn_sparse.cuh): records at the CSR slot of each nonzero, heavy columns in chunks
    const uint32_t *cslot;   // CSR offset of each CSC nonzero [nnz]
    uint32_t *sbits;         // written-slot bitmap over the CSR offsets (zero between steps)
    double *rv;              // record value d_j x_ij at the CSR offset of (i, j)
    const int4 *cdesc;       // chunk descriptors of the list set (chunk_decode)
    const int64_t *cpos;     // chunks before each position [ntot+1]
    double2 *cpart;          // chunk partials (g, h) by chunk index within the step
    int *ccnt;               // arrivals per heavy entry (zero between steps)
    DFlag *dflag;            // finished direction per heavy entry, stamped
    unsigned long long stamp0;   // step t of this launch publishes stamp0 + t + 1
    // sync
    unsigned long long *bar;
    int *status;
};

// ------------------------------------------------------------------------------------
// small device helpers
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }
__device__ __forceinline__ double2 ldcg(const double2 *p) { return __ldcg(p); }
__device__ __forceinline__ int32_t ldcg(const int32_t *p) { return __ldcg(p); }
__device__ __forceinline__ uint32_t ldcg(const uint32_t *p) { return __ldcg(p); }
__device__ __forceinline__ int64_t ldcg(const int64_t *p) { return __ldcg((const long long *)p); }

__device__ __forceinline__ HPart ld_hpart(const HPart *p)
{
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a0 = __ldcg(q), a1 = __ldcg(q + 1);
    HPart r;
    r.e = __double_as_longlong(a0.x);
    r.g = a0.y;
    r.h = a1.x;
    r.pad = a1.y;
    return r;
}

__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Software grid barrier for a cooperative launch (all CTAs co-resident).  `target`
// advances by gridDim.x per barrier; the counter only grows within a launch.
__device__ __forceinline__ void bar_arrive_gpu(unsigned long long *ctr)
{
    __threadfence();          // release: the CTA's writes (ordered by the bar.sync before it)
    atomicAdd(ctr, 1ULL);
}
__device__ __forceinline__ void bar_wait_gpu(const unsigned long long *ctr, unsigned long long target)
{
    const long long t0 = clock64();
    while (ld_acquire(ctr) < target) {   // acquire: no trailing fence needed
        if (clock64() - t0 > 8000000000LL) __trap();   // a broken protocol: fail, do not hang
    }
}
__device__ __forceinline__ void grid_sync(unsigned long long *ctr, unsigned long long &target)
{
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        bar_arrive_gpu(ctr);
        bar_wait_gpu(ctr, target);
    }
    __syncthreads();
}

// Sync policies of the persistent step kernel.  GridSync: cooperative launch of G CTAs (up to
// 2 per SM), software barrier through an L2 counter.  ClusterSync: one thread-block cluster of
// G <= 16 CTAs, hardware cluster barrier (release/acquire at cluster scope covers the global
// memory the phases exchange).
struct GridSync {
    static constexpr int kMinBlocks = 1;
    unsigned long long *ctr;
    unsigned long long target;
    __device__ __forceinline__ explicit GridSync(unsigned long long *c) : ctr(c), target(0) {}
    __device__ __forceinline__ void sync() { grid_sync(ctr, target); }
    // split barrier: arrive (the CTA's prior writes released), independent work, then wait
    __device__ __forceinline__ void arrive()
    {
        target += gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) bar_arrive_gpu(ctr);
    }
    __device__ __forceinline__ void wait()
    {
        if (threadIdx.x == 0) bar_wait_gpu(ctr, target);
        __syncthreads();
    }
};

struct ClusterSync {
    static constexpr int kMinBlocks = 1;
    __device__ __forceinline__ explicit ClusterSync(unsigned long long *) {}
    __device__ __forceinline__ void sync()
    {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    __device__ __forceinline__ void arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
    // the trailing CTA barrier orders the work done between arrive and wait (by some warps of this
    // CTA) before everything after the wait, as GridSync::wait does
    __device__ __forceinline__ void wait()
    {
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        __syncthreads();
    }
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// SplitMix64 finalizer; the partition generator of reading Z2.
__device__ __forceinline__ uint64_t mix64(uint64_t x)
{
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

// Per-sample factors (G, H) of Eq.13 (logistic) and App. A.2 (L2-SVM,
// PAPER.md:825-829, gradient per reading Z5).  sigma(+-m) evaluated without overflow.
__device__ __forceinline__ double2 coef_of(int loss, double z, int yi)
{
    const double yd = (double)yi;
    if (loss == LOSS_LOGISTIC) {
        const double m = yd * z;
        const double e = exp(-fabs(m));   // one exp: exp(-m) for m >= 0, exp(m) below
        const double q1 = 1.0 / (1.0 + e), q2 = e / (1.0 + e);
        const double sm = m >= 0 ? q1 : q2, snm = m >= 0 ? q2 : q1;
        return make_double2(-snm * yd, sm * snm);
    }
    const double b = 1.0 - yd * z;
    if (b > 0) return make_double2(-2.0 * yd * b, 2.0);
    return make_double2(0.0, 0.0);
}

// The per-sample factors after a step alpha*dx from (z, cf_old): the squared loss's G = 2(z - t) is
// linear in z, so it is carried forward by adding 2 alpha dx (no target needed; Z26); the other
// losses re-evaluate at the new z.
__device__ __forceinline__ double2 coef_next(int loss, double2 cf_old, double z_new, double adx, int yi)
{
    if (loss == LOSS_SQ) return make_double2(cf_old.x + 2.0 * adx, 2.0);
    return coef_of(loss, z_new, yi);
}

__device__ __forceinline__ double softplus(double t) { return (t > 0 ? t : 0.0) + log1p(exp(-fabs(t))); }

// phi(m), Eq.2 / Eq.3 (overflow-safe, reading Z19)
__device__ __forceinline__ double phi_of(int loss, double m)
{
    if (loss == LOSS_LOGISTIC) return softplus(-m);
    const double b = 1.0 - m;
    return b > 0 ? b * b : 0.0;
}

// Per-sample loss change at step alpha (reading Z7).  For the logistic loss sigma(-m) is taken
// from the cached factor: G = -sigma(-m) y  =>  sigma(-m) = -G y (exact).
// The logistic branch is out of line: its log1p / expm1 / softplus bodies are large, and one shared
// copy keeps the step kernels' hot instruction footprint small (they are latency-bound loops).
// (Inlining it in the sparse kernel's fold, next to the speculative commit's factors so that the
// two transcendental chains could interleave, measured slower: config 5 LR P = 4096 20.37 ->
// 20.72 us per step, profiles/r2c/ab_inl.)
__device__ __noinline__ double lr_loss_change(double m, double u, double snm)
{
    if (fabs(u) <= 1.0) return log1p(expm1(-u) * snm);
    return softplus(-(m + u)) - softplus(-m);
}

__device__ __forceinline__ double loss_change(int loss, double z, int yi, double cg, double dx, double alpha)
{
    const double yd = (double)yi;
    if (loss == LOSS_LOGISTIC) return lr_loss_change(yd * z, alpha * (yd * dx), -cg * yd);
    if (loss == LOSS_SQ) {   // (t - z - a)^2 - (t - z)^2 = a (a + 2(z - t)) = a (a + G), a = alpha dx (Z26)
        const double u = alpha * dx;
        return u * (u + cg);
    }
    const double b1 = 1.0 - yd * (z + alpha * dx);
    const double b0 = 1.0 - yd * z;
    const double p1 = b1 > 0 ? b1 * b1 : 0.0;
    const double p0 = b0 > 0 ? b0 * b0 : 0.0;
    return p1 - p0;
}

// Eq.5, branches tested in printed order (reading Z17).
__device__ __forceinline__ double newton_dir(double g, double h, double wj)
{
    const double hw = h * wj;
    if (g + 1.0 <= hw) return -(g + 1.0) / h;
    if (g - 1.0 >= hw) return -(g - 1.0) / h;
    return -wj;
}

// Finish one feature: c-scaling, nu floor (reading Z4), d_j (Eq.5), Delta term (Eq.7).
struct Dir {
    double g, h, d, delta;
};
__device__ __forceinline__ Dir finish_feature(const StepArgs &a, double gs, double hs, double wj)
{
    Dir r;
    r.g = a.c * gs + a.mu * wj;   // + the elastic-net gradient / curvature (Z25)
    r.h = a.c * hs + a.mu;
    if (!(r.h > a.nu)) r.h = a.nu;
    r.d = newton_dir(r.g, r.h, wj);
    r.delta = r.g * r.d + a.gamma * r.h * r.d * r.d + fabs(wj + r.d) - fabs(wj);
    return r;
}

// Record one contribution d_k x_ik of bundle position k to sample i (a3).  The slot inside the
// sample's segment comes from an integer atomic; the fold in phase C sorts by k, so the slot
// order never reaches the arithmetic.
__device__ __forceinline__ void emit(const StepArgs &a, int32_t i, int32_t k, double v)
{
    const int32_t slot = atomicAdd(&a.cnt[i], 1);
    Rec r;
    r.k = k;
    r.pad = 0;
    r.v = v;
    __stcg(reinterpret_cast<double2 *>(&a.rec[__ldg(&a.row_ptr[i]) + slot]),
           *reinterpret_cast<double2 *>(&r));
    if (slot == 0) atomicOr(&a.bits[i >> 5], 1u << (i & 31));
}

// ------------------------------------------------------------------------------------
// a0: partition (Eq.8, Alg.3 l.4, reading Z2)
// ------------------------------------------------------------------------------------
struct FeistelKeys {
    uint64_t key[8];
    uint64_t mask;
    int hb;
};

__device__ __forceinline__ FeistelKeys feistel_keys(uint64_t seed, int64_t k, int64_t n)
{
    FeistelKeys f;
    int bits = 0;
    while (bits < 63 && ((int64_t)1 << bits) < n) bits++;
    f.hb = (bits + 1) / 2;
    if (f.hb < 1) f.hb = 1;
    f.mask = ((uint64_t)1 << f.hb) - 1;
    const uint64_t base = mix64(seed ^ 0x6A09E667F3BCC909ULL);
    const uint64_t kk = mix64(base ^ (uint64_t)k);
#pragma unroll
    for (int r = 0; r < 8; r++) f.key[r] = mix64(kk + (uint64_t)(r + 1) * 0x9E3779B97F4A7C15ULL);
    return f;
}

__device__ __forceinline__ int64_t feistel_perm(const FeistelKeys &f, int64_t n, int64_t t)
{
    uint64_t x = (uint64_t)t;
    do {
        uint64_t L = x >> f.hb, R = x & f.mask;
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const uint64_t nr = L ^ (mix64(f.key[r] ^ R) & f.mask);
            L = R;
            R = nr;
        }
        x = (L << f.hb) | R;
    } while (x >= (uint64_t)n);
    return (int64_t)x;
}

// packed per-position column descriptor: (feature j, column length, col_ptr[j] lo, hi) -- one
// 16-byte load gives the step kernel everything it needs to issue a column's loads
__device__ __forceinline__ int4 make_colinfo(int32_t j, int64_t p0, int64_t len)
{
    return make_int4(j, (int)len, (int)(uint32_t)(p0 & 0xffffffffLL), (int)(p0 >> 32));
}
__device__ __forceinline__ int64_t colinfo_p0(const int4 &ci)
{
    return (int64_t)(((uint64_t)(uint32_t)ci.w << 32) | (uint64_t)(uint32_t)ci.z);
}

// Chunks of the sparse step kernel (pcdn_sparse.cuh): a column longer than heavy_len is reduced by
// whole CTAs in chunks of SP_CTA_MUL * max(heavy_len, SP_CHMIN) nonzeros (a warp's share of a chunk
// is then about a medium column), the last chunk to arrive finishes the column.  So the
// descriptor array of a list set needs at most nnz/SP_CHMIN + n entries; a column has at most
// SP_NCHMAX chunks (the finishing warp sums <= 16 partials per lane).
constexpr int SP_CHMIN = 4;
constexpr int SP_CTA_MUL = 12;   // = the warps of a sparse-kernel CTA (pcdn_sparse.cuh)
constexpr int SP_NCHMAX = 512;
__host__ __device__ __forceinline__ int chunk_count(int64_t len, int heavy_len)
{
    if (len <= heavy_len) return 0;
    const int64_t ch = (int64_t)SP_CTA_MUL * (heavy_len > SP_CHMIN ? heavy_len : SP_CHMIN);
    const int64_t c = (len + ch - 1) / ch;
    return (int)(c < SP_NCHMAX ? c : SP_NCHMAX);
}
// descriptor of chunk c of nch of heavy entry e over nonzeros [pb, pb + clen):
// (e, c | nch << 10 | full << 20, pb lo, pb hi (8 bits) | clen << 8)
__host__ __device__ __forceinline__ int64_t chunk_begin(int64_t cs, int64_t len, int c, int nch)
{
    return cs + (int64_t)c * len / nch;
}
__device__ __forceinline__ void write_chunks(int4 *out, int32_t e, int nch, int64_t cs, int64_t len, bool full)
{
    for (int c = 0; c < nch; c++) {
        const int64_t pb = chunk_begin(cs, len, c, nch), pe = chunk_begin(cs, len, c + 1, nch);
        out[c] = make_int4(e, c | (nch << 10) | ((full ? 1 : 0) << 20), (int)(uint32_t)(pb & 0xffffffffLL),
                           (int)(uint32_t)(((uint64_t)pb >> 32) & 0xffu) | (int)((uint32_t)(pe - pb) << 8));
    }
}
struct ChunkDesc {
    int32_t e;
    int c, nch;
    bool full;
    int64_t pb, len;
};
__device__ __forceinline__ ChunkDesc chunk_decode(const int4 &d)
{
    ChunkDesc r;
    r.e = d.x;
    r.c = d.y & 1023;
    r.nch = (d.y >> 10) & 1023;
    r.full = ((d.y >> 20) & 1) != 0;
    r.pb = (int64_t)(((uint64_t)((uint32_t)d.w & 0xffu) << 32) | (uint64_t)(uint32_t)d.z);
    r.len = (int64_t)((uint32_t)d.w >> 8);
    return r;
}

// order[t] = pi_k(t); flag[t] = column length > heavy_len; fflag[t] = column is full (holds a
// nonzero in every row: its entry for row i sits at col_ptr[j] + i); colinfo[t] (nullable)
// (t0, stride: this thread's first position and the stride; by default the grid-stride order)
__device__ __forceinline__ void perm_positions(uint64_t seed, int64_t k, int64_t n, int64_t s,
                                               const int64_t *__restrict__ col_ptr, int heavy_len, int32_t *order,
                                               int32_t *flag, int32_t *fflag, int4 *colinfo, int64_t t0 = -1,
                                               int64_t stride = 0)
{
    const FeistelKeys f = feistel_keys(seed, k, n);
    if (t0 < 0) {
        t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        stride = (int64_t)gridDim.x * blockDim.x;
    }
    for (int64_t t = t0; t < n; t += stride) {
        const int64_t j = feistel_perm(f, n, t);
        order[t] = (int32_t)j;
        if (flag) {
            const int64_t p0 = __ldg(&col_ptr[j]), len = __ldg(&col_ptr[j + 1]) - p0;
            flag[t] = len > heavy_len ? 1 : 0;
            fflag[t] = len == s ? 1 : 0;
            if (colinfo) colinfo[t] = make_colinfo((int32_t)j, p0, len);
        }
    }
}

__global__ void k_perm(uint64_t seed, int64_t k, int64_t n, int64_t s, const int64_t *__restrict__ col_ptr,
                       int heavy_len, int32_t *order, int32_t *flag, int32_t *fflag, int4 *colinfo)
{
    perm_positions(seed, k, n, s, col_ptr, heavy_len, order, flag, fflag, colinfo);
}

// full-column compaction: flist[e] = position of the e-th full column (fpos = exclusive scan)
__global__ void k_full_compact(const int64_t *__restrict__ fpos, int64_t ntot, int32_t *flist)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntot; t += (int64_t)gridDim.x * blockDim.x)
        if (fpos[t + 1] != fpos[t]) flist[fpos[t]] = (int32_t)t;
}

// user bundle: validate (distinct, in range) and copy
__global__ void k_bundle_prep(const int32_t *__restrict__ bundle, int64_t P, int64_t n, int64_t s,
                              const int64_t *__restrict__ col_ptr, int heavy_len, int32_t *order,
                              int32_t *flag, int32_t *fflag, uint32_t *seen, int *status, long long *err_idx,
                              unsigned long long *bundle_nnz, int4 *colinfo)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < P; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = bundle[t];
        if (j < 0 || j >= n) {
            atomicMax(status, 1);
            atomicMin(err_idx, (long long)t);
            order[t] = 0;
            flag[t] = 0;
            fflag[t] = 0;
            colinfo[t] = make_colinfo(0, 0, 0);
            continue;
        }
        const uint32_t bit = 1u << (j & 31);
        const uint32_t old = atomicOr(&seen[j >> 5], bit);
        if (old & bit) {
            atomicMax(status, 1);
            atomicMin(err_idx, (long long)t);
        }
        order[t] = j;
        const int64_t p0 = __ldg(&col_ptr[j]), len = __ldg(&col_ptr[j + 1]) - p0;
        flag[t] = len > heavy_len ? 1 : 0;
        fflag[t] = len == s ? 1 : 0;
        colinfo[t] = make_colinfo(j, p0, len);
        atomicAdd(bundle_nnz, (unsigned long long)len);   // integer: order-independent
    }
}

__global__ void k_bundle_unseen(const int32_t *__restrict__ bundle, int64_t P, int64_t n, uint32_t *seen)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < P; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = bundle[t];
        if (j >= 0 && j < n) seen[j >> 5] = 0;
    }
}

// ------------------------------------------------------------------------------------
// device-wide exclusive scan (reduce -> scan of tile sums -> apply).  out[n] = total.
// `n_dev` (nullable) bounds n at run time (launch sized for the host-side upper bound).
// ------------------------------------------------------------------------------------
template <typename Tin, typename Tout>
__device__ __forceinline__ Tout scan_load(const Tin *in, const int32_t *hlen_pos, int64_t i)
{
    return (Tout)in[i];
}

template <typename Tin, typename Tout>
__global__ void k_scan_reduce(const Tin *__restrict__ in, int64_t n, const int64_t *n_dev, Tout *tile_sum)
{
    if (n_dev) n = min(n, *n_dev);
    const int64_t t0 = (int64_t)blockIdx.x * SCAN_TILE;
    Tout s = 0;
    for (int64_t i = t0 + threadIdx.x; i < min(n, t0 + SCAN_TILE); i += SCAN_NT) s += (Tout)in[i];
    s = warp_sum(s);
    __shared__ Tout ws[SCAN_NT / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        Tout tot = 0;
        for (int w = 0; w < SCAN_NT / 32; w++) tot += ws[w];
        tile_sum[blockIdx.x] = tot;
    }
}

template <typename Tout>
__global__ void k_scan_tiles(Tout *tile_sum, int64_t ntiles)
{
    // single CTA, exclusive scan in place; sequential chunks of SCAN_NT
    __shared__ Tout sh[SCAN_NT];
    __shared__ Tout carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b = 0; b < ntiles; b += SCAN_NT) {
        const int64_t i = b + threadIdx.x;
        const Tout v = i < ntiles ? tile_sum[i] : 0;
        sh[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < SCAN_NT; o <<= 1) {
            const Tout t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
            __syncthreads();
            sh[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < ntiles) tile_sum[i] = carry + sh[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += sh[SCAN_NT - 1];
        __syncthreads();
    }
}

template <typename Tin, typename Tout>
__global__ void k_scan_apply(const Tin *__restrict__ in, int64_t n, const int64_t *n_dev,
                             const Tout *__restrict__ tile_sum, Tout *out, int64_t *total_out)
{
    if (n_dev) n = min(n, *n_dev);
    const int64_t t0 = (int64_t)blockIdx.x * SCAN_TILE;
    if (t0 >= n && !(t0 == 0)) return;
    constexpr int IPT = SCAN_TILE / SCAN_NT;  // items per thread, contiguous
    Tout v[IPT];
    Tout s = 0;
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const int64_t i = t0 + (int64_t)threadIdx.x * IPT + r;
        v[r] = i < n ? (Tout)in[i] : 0;
        s += v[r];
    }
    // block exclusive scan of s
    __shared__ Tout sh[SCAN_NT];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < SCAN_NT; o <<= 1) {
        const Tout t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
        __syncthreads();
        sh[threadIdx.x] += t;
        __syncthreads();
    }
    Tout run = tile_sum[blockIdx.x] + sh[threadIdx.x] - s;
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const int64_t i = t0 + (int64_t)threadIdx.x * IPT + r;
        if (i < n) out[i] = run;
        run += v[r];
        if (i == n - 1) {
            out[n] = run;
            if (total_out) *total_out = (int64_t)run;
        }
    }
    if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
        out[0] = 0;
        if (total_out) *total_out = 0;
    }
}

// heavy compaction: for flagged positions, hlist[e] = position, hlen[e] = column length
// hdesc[e] = packed (position, feature j, col_ptr[j]) of heavy entry e: one load in the kernels
__global__ void k_heavy_compact(const int64_t *__restrict__ hpos, int64_t ntot, const int32_t *__restrict__ order,
                                const int64_t *__restrict__ col_ptr, int32_t *hlist, int64_t *hlen, int4 *hdesc)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = hpos[t];
        if (hpos[t + 1] != e) {
            const int32_t j = order[t];
            const int64_t cs = __ldg(&col_ptr[j]);
            hlist[e] = (int32_t)t;
            hlen[e] = __ldg(&col_ptr[j + 1]) - cs;
            hdesc[e] = make_int4((int)t, j, (int)(uint32_t)(cs & 0xffffffffLL), (int)(cs >> 32));
        }
    }
}

// chunk counts per position (the reference build of the sparse kernel's chunk lists)
__global__ void k_chunk_count(const int4 *__restrict__ colinfo, int64_t ntot, int heavy_len, int32_t *cnt)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntot; t += (int64_t)gridDim.x * blockDim.x)
        cnt[t] = chunk_count(colinfo[t].y, heavy_len);
}

// chunk descriptors of every heavy position (cpos = exclusive scan of k_chunk_count, hpos = heavy
// entry numbers)
__global__ void k_chunk_compact(const int64_t *__restrict__ cpos, const int64_t *__restrict__ hpos,
                                const int4 *__restrict__ colinfo, int64_t ntot, int64_t s, int4 *cdesc)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntot; t += (int64_t)gridDim.x * blockDim.x) {
        const int nch = (int)(cpos[t + 1] - cpos[t]);
        if (nch > 0) {
            const int4 ci = colinfo[t];
            write_chunks(cdesc + cpos[t], (int32_t)hpos[t], nch, colinfo_p0(ci), ci.y, ci.y == s);
        }
    }
}

// a0 in one launch: the permutation pi_k of a whole outer iteration and the lists the step kernels
// read -- column descriptors, heavy-column lists (hpos, hlist, hdesc, hstart) and full-column
// lists (fpos, flist) -- with the three position-order prefix sums taken by a single-pass scan
// (tiles claimed in order from a ticket; decoupled look-back over the tiles' published aggregate /
// inclusive sums; integer sums, so exact).  The output equals k_perm + build_heavy's twelve
// launches.  Tile states carry the launch's epoch, so they need no clearing between launches; the
// last tile to finish re-arms the ticket.
constexpr int PL_NT = 256, PL_PER = 8, PL_TILE = PL_NT * PL_PER;   // (8 positions per thread: their col_ptr loads in flight together)
constexpr int PL_Q = 4;   // prefix sums of the list build: heavy count, heavy nnz, full count, chunk count
struct alignas(64) LbTile {
    long long agg[PL_Q];   // the tile's sums
    long long inc[PL_Q];   // the same, inclusive of every earlier tile
    unsigned flag;         // epoch << 2 | 1 (agg valid) or | 2 (inc valid)
};
struct PrepLists {
    int32_t *order;
    int4 *colinfo;
    int64_t *hpos, *hstart, *fpos, *nheavy;
    int32_t *hlist, *flist;
    int4 *hdesc;
    int64_t *cpos;   // chunks of the sparse kernel before each position [n+1]
    int4 *cdesc;     // chunk descriptors (chunk_desc)
    LbTile *lb;
    unsigned *ticket;   // [0] next tile, [1] tiles done
};
__global__ void __launch_bounds__(PL_NT) k_prep_lists(uint64_t seed, int64_t k, int64_t n, int64_t s,
                                                      const int64_t *__restrict__ col_ptr, int heavy_len,
                                                      unsigned epoch, PrepLists o)
{
    __shared__ unsigned s_tile;
    __shared__ long long s_w[PL_Q][PL_NT / 32];
    __shared__ long long s_pre[PL_Q];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned ntiles = (unsigned)((n + PL_TILE - 1) / PL_TILE);
    if (tid == 0) s_tile = atomicAdd(&o.ticket[0], 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const FeistelKeys f = feistel_keys(seed, k, n);
    // this thread's PL_PER consecutive positions
    int32_t jv[PL_PER];
    int64_t p0v[PL_PER], lenv[PL_PER];
    long long v[PL_Q] = {0, 0, 0, 0};
    const int64_t tb = (int64_t)tile * PL_TILE + (int64_t)tid * PL_PER;
#pragma unroll
    for (int e = 0; e < PL_PER; e++) jv[e] = tb + e < n ? (int32_t)feistel_perm(f, n, tb + e) : 0;
    int64_t p1v[PL_PER];
#pragma unroll
    for (int e = 0; e < PL_PER; e++) {
        p0v[e] = tb + e < n ? __ldg(&col_ptr[jv[e]]) : 0;
        p1v[e] = tb + e < n ? __ldg(&col_ptr[jv[e] + 1]) : -1;
    }
#pragma unroll
    for (int e = 0; e < PL_PER; e++) {
        const int64_t t = tb + e;
        lenv[e] = -1;
        if (t < n) {
            const int32_t j = jv[e];
            const int64_t p0 = p0v[e], len = p1v[e] - p0;
            lenv[e] = len;
            o.order[t] = j;
            o.colinfo[t] = make_colinfo(j, p0, len);
            if (len > heavy_len) {
                v[0] += 1;
                v[1] += len;
                v[3] += chunk_count(len, heavy_len);
            }
            if (len == s) v[2] += 1;
        }
    }
    // block exclusive scan of v (warp shuffles, then the warp totals)
    long long inc[PL_Q] = {v[0], v[1], v[2], v[3]};
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int q = 0; q < PL_Q; q++) {
            const long long u = __shfl_up_sync(0xffffffffu, inc[q], d);
            if (lane >= d) inc[q] += u;
        }
    }
    if (lane == 31)
        for (int q = 0; q < PL_Q; q++) s_w[q][warp] = inc[q];
    __syncthreads();
    long long wpre[PL_Q] = {0, 0, 0, 0}, tot[PL_Q] = {0, 0, 0, 0};
    for (int w2 = 0; w2 < PL_NT / 32; w2++)
        for (int q = 0; q < PL_Q; q++) {
            if (w2 < warp) wpre[q] += s_w[q][w2];
            tot[q] += s_w[q][w2];
        }
    // publish the aggregate, look back (warp 0, 32 tiles at a time), publish the inclusive sum
    if (warp == 0) {
        LbTile &me = o.lb[tile];
        if (lane == 0) {
            for (int q = 0; q < PL_Q; q++) me.agg[q] = tot[q];
            if (tile == 0)
                for (int q = 0; q < PL_Q; q++) me.inc[q] = tot[q];
            __threadfence();
            *(volatile unsigned *)&me.flag = (epoch << 2) | (tile == 0 ? 2u : 1u);
        }
        long long pre[PL_Q] = {0, 0, 0, 0};
        long long base = (long long)tile - 1;
        while (base >= 0) {
            const long long i = base - lane;
            unsigned st = 2u;   // before tile 0: an inclusive sum of zero
            long long val[PL_Q] = {0, 0, 0, 0};
            if (i >= 0) {
                const volatile unsigned *fp = &o.lb[i].flag;
                unsigned fl;
                do {
                    fl = *fp;
                } while ((fl >> 2) != epoch || (fl & 3u) == 0u);
                st = fl & 3u;
                __threadfence();
                const long long *src = st == 2u ? o.lb[i].inc : o.lb[i].agg;
                for (int q = 0; q < PL_Q; q++) val[q] = __ldcg(&src[q]);
            }
            const unsigned pm = __ballot_sync(0xffffffffu, st == 2u);
            const int lp = pm ? __ffs(pm) - 1 : 32;   // the nearest tile with an inclusive sum
            for (int q = 0; q < PL_Q; q++) {
                long long x = lane <= lp ? val[q] : 0;
                for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
                pre[q] += x;
            }
            if (pm) break;
            base -= 32;
        }
        if (lane == 0) {
            if (tile != 0) {
                for (int q = 0; q < PL_Q; q++) me.inc[q] = pre[q] + tot[q];
                __threadfence();
                *(volatile unsigned *)&me.flag = (epoch << 2) | 2u;
            }
            for (int q = 0; q < PL_Q; q++) s_pre[q] = pre[q];
        }
    }
    __syncthreads();
    long long run[PL_Q];
    for (int q = 0; q < PL_Q; q++) run[q] = s_pre[q] + wpre[q] + inc[q] - v[q];   // exclusive, at tb
#pragma unroll
    for (int e = 0; e < PL_PER; e++) {
        const int64_t t = tb + e;
        if (t >= n) break;
        o.hpos[t] = run[0];
        o.fpos[t] = run[2];
        o.cpos[t] = run[3];
        const int64_t len = lenv[e];
        if (len > heavy_len) {
            const int64_t cs = p0v[e];
            o.hlist[run[0]] = (int32_t)t;
            o.hdesc[run[0]] = make_int4((int)t, jv[e], (int)(uint32_t)(cs & 0xffffffffLL), (int)(cs >> 32));
            o.hstart[run[0]] = run[1];
            const int nch = chunk_count(len, heavy_len);
            write_chunks(o.cdesc + run[3], (int32_t)run[0], nch, cs, len, len == s);
            run[0] += 1;
            run[1] += len;
            run[3] += nch;
        }
        if (len == s) {
            o.flist[run[2]] = (int32_t)t;
            run[2] += 1;
        }
        if (t == n - 1) {   // the totals
            o.hpos[n] = run[0];
            o.fpos[n] = run[2];
            o.cpos[n] = run[3];
            o.hstart[run[0]] = run[1];
            *o.nheavy = run[0];
        }
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&o.ticket[1], 1u) == ntiles - 1) {   // every tile claimed and finished
            o.ticket[0] = 0u;
            o.ticket[1] = 0u;
        }
    }
}

// ------------------------------------------------------------------------------------
// a1..a5: the persistent bundle-step kernel
// ------------------------------------------------------------------------------------
// The heavy-column work of one CTA in one step: entries [e_lo, e_hi) of the step, heavy nonzero
// offsets relative to hb0, NH in total, this CTA's range [lo_c, hi_c) and the entries [ce0, ce1)
// overlapping it.  Static per launch, so it is computed a step ahead by an otherwise idle warp.
struct HeavyPlan {
    int64_t e_lo, e_hi, hb0, NH, ce0, ce1;
    int64_t f_lo, nf;   // the step's full columns: entries [f_lo, f_lo + nf) of flist
};

struct StepSmem {
    HeavyPlan plan[2];   // heavy-column plan of this and the next step (by step parity)
    int32_t midq[MIDQ];  // positions of this CTA's CTA-level columns in the step
    int nmid;
    // heavy-column rounds
    int64_t hst[NE_MAX + 1];
    double hg[NE_MAX][NW];
    double hh[NE_MAX][NW];
    double hd[NE_MAX];
    int64_t ce0, ce1;
    int64_t cross_e[2];
    double cross_d[2];
    // reductions
    double red[NW][32];
    double tot[32];
    int64_t scan_w[NW];
    int64_t nT;
    int has_heavy_rows;
    int q_acc;
    // CTA 0 bookkeeping (maintained F, step counters) and profile counters
    double F;
    long long cnt[4];
    long long pacc[16];
    // line-search decision broadcast
    int dec_q, dec_bad;
    double dec_alpha, dec_lhs, dec_rhs, dec_Delta, dec_nT;
    // full columns of the step (d, col_ptr[j]), the first FMAX of them, and their d'x part for the
    // rows of the block (dense pass, when the block has <= TSM rows)
    double fd[FMAX];
    int64_t fcp[FMAX];
    double dxd[TSM];
    int64_t row_base;
    // touched samples of the row block (when they fit)
    int32_t tl[TSM];
    // rows with > NREG records: per-warp sort buffers
    int32_t sk[NHW][HB];
    double sv[NHW][HB];
};

// Warp-level gh over columns' nonzeros [p0, p1): lanes strided, fixed xor tree.  The nonzeros of a
// lane are taken in batches of B: the B index/value loads, then the B gathers they address, all in
// flight together (a plain unrolled loop left each gather waiting on its own index load); the
// per-lane summation order (ascending p) is unchanged.  full_base >= 0: the column is full, its
// row index is p - full_base (no index load).
template <int B = 8>
__device__ __forceinline__ void col_gh(const StepArgs &a, int64_t p0, int64_t p1, int lane, double &gs, double &hs,
                                       int64_t full_base = -1)
{
    double g = 0.0, h = 0.0;
    for (int64_t pb = p0 + lane; pb < p1; pb += 32 * B) {
        int32_t ri[B];
        float xv[B];
#pragma unroll
        for (int e = 0; e < B; e++) {
            const int64_t p = pb + 32 * e;
            ri[e] = -1;
            xv[e] = 0.f;
            if (p < p1) {
                ri[e] = full_base >= 0 ? (int32_t)(p - full_base) : __ldg(&a.row_idx[p]);
                xv[e] = __ldg(&a.val[p]);
            }
        }
        double2 cf[B];
#pragma unroll
        for (int e = 0; e < B; e++) cf[e] = ri[e] >= 0 ? ldcg(&a.coef[ri[e]]) : make_double2(0.0, 0.0);
#pragma unroll
        for (int e = 0; e < B; e++) {
            if (ri[e] >= 0) {
                const double x = (double)xv[e];
                g += x * cf[e].x;
                h += (x * x) * cf[e].y;
            }
        }
    }
    gs = warp_sum(g);
    hs = warp_sum(h);
}

// N records of one thread at once: all slot atomics (and segment offsets) in flight together,
// then the stores -- one emit() after another would serialise on each atomic's return.
template <int N>
__device__ __forceinline__ void emit_batch(const StepArgs &a, const int32_t (&ri)[N], const double (&v)[N], int nv,
                                           int32_t k)
{
    int32_t slot[N];
    int64_t off[N];
#pragma unroll
    for (int e = 0; e < N; e++) {
        slot[e] = 0;
        off[e] = 0;
        if (e < nv) {
            slot[e] = atomicAdd(&a.cnt[ri[e]], 1);
            off[e] = __ldg(&a.row_ptr[ri[e]]);
        }
    }
#pragma unroll
    for (int e = 0; e < N; e++) {
        if (e < nv) {
            Rec r;
            r.k = k;
            r.pad = 0;
            r.v = v[e];
            __stcg(reinterpret_cast<double2 *>(&a.rec[off[e] + slot[e]]), *reinterpret_cast<double2 *>(&r));
            if (slot[e] == 0) atomicOr(&a.bits[ri[e] >> 5], 1u << (ri[e] & 31));
        }
    }
}

__device__ __forceinline__ void col_scatter(const StepArgs &a, int64_t p0, int64_t p1, int lane, int32_t kpos, double d)
{
    constexpr int B = 4;   // records per lane per batch
    for (int64_t pb = p0 + lane; pb < p1; pb += 32 * B) {
        int32_t ri[B];
        double v[B];
        int nv = 0;
#pragma unroll
        for (int e = 0; e < B; e++) {
            const int64_t p = pb + 32 * e;
            ri[e] = 0;
            v[e] = 0.0;
            if (p < p1) {
                ri[e] = __ldg(&a.row_idx[p]);
                v[e] = d * (double)__ldg(&a.val[p]);
                nv = e + 1;
            }
        }
        emit_batch<B>(a, ri, v, nv, kpos);
    }
}

// First e in [lo, hi) with pred(e) true (pred monotone: false..false true..true), hi if none.
// All 32 lanes probe evenly spaced candidates, so each round narrows the range 32-fold.
template <class Pred>
__device__ __forceinline__ int64_t warp_first(int64_t lo, int64_t hi, int lane, Pred pred)
{
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t e = lo + (int64_t)lane * step;
        const unsigned m = __ballot_sync(0xffffffffu, e < hi ? pred(e) : true);
        if (m == 0) {               // false up to lo + 31*step
            lo = lo + 31 * step + 1;
            continue;
        }
        const int f = __ffs(m) - 1;
        if (f == 0) return lo;      // pred(lo)
        // false at lo + (f-1)*step, true at lo + f*step (or beyond hi)
        const int64_t nhi = min(hi, lo + (int64_t)f * step);
        lo = lo + (int64_t)(f - 1) * step + 1;
        hi = nhi;
    }
    const int64_t e = lo + lane;
    const unsigned m = __ballot_sync(0xffffffffu, e < hi ? pred(e) : true);
    return m == 0 ? hi : min(hi, lo + (int64_t)(__ffs(m) - 1));
}


__device__ __forceinline__ void heavy_plan_warp(const StepArgs &a, int64_t k0, int64_t k1, int c, int G, int lane,
                                                HeavyPlan *out)
{
    HeavyPlan hp;
    hp.e_lo = __ldg(&a.hpos[k0]);
    hp.e_hi = __ldg(&a.hpos[k1]);
    hp.f_lo = __ldg(&a.fpos[k0]);
    hp.nf = __ldg(&a.fpos[k1]) - hp.f_lo;
    hp.hb0 = 0;
    hp.NH = 0;
    hp.ce0 = hp.ce1 = hp.e_lo;
    if (hp.e_hi > hp.e_lo) {
        hp.hb0 = __ldg(&a.hstart[hp.e_lo]);
        hp.NH = __ldg(&a.hstart[hp.e_hi]) - hp.hb0;
        const int64_t lo_c = (int64_t)c * hp.NH / G, hi_c = (int64_t)(c + 1) * hp.NH / G;
        const int64_t hb0 = hp.hb0;
        hp.ce0 = warp_first(hp.e_lo, hp.e_hi, lane, [&](int64_t e) { return __ldg(&a.hstart[e + 1]) - hb0 > lo_c; });
        hp.ce1 = warp_first(hp.ce0, hp.e_hi, lane, [&](int64_t e) { return __ldg(&a.hstart[e]) - hb0 >= hi_c; });
        if (!(hi_c > lo_c)) hp.ce1 = hp.ce0;
    }
    if (lane == 0) *out = hp;
}

// index of the CTA whose heavy range [floor(c NH/G), floor((c+1) NH/G)) holds offset o
__device__ __forceinline__ int cta_of(int64_t o, int64_t NH, int G)
{
    return (int)(((o + 1) * (int64_t)G - 1) / NH);
}

// Fold of one sample's records in ascending bundle position (<= NREG records): thread-level.
__device__ __forceinline__ double fold_small(const StepArgs &a, int64_t off, int ni)
{
    int kk[NREG];
    double vv[NREG];
#pragma unroll
    for (int r = 0; r < NREG; r++) {
        if (r < ni) {
            const double2 raw = __ldcg(reinterpret_cast<const double2 *>(&a.rec[off + r]));
            kk[r] = __double_as_longlong(raw.x) & 0xffffffffLL;
            vv[r] = raw.y;
        } else {
            kk[r] = 0x7fffffff;
            vv[r] = 0.0;
        }
    }
    double dx = 0.0;
    int last = -1;
#pragma unroll 1
    for (int t = 0; t < ni; t++) {
        int best = 0x7fffffff;
        double bv = 0.0;
#pragma unroll
        for (int r = 0; r < NREG; r++) {
            const bool take = kk[r] > last && kk[r] < best;
            best = take ? kk[r] : best;
            bv = take ? vv[r] : bv;
        }
        last = best;
        dx += bv;
    }
    // every record of a sample has its own bundle position: a repeat would have been dropped above
    // (and summed by the warp fold), so it is an internal error, never a silent fix
    if (last == 0x7fffffff) atomicMax(a.status, 6);
    return dx;
}

// Fold of one sample with > NREG records by a warp: bitonic sort by bundle position in shared
// memory, then lane-contiguous partial sums combined by a fixed tree (deterministic).
__device__ double fold_warp(const StepArgs &a, int64_t off, int ni, int32_t *sk, double *sv, int lane)
{
    if (ni <= HB) {
        int npow = 32;
        while (npow < ni) npow <<= 1;
        for (int r = lane; r < npow; r += 32) {
            if (r < ni) {
                const double2 raw = __ldcg(reinterpret_cast<const double2 *>(&a.rec[off + r]));
                sk[r] = (int32_t)(__double_as_longlong(raw.x) & 0xffffffffLL);
                sv[r] = raw.y;
            } else {
                sk[r] = 0x7fffffff;
                sv[r] = 0.0;
            }
        }
        __syncwarp();
        for (int kbit = 2; kbit <= npow; kbit <<= 1) {
            for (int jbit = kbit >> 1; jbit > 0; jbit >>= 1) {
                for (int r = lane; r < npow; r += 32) {
                    const int pr = r ^ jbit;
                    if (pr > r) {
                        const bool up = (r & kbit) == 0;
                        const int32_t k1 = sk[r], k2 = sk[pr];
                        if ((k1 > k2) == up) {
                            sk[r] = k2;
                            sk[pr] = k1;
                            const double t = sv[r];
                            sv[r] = sv[pr];
                            sv[pr] = t;
                        }
                    }
                }
                __syncwarp();
            }
        }
        const int chunk = (ni + 31) / 32;
        double s = 0.0;
        for (int r = lane * chunk; r < min(ni, (lane + 1) * chunk); r++) s += sv[r];
        // fixed-order tree over lanes (lane order preserved pairwise)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_down_sync(0xffffffffu, s, o);
            if ((lane & (2 * o - 1)) == 0) s += t;
        }
        __syncwarp();
        return __shfl_sync(0xffffffffu, s, 0);
    }
    // very long rows: repeated warp-wide min extraction (correct, O(ni^2/32))
    double dx = 0.0;
    int last = -1;
    for (int t = 0; t < ni; t++) {
        int best = 0x7fffffff;
        double bv = 0.0;
        for (int r = lane; r < ni; r += 32) {
            const double2 raw = __ldcg(reinterpret_cast<const double2 *>(&a.rec[off + r]));
            const int32_t k = (int32_t)(__double_as_longlong(raw.x) & 0xffffffffLL);
            if (k > last && k < best) {
                best = k;
                bv = raw.y;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int ob = __shfl_xor_sync(0xffffffffu, best, o);
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            if (ob < best) {
                best = ob;
                bv = ov;
            }
        }
        last = best;
        dx += bv;
    }
    return dx;
}

// ------------------------------------------------------------------------------------
// register-resident per-step data (prefetch / reuse across phases)
// ------------------------------------------------------------------------------------
constexpr int PF = 4;  // nonzeros per lane of a light column prefetched into registers

// The CTA's first bundle-share position (L1 term, Delta, w commit) and the thread's first
// touched sample (loss change, commit), kept in registers from the line search to the commit.
struct ShareReg {
    int64_t kk;  // -1 = none
    int32_t j;
    double wj, d, delta;
};
struct RowReg {
    int32_t i;  // -1 = none
    int yi;
    int has_dx;  // 0 when the sample had > NREG records (folded by a warp into dxg)
    double zi, dx;
    int64_t r0, r1;   // the sample's CSR segment (sparse kernel)
    double cg;        // the sample's cached G before the step (sparse kernel: speculative commit)
};

// ------------------------------------------------------------------------------------
// line-search window helpers
// ------------------------------------------------------------------------------------
// Transpose-reduce of W values per lane across a warp: after the call, lane l holds the warp
// total of slot l / (32 / W).  Fixed tree (deterministic); log2(W) halving levels exchange
// W/2, W/4, .. values, then single-value xor levels: W=8 costs 9 shuffles instead of 40.
template <int W>
__device__ __forceinline__ double xreduce(double (&v)[W], int lane)
{
    constexpr int LOGW = W == 2 ? 1 : W == 4 ? 2 : W == 8 ? 3 : W == 16 ? 4 : 5;
#pragma unroll
    for (int lvl = 0; lvl < 5; lvl++) {
        const int o = 16 >> lvl;
        if (lvl < LOGW) {
            const int half = W >> (lvl + 1);
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < W / 2; i++) {
                if (i < half) {
                    const double send = up ? v[i] : v[i + half];
                    const double keep = up ? v[i + half] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    return v[0];
}

// Totals of the G per-CTA partial rows part[c2][0..W) in a fixed order: warp w sums rows
// c2 = w, w+NW, ... (lanes = slots), then warp 0 adds the NW warp sums in warp order.  red is a
// [NW][32] shared scratch, tot the [32] shared result (valid after the __syncthreads inside).
template <int W>
__device__ __forceinline__ void grid_totals(const double *part, int G, double (*red)[32], double *tot, int lane,
                                            int warp)
{
    double v = 0.0;
    if (lane < W) {
#pragma unroll 4
        for (int c2 = warp; c2 < G; c2 += NW) v += ldcg(&part[(int64_t)c2 * NPART + lane]);
    }
    red[warp][lane] = v;
    __syncthreads();
    if (warp == 0 && lane < W) {
        double t = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < NW; w2++) t += red[w2][lane];
        tot[lane] = t;
    }
    __syncwarp();
}

struct WinState {
    int q0, nq, qacc, bad, win;
    int nospec;       // sparse kernel: some CTA did not commit speculatively in this window
    unsigned tmask;   // cluster-resident kernel: owned samples (bit r) touched in this step
    double alpha, lhs, rhs, Delta, nT_tot;
};

// The step's full columns (a nonzero in every row, so x_ij sits at col_ptr[j] + i): their d'x_i
// terms are read straight from CSC in bundle order instead of travelling as records (dense
// workloads would otherwise send every sample one record per bundle column).
struct DenseInfo {
    int64_t f_lo, nf;   // entries [f_lo, f_lo + nf) of flist
    bool any;           // some full column of the step has d_j != 0 (then every sample is in T)
};

__device__ __forceinline__ double dense_dx(const StepArgs &a, const double *fd, const int64_t *fcp, const DenseInfo &di,
                                           int64_t k0, int64_t i)
{
    double dx = 0.0;
    for (int64_t e = 0; e < di.nf; e++) {
        double d;
        int64_t cp;
        if (e < FMAX) {
            d = fd[e];
            cp = fcp[e];
        } else {
            const int32_t kk = __ldg(&a.flist[di.f_lo + e]);
            d = ldcg(&a.dk[kk - k0]);
            cp = __ldg(&a.col_ptr[__ldg(&a.order[kk])]);
        }
        if (d != 0.0) dx += d * (double)__ldg(&a.val[cp + i]);
    }
    return dx;
}

template <int NQ>
struct WinLayout {  // packed partial slots: Ls[0,NQ) L1[NQ,2NQ) Delta |T| [no-speculation count]
    static constexpr int W = 2 * NQ + 3 <= 8 ? 8 : (2 * NQ + 3 <= 16 ? 16 : 32);
    static constexpr int DELTA = 2 * NQ, NTOUCH = 2 * NQ + 1, NOSPEC = 2 * NQ + 2;
};

// the full columns' d'x part of sample i: from the dense pass (the block's rows are T when a
// full column has d != 0, so T[li] = row_base + li) or computed here for big blocks
__device__ __forceinline__ double dense_part(const StepArgs &a, const StepSmem &sm, const DenseInfo &di, int64_t k0,
                                            int64_t i, int64_t nT)
{
    if (nT <= TSM) {
        const int64_t li = i - sm.row_base;
        return sm.dxd[li];
    }
    return dense_dx(a, sm.fd, sm.fcp, di, k0, i);
}

// One Armijo window over candidates q0 .. q0+NQ-1 (Eq.6 with Eq.12 from retained quantities):
// per-sample loss changes over this CTA's touched samples (window 0 also folds d'x_i), the L1
// term and Delta over this CTA's bundle share, a fixed-order CTA partial, a barrier, then every
// CTA reduces the G partials in the same order and takes the same decision.
template <int NQ, class Sync>
__device__ __forceinline__ void window(const StepArgs &a, StepSmem &sm, Sync &sy, WinState &ws, const int32_t *Tl,
                                      int64_t nT, int64_t k0, int64_t pb0, int64_t pb1, int G, int c, int tid,
                                      int lane, int warp, const ShareReg &sh, RowReg &rr, const DenseInfo &di)
{
    using LY = WinLayout<NQ>;
    constexpr int W = LY::W;
    double alpha0 = 1.0;
    for (int q = 0; q < ws.q0; q++) alpha0 *= a.beta;
    double acc[W];
#pragma unroll
    for (int q = 0; q < W; q++) acc[q] = 0.0;
    if (ws.win == 0) {
        for (int64_t li = tid; li < nT; li += NT) {
            const int32_t i = Tl[li];
            const int ni = ldcg(&a.cnt[i]);
            const int64_t off = __ldg(&a.row_ptr[i]);
            const double zi = ldcg(&a.z[i]);
            const double cg = ldcg(&a.coef[i]).x;
            const int yi = a.y[i];
            if (li == tid) {
                rr.i = i;
                rr.yi = yi;
                rr.zi = zi;
                rr.has_dx = ni <= NREG;
            }
            if (ni <= NREG) {
                const double dx = (di.any ? dense_part(a, sm, di, k0, i, nT) : 0.0) + fold_small(a, off, ni);
                a.dxg[i] = dx;
                if (li == tid) rr.dx = dx;
                double al = alpha0;
#pragma unroll
                for (int q = 0; q < NQ; q++) {
                    acc[q] += loss_change(a.loss, zi, yi, cg, dx, al);
                    al *= a.beta;
                }
            } else {
                sm.has_heavy_rows = 1;
            }
        }
        __syncthreads();
        if (sm.has_heavy_rows && warp < NHW) {
            // samples with > NREG records: one warp each, fixed warp assignment
            for (int64_t lb = (int64_t)warp * 32; lb < nT; lb += 32 * NHW) {
                const int64_t li = lb + lane;
                int32_t i = -1;
                int ni = 0;
                if (li < nT) {
                    i = Tl[li];
                    ni = ldcg(&a.cnt[i]);
                }
                unsigned heavy = __ballot_sync(0xffffffffu, ni > NREG);
                while (heavy) {
                    const int src = __ffs(heavy) - 1;
                    heavy &= heavy - 1;
                    const int32_t ih = __shfl_sync(0xffffffffu, i, src);
                    const int nih = __shfl_sync(0xffffffffu, ni, src);
                    const double dxr = fold_warp(a, __ldg(&a.row_ptr[ih]), nih, sm.sk[warp], sm.sv[warp], lane);
                    if (lane == 0) {
                        const double dx = (di.any ? dense_part(a, sm, di, k0, ih, nT) : 0.0) + dxr;
                        a.dxg[ih] = dx;
                        const double zi = ldcg(&a.z[ih]);
                        const double cg = ldcg(&a.coef[ih]).x;
                        const int yi = a.y[ih];
                        double al = alpha0;
#pragma unroll
                        for (int q = 0; q < NQ; q++) {
                            acc[q] += loss_change(a.loss, zi, yi, cg, dx, al);
                            al *= a.beta;
                        }
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        for (int64_t li = tid; li < nT; li += NT) {
            const int32_t i = Tl[li];
            const double dx = ldcg(&a.dxg[i]);
            const double zi = ldcg(&a.z[i]);
            const double cg = ldcg(&a.coef[i]).x;
            const int yi = a.y[i];
            double al = alpha0;
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                acc[q] += loss_change(a.loss, zi, yi, cg, dx, al);
                al *= a.beta;
            }
        }
    }
    // L1 part of Eq.12 and Delta over this CTA's share of the bundle
    for (int64_t kk = pb0 + tid; kk < pb1; kk += NT) {
        const bool reg = kk == sh.kk;
        const double wj = reg ? sh.wj : ldcg(&a.w[__ldg(&a.order[kk])]);
        const double d = reg ? sh.d : ldcg(&a.dk[kk - k0]);
        double al = alpha0;
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            acc[NQ + q] += fabs(wj + al * d) - fabs(wj) + a.mu * al * d * (wj + 0.5 * al * d);
            al *= a.beta;
        }
        acc[LY::DELTA] += reg ? sh.delta : ldcg(&a.deltak[kk - k0]);
    }
    if (tid == 0) acc[LY::NTOUCH] = (double)nT;
    // CTA partial: transpose-reduce per warp, warps combined in order by warp 0
    constexpr int SPL = 32 / W;  // lanes per slot after xreduce
    {
        const double tot = xreduce<W>(acc, lane);
        if ((lane % SPL) == 0) sm.red[warp][lane / SPL] = tot;
    }
    double *part = a.part + (int64_t)(ws.win & 1) * G * NPART;
    __syncthreads();
    if (warp == 0 && lane < W) {
        double s = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < NW; w2++) s += sm.red[w2][lane];
        part[(int64_t)c * NPART + lane] = s;
    }
    sy.sync();
    // every CTA reduces the G partials in the same fixed order (all warps, then warp 0) and decides
    grid_totals<W>(part, G, sm.red, sm.tot, lane, warp);
    if (warp == 0) {
        if (lane == 0) {
            const double Dl = sm.tot[LY::DELTA];
            int qa = -1, badl = 0;
            double al = alpha0, la = 0.0, ra = 0.0, alpha_a = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                if (qa < 0 && !badl) {
                    const double lhs = sm.tot[NQ + q] + a.c * sm.tot[q];
                    const double rhs = a.sigma * al * Dl;
                    if (!isfinite(lhs) || !isfinite(Dl)) {
                        badl = 1;
                    } else if (lhs <= rhs) {
                        qa = ws.q0 + q;
                        alpha_a = al;
                        la = lhs;
                        ra = rhs;
                    }
                    al *= a.beta;
                }
            }
            sm.dec_q = qa;
            sm.dec_bad = badl;
            sm.dec_alpha = alpha_a;
            sm.dec_lhs = la;
            sm.dec_rhs = ra;
            sm.dec_Delta = Dl;
            sm.dec_nT = sm.tot[LY::NTOUCH];
        }
    }
    __syncthreads();
    ws.qacc = sm.dec_q;
    ws.bad = sm.dec_bad;
    ws.alpha = sm.dec_alpha;
    ws.lhs = sm.dec_lhs;
    ws.rhs = sm.dec_rhs;
    ws.Delta = sm.dec_Delta;
    ws.nT_tot = sm.dec_nT;
    ws.win++;
    __syncthreads();  // sm.dec_* / sm.red / sm.tot are reused by the next window
}

template <class Sync>
__global__ void __launch_bounds__(NT, Sync::kMinBlocks) k_step(StepArgs a)
{
    if (a.stop && ldcg(a.stop)) return;   // the solve already ended (queued ahead; grid-uniform)
    Sync sy(a.bar);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    StepSmem &sm = *reinterpret_cast<StepSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t nwords = (a.s + 31) >> 5;
    const int64_t wb = (int64_t)c * nwords / G, we = (int64_t)(c + 1) * nwords / G;
    const int64_t row_base = wb * 32;
    if (tid == 0) sm.row_base = row_base;
    int prev_q = 0;
    const int64_t pbs0 = (int64_t)c * a.P / G, pbs1 = (int64_t)(c + 1) * a.P / G;

    long long tprev = 0;
    const bool prof = PCDN_PROFILE && a.prof != nullptr && c == 0 && tid == 0;
    if (tid < 16) sm.pacc[tid] = 0;
#define PROF_MARK(i)                              \
    do {                                          \
        if (prof) {                               \
            const long long now_ = clock64();     \
            sm.pacc[i] += now_ - tprev;           \
            tprev = now_;                         \
        }                                         \
    } while (0)
    const int64_t gw = (int64_t)c * NW + warp;
    if (c == 0 && tid == 0) {
        sm.F = ldcg(a.F);
        for (int i = 0; i < 4; i++) sm.cnt[i] = 0;
    }
    if (warp == 1 && a.nsteps > 0) heavy_plan_warp(a, 0, min(a.P, a.ntot), c, G, lane, &sm.plan[0]);
    if (tid == 0) sm.nmid = 0;
    __syncthreads();
    for (int64_t t = 0; t < a.nsteps; t++) {
        if (prof) tprev = clock64();
        const int64_t k0 = t * a.P;
        const int64_t k1 = min(k0 + a.P, a.ntot);
        const int64_t Pt = k1 - k0;

        // ---------------- phase A: light columns (a1, a2, a3) --------------------------------
        // Positions in chunks of 32 per warp (one coalesced descriptor load): a short column
        // (<= SHORT nonzeros) is reduced by its lane alone, in row order (no shuffles; the
        // independent loads of all lanes' columns are in flight together); a medium one by the
        // whole warp.  Heavy columns (> heavy_len) are split below (A').
        // chunk width: 32 positions, fewer when the bundle would leave warps idle (small P)
        const int cw = (int)min((int64_t)32, max((int64_t)1, (Pt + (int64_t)G * NW - 1) / ((int64_t)G * NW)));
        for (int64_t ch = gw;; ch += (int64_t)G * NW) {
            const int64_t kb = k0 + ch * cw;
            if (kb >= k1) break;
            const int64_t kk = kb + lane;
            const int4 ci = (lane < cw && kk < k1) ? __ldg(&a.colinfo[kk]) : make_int4(0, -1, 0, 0);
            const int len = ci.y;
            // (a column longer than heavy_len belongs to the heavy path alone, however short)
            if (len >= 0 && len <= SHORT && len <= a.heavy_len) {
                const int32_t j = ci.x;
                const int64_t p0 = colinfo_p0(ci);
                int32_t ri[SHORT];
                float xv[SHORT];
#pragma unroll
                for (int e = 0; e < SHORT; e++) {
                    ri[e] = 0;
                    xv[e] = 0.f;
                    if (e < len) {
                        ri[e] = __ldg(&a.row_idx[p0 + e]);
                        xv[e] = __ldg(&a.val[p0 + e]);
                    }
                }
                const double wj = ldcg(&a.w[j]);
                double2 cf[SHORT];
#pragma unroll
                for (int e = 0; e < SHORT; e++) cf[e] = e < len ? ldcg(&a.coef[ri[e]]) : make_double2(0.0, 0.0);
                double g = 0.0, h = 0.0;
#pragma unroll
                for (int e = 0; e < SHORT; e++) {
                    if (e < len) {
                        const double x = (double)xv[e];
                        g += x * cf[e].x;
                        h += (x * x) * cf[e].y;
                    }
                }
                const Dir r = finish_feature(a, g, h, wj);
                a.dk[kk - k0] = r.d;
                a.deltak[kk - k0] = r.delta;
                if (a.g_out) {
                    a.g_out[kk - k0] = r.g;
                    a.h_out[kk - k0] = r.h;
                }
                if (a.d_out) a.d_out[kk - k0] = r.d;
                if (r.d != 0.0 && len != a.s) {   // full columns are folded from CSC (dense_dx)
                    double v[SHORT];
#pragma unroll
                    for (int e = 0; e < SHORT; e++) v[e] = r.d * (double)xv[e];
                    emit_batch<SHORT>(a, ri, v, len, (int32_t)(kk - k0));
                }
            }
            const int med_len = min(a.heavy_len, MED_LEN);
            unsigned med = __ballot_sync(0xffffffffu, len > SHORT && len <= med_len);
            // longer columns up to heavy_len: one CTA each, after the light loop (queued here)
            const unsigned mid = __ballot_sync(0xffffffffu, len > med_len && len <= a.heavy_len);
            if (mid) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&sm.nmid, __popc(mid));
                base = __shfl_sync(0xffffffffu, base, 0);
                const int slot = base + __popc(mid & ((1u << lane) - 1u));
                if (((mid >> lane) & 1u) && slot < MIDQ) sm.midq[slot] = (int32_t)kk;
                // beyond the queue (very large bundles on few CTAs): reduced by this warp below
                med |= __ballot_sync(0xffffffffu, ((mid >> lane) & 1u) && slot >= MIDQ);
            }
            while (med) {
                const int src = __ffs(med) - 1;
                med &= med - 1;
                const int32_t j = __shfl_sync(0xffffffffu, ci.x, src);
                const int ml = __shfl_sync(0xffffffffu, len, src);
                const int lo = __shfl_sync(0xffffffffu, ci.z, src), hi = __shfl_sync(0xffffffffu, ci.w, src);
                const int64_t p0 = (int64_t)(((uint64_t)(uint32_t)hi << 32) | (uint64_t)(uint32_t)lo);
                const int64_t p1 = p0 + ml;
                const int64_t km = kb + src;
                double gs, hs;
                col_gh(a, p0, p1, lane, gs, hs);
                const Dir r = finish_feature(a, gs, hs, ldcg(&a.w[j]));
                if (lane == 0) {
                    a.dk[km - k0] = r.d;
                    a.deltak[km - k0] = r.delta;
                    if (a.g_out) {
                        a.g_out[km - k0] = r.g;
                        a.h_out[km - k0] = r.h;
                    }
                    if (a.d_out) a.d_out[km - k0] = r.d;
                }
                if (r.d != 0.0 && ml != a.s) col_scatter(a, p0, p1, lane, (int32_t)(km - k0), r.d);
            }
        }

        // ---------------- CTA-level columns (med_len < length <= heavy_len) --------------------
        // each queued column is reduced by all warps of this CTA (nnz split evenly, warp partials
        // added in warp order: a fixed order), then scattered by the same split; no grid exchange
        __syncthreads();
        {
            const int nm = min(sm.nmid, MIDQ);
            for (int q = 0; q < nm; q++) {
                const int64_t km = sm.midq[q];
                const int4 ci = __ldg(&a.colinfo[km]);
                const int64_t p0 = colinfo_p0(ci);
                const int64_t ml = ci.y;
                const int64_t w0 = p0 + (int64_t)warp * ml / NW, w1 = p0 + (int64_t)(warp + 1) * ml / NW;
                double gs, hs;
                col_gh(a, w0, w1, lane, gs, hs, ml == a.s ? p0 : -1);
                if (lane == 0) {
                    sm.hg[0][warp] = gs;
                    sm.hh[0][warp] = hs;
                }
                __syncthreads();
                if (tid == 0) {
                    double g = 0.0, h = 0.0;
                    for (int w2 = 0; w2 < NW; w2++) {
                        g += sm.hg[0][w2];
                        h += sm.hh[0][w2];
                    }
                    const Dir r = finish_feature(a, g, h, ldcg(&a.w[ci.x]));
                    a.dk[km - k0] = r.d;
                    a.deltak[km - k0] = r.delta;
                    if (a.g_out) {
                        a.g_out[km - k0] = r.g;
                        a.h_out[km - k0] = r.h;
                    }
                    if (a.d_out) a.d_out[km - k0] = r.d;
                    sm.hd[0] = r.d;
                }
                __syncthreads();
                const double d = sm.hd[0];
                if (d != 0.0 && ml != a.s) col_scatter(a, w0, w1, lane, (int32_t)(km - k0), d);
                __syncthreads();   // hg / hd reused by the next column
            }
            if (tid == 0) sm.nmid = 0;   // ordered before the next step's queue by this step's barriers
        }
        PROF_MARK(8);
        // ---------------- phase A': heavy columns, nnz-balanced over all warps -----------
        // the plan (entry ranges from 32-ary warp searches) was computed a step ahead, inside the
        // previous step's final barrier
        const HeavyPlan hpl = sm.plan[t & 1];
        const int64_t e_lo = hpl.e_lo, e_hi = hpl.e_hi;
        if (e_hi > e_lo) {
            const int64_t hb0 = hpl.hb0;
            const int64_t NH = hpl.NH;
            const int64_t lo_c = (int64_t)c * NH / G, hi_c = (int64_t)(c + 1) * NH / G;
            if (tid == 0) sm.cross_e[0] = sm.cross_e[1] = -1;   // ordered by the rounds' barriers / sy
            PROF_MARK(9);
            const int64_t ce0 = hpl.ce0, ce1 = hpl.ce1;
            const int64_t a_w = lo_c + (int64_t)warp * (hi_c - lo_c) / NW;
            const int64_t b_w = lo_c + (int64_t)(warp + 1) * (hi_c - lo_c) / NW;
            for (int64_t rb = ce0; rb < ce1; rb += NE_MAX) {
                const int ne = (int)min((int64_t)NE_MAX, ce1 - rb);
                for (int i = tid; i <= ne; i += NT) sm.hst[i] = __ldg(&a.hstart[rb + i]) - hb0;
                for (int i = tid; i < ne * NW; i += NT) {
                    sm.hg[i / NW][i % NW] = 0.0;
                    sm.hh[i / NW][i % NW] = 0.0;
                }
                __syncthreads();
                for (int le = 0; le < ne; le++) {
                    const int64_t st = sm.hst[le], en = sm.hst[le + 1];
                    if (en <= a_w) continue;
                    if (st >= b_w) break;
                    const int64_t s0 = max(a_w, st), s1 = min(b_w, en);
                    const int32_t kk = __ldg(&a.hlist[rb + le]);
                    const int32_t j = __ldg(&a.order[kk]);
                    const int64_t cs = __ldg(&a.col_ptr[j]);
                    double gs, hs;
                    col_gh(a, cs + (s0 - st), cs + (s1 - st), lane, gs, hs, en - st == a.s ? cs : -1);
                    if (lane == 0) {
                        sm.hg[le][warp] = gs;
                        sm.hh[le][warp] = hs;
                    }
                }
                __syncthreads();
                for (int le = tid; le < ne; le += NT) {
                    double gs = 0.0, hs = 0.0;
                    for (int w2 = 0; w2 < NW; w2++) {
                        gs += sm.hg[le][w2];
                        hs += sm.hh[le][w2];
                    }
                    const int64_t st = sm.hst[le], en = sm.hst[le + 1];
                    const int64_t e = rb + le;
                    if (st >= lo_c && en <= hi_c) {  // column interior to this CTA: finish now
                        const int32_t kk = __ldg(&a.hlist[e]);
                        const int32_t j = __ldg(&a.order[kk]);
                        const Dir r = finish_feature(a, gs, hs, ldcg(&a.w[j]));
                        sm.hd[le] = r.d;
                        a.dk[kk - k0] = r.d;
                        a.deltak[kk - k0] = r.delta;
                        if (a.g_out) {
                            a.g_out[kk - k0] = r.g;
                            a.h_out[kk - k0] = r.h;
                        }
                        if (a.d_out) a.d_out[kk - k0] = r.d;
                    } else {  // crossing: CTA partial, finished after the grid barrier
                        const int slot = st < lo_c ? 0 : 1;
                        HPart hp;
                        hp.e = e;
                        hp.g = gs;
                        hp.h = hs;
                        hp.pad = 0.0;
                        a.hpart[(int64_t)c * 2 + slot] = hp;
                        sm.cross_e[slot] = e;
                        sm.hd[le] = 0.0;  // not scattered in this round
                    }
                }
                __syncthreads();
                // scatter interior columns of this round
                for (int le = 0; le < ne; le++) {
                    const int64_t st = sm.hst[le], en = sm.hst[le + 1];
                    if (en <= a_w) continue;
                    if (st >= b_w) break;
                    if (!(st >= lo_c && en <= hi_c)) continue;
                    const double d = sm.hd[le];
                    if (d == 0.0 || en - st == a.s) continue;   // full columns: dense_dx
                    const int64_t s0 = max(a_w, st), s1 = min(b_w, en);
                    const int32_t kk = __ldg(&a.hlist[rb + le]);
                    const int32_t j = __ldg(&a.order[kk]);
                    const int64_t cs = __ldg(&a.col_ptr[j]);
                    col_scatter(a, cs + (s0 - st), cs + (s1 - st), lane, kk - (int32_t)k0, d);
                }
                __syncthreads();
            }
            PROF_MARK(10);
            sy.sync();
            PROF_MARK(11);
            // finish the (at most two) columns crossing this CTA's boundaries
            if (warp < 2) {   // one warp per crossing column, lanes over the CTA partials
                const int64_t e = sm.cross_e[warp];
                if (lane == 0) sm.cross_d[warp] = 0.0;
                if (e >= 0) {
                    const int64_t st = __ldg(&a.hstart[e]) - hb0, en = __ldg(&a.hstart[e + 1]) - hb0;
                    const int clo = cta_of(st, NH, G), chi = cta_of(en - 1, NH, G);
                    double gs = 0.0, hs = 0.0;
                    for (int c2 = clo + lane; c2 <= chi; c2 += 32) {
                        if ((int64_t)c2 * NH / G == (int64_t)(c2 + 1) * NH / G) continue;  // empty range
                        const HPart hp = ld_hpart(&a.hpart[(int64_t)c2 * 2 + (c2 == clo ? 1 : 0)]);
                        if (hp.e != e) atomicMax(a.status, 4);  // internal consistency check
                        gs += hp.g;
                        hs += hp.h;
                    }
                    gs = warp_sum(gs);
                    hs = warp_sum(hs);
                    if (lane == 0) {
                        const int32_t kk = __ldg(&a.hlist[e]);
                        const int32_t j = __ldg(&a.order[kk]);
                        const Dir r = finish_feature(a, gs, hs, ldcg(&a.w[j]));
                        sm.cross_d[warp] = r.d;
                        if (c == clo) {
                            a.dk[kk - k0] = r.d;
                            a.deltak[kk - k0] = r.delta;
                            if (a.g_out) {
                                a.g_out[kk - k0] = r.g;
                                a.h_out[kk - k0] = r.h;
                            }
                            if (a.d_out) a.d_out[kk - k0] = r.d;
                        }
                    }
                }
            }
            __syncthreads();
            for (int sl = 0; sl < 2; sl++) {
                const int64_t e = sm.cross_e[sl];
                if (e < 0 || (sl == 1 && e == sm.cross_e[0])) continue;
                const double d = sm.cross_d[sl];
                if (d == 0.0) continue;
                const int64_t st = __ldg(&a.hstart[e]) - hb0, en = __ldg(&a.hstart[e + 1]) - hb0;
                if (en <= a_w || st >= b_w || en - st == a.s) continue;
                const int64_t s0 = max(a_w, st), s1 = min(b_w, en);
                const int32_t kk = __ldg(&a.hlist[e]);
                const int32_t j = __ldg(&a.order[kk]);
                const int64_t cs = __ldg(&a.col_ptr[j]);
                col_scatter(a, cs + (s0 - st), cs + (s1 - st), lane, kk - (int32_t)k0, d);
            }
        }
        PROF_MARK(0);
        sy.sync();
        PROF_MARK(1);
        const bool full = Pt == a.P;
        const int64_t pb0 = k0 + (full ? pbs0 : (int64_t)c * Pt / G);
        const int64_t pb1 = k0 + (full ? pbs1 : (int64_t)(c + 1) * Pt / G);
        ShareReg sh;
        sh.kk = -1;
        if (pb0 + tid < pb1) {  // loads issued here, consumed by the line search
            sh.kk = pb0 + tid;
            sh.j = __ldg(&a.order[sh.kk]);
            sh.wj = ldcg(&a.w[sh.j]);
            sh.d = ldcg(&a.dk[sh.kk - k0]);
            sh.delta = ldcg(&a.deltak[sh.kk - k0]);
        }
        RowReg rr;
        rr.i = -1;

        // ---------------- the step's full columns (dense_dx) -----------------------------
        DenseInfo di;
        di.f_lo = hpl.f_lo;
        di.nf = hpl.nf;
        di.any = false;
        if (di.nf > 0) {
            int any = 0;
            for (int64_t e = tid; e < di.nf; e += NT) {
                const int32_t kk = __ldg(&a.flist[di.f_lo + e]);
                const double d = ldcg(&a.dk[kk - k0]);
                if (e < FMAX) {
                    sm.fd[e] = d;
                    sm.fcp[e] = __ldg(&a.col_ptr[__ldg(&a.order[kk])]);
                }
                any |= d != 0.0;
            }
            di.any = __syncthreads_or(any) != 0;
        }

        // ---------------- phase C1: touched set of this CTA's row block ------------------
        // each thread owns a contiguous run of bitmap words; a ballot-based warp scan plus
        // warp totals gives every touched sample its slot in T (ascending sample order).  A full
        // column with d_j != 0 touches every sample (reading Z8): T = the whole block.
        if (di.any) {
            const int64_t nrows = min(a.s, we * 32) - row_base;
            int32_t *Tw = nrows <= TSM ? sm.tl : a.tlist + row_base;
            for (int64_t li = tid; li < nrows; li += NT) Tw[li] = (int32_t)(row_base + li);
            if (tid == 0) {
                sm.nT = nrows > 0 ? nrows : 0;
                sm.has_heavy_rows = 0;
            }
            __syncthreads();
        } else {
            const int64_t nwc = we - wb;
            const int64_t wpt = (nwc + NT - 1) / NT;
            const int64_t w0 = wb + (int64_t)tid * wpt, w1 = min(we, w0 + wpt);
            uint32_t wv[WREG];
            unsigned cntb = 0;
#pragma unroll
            for (int r = 0; r < WREG; r++) {
                wv[r] = (w0 + r < w1) ? ldcg(&a.bits[w0 + r]) : 0u;
                cntb += __popc(wv[r]);
            }
            for (int64_t wi = w0 + WREG; wi < w1; wi++) cntb += __popc(ldcg(&a.bits[wi]));
            unsigned incl = 0;
            const unsigned lemask = 0xffffffffu >> (31 - lane);
#pragma unroll
            for (int b = 0; b < 16; b++) {
                const unsigned m = __ballot_sync(0xffffffffu, (cntb >> b) & 1u);
                if (!m && (b >= 8)) break;
                incl += (unsigned)__popc(m & lemask) << b;
            }
            const unsigned wtot = __reduce_add_sync(0xffffffffu, cntb);
            if (lane == 0) sm.scan_w[warp] = wtot;
            __syncthreads();
            const unsigned sw = lane < NW ? (unsigned)sm.scan_w[lane] : 0u;
            const unsigned woff = __reduce_add_sync(0xffffffffu, lane < warp ? sw : 0u);
            const unsigned total = __reduce_add_sync(0xffffffffu, sw);
            int32_t *Tw = total <= (unsigned)TSM ? sm.tl : a.tlist + row_base;
            if (cntb) {
                int64_t pos = (int64_t)woff + incl - cntb;
#pragma unroll
                for (int r = 0; r < WREG; r++) {
                    uint32_t m = wv[r];
                    while (m) {
                        const int b = __ffs(m) - 1;
                        m &= m - 1;
                        Tw[pos++] = (int32_t)((w0 + r) * 32 + b);
                    }
                }
                for (int64_t wi = w0 + WREG; wi < w1; wi++) {
                    uint32_t m = ldcg(&a.bits[wi]);
                    while (m) {
                        const int b = __ffs(m) - 1;
                        m &= m - 1;
                        Tw[pos++] = (int32_t)(wi * 32 + b);
                    }
                }
            }
            if (tid == 0) {
                sm.nT = total;
                sm.has_heavy_rows = 0;
            }
            __syncthreads();
        }
        const int64_t nT = sm.nT;
        const int32_t *Tl = nT <= TSM ? sm.tl : a.tlist + row_base;
        if (di.any && nT <= TSM) {
            // dense pass: the full columns' d'x part of every row of the block, split over all
            // threads as (row, column chunk) so the loads of a column are coalesced over rows;
            // chunk partials are added in chunk order (a fixed order)
            const int R = (int)nT;
            const int C = R >= NT ? 1 : (int)min((int64_t)(NT / max(R, 1)), di.nf);
            double *dpart = &sm.red[0][0];   // NW*32 = NT doubles
            for (int r0 = 0; r0 < R; r0 += NT) {
                const int t = tid;
                if (C == 1) {
                    if (r0 + t < R) sm.dxd[r0 + t] = dense_dx(a, sm.fd, sm.fcp, di, k0, row_base + r0 + t);
                } else if (t < R * C) {
                    const int r = t % R, ch = t / R;
                    const int64_t e0 = (int64_t)ch * di.nf / C, e1 = (int64_t)(ch + 1) * di.nf / C;
                    const int64_t i = row_base + r;
                    double part = 0.0;
#pragma unroll 16
                    for (int64_t e = e0; e < e1; e++) {
                        double d;
                        int64_t cp;
                        if (e < FMAX) {
                            d = sm.fd[e];
                            cp = sm.fcp[e];
                        } else {
                            const int32_t kk = __ldg(&a.flist[di.f_lo + e]);
                            d = ldcg(&a.dk[kk - k0]);
                            cp = __ldg(&a.col_ptr[__ldg(&a.order[kk])]);
                        }
                        if (d != 0.0) part += d * (double)__ldg(&a.val[cp + i]);
                    }
                    dpart[t] = part;
                }
            }
            if (C > 1) {
                __syncthreads();
                for (int r = tid; r < R; r += NT) {
                    double x = 0.0;
                    for (int ch = 0; ch < C; ch++) x += dpart[ch * R + r];
                    sm.dxd[r] = x;
                }
            }
            __syncthreads();
        }
        PROF_MARK(2);

        // ---------------- phase C2+C3: fold d'x_i (a3) and the Armijo windows (a4) ----------
        WinState ws;
        ws.q0 = 0;
        ws.nq = prev_q <= 1 ? 2 : QW;
        ws.qacc = -1;
        ws.bad = 0;
        ws.win = 0;
        while (true) {
            if (ws.nq <= 2) window<2>(a, sm, sy, ws, Tl, nT, k0, pb0, pb1, G, c, tid, lane, warp, sh, rr, di);
            else window<QW>(a, sm, sy, ws, Tl, nT, k0, pb0, pb1, G, c, tid, lane, warp, sh, rr, di);
            PROF_MARK(5);
            if (ws.qacc >= 0 || ws.bad) break;
            ws.q0 += ws.nq;
            if (ws.q0 > a.qmax) break;
            ws.nq = QW;
        }
        int qacc = ws.qacc;
        const bool bad = ws.bad != 0;
        if (qacc > a.qmax) qacc = -1;   // window overshoot past q_max counts as exhausted
        const double alpha_acc = qacc < 0 ? 0.0 : ws.alpha;   // null step (Z10)
        prev_q = qacc < 0 ? QW : qacc;

        // ---------------- commit (a5): this CTA's samples and bundle share; clear marks -----
        // CB samples of a thread per round: all their loads in flight together (large steps touch
        // ~10^4 samples per row block); the per-sample arithmetic is unchanged
        constexpr int CB = 4;
        if (nT <= NT) {   // small steps: at most one sample per thread
            if (tid < nT) {
                const bool reg = rr.has_dx;
                const int32_t i = rr.i;
                const double dx = reg ? rr.dx : ldcg(&a.dxg[i]);
                if (qacc >= 0) {
                    const double zn = rr.zi + alpha_acc * dx;
                    a.z[i] = zn;
                    const double2 cfo = a.loss == LOSS_SQ ? ldcg(&a.coef[i]) : make_double2(0.0, 0.0);
                    a.coef[i] = coef_next(a.loss, cfo, zn, alpha_acc * dx, rr.yi);
                }
                a.cnt[i] = 0;
                if (a.debug) {
                    a.dbg_dx[i] = dx;
                    a.dbg_mark[i] = 1;
                }
            }
        } else
        for (int64_t lb = tid; lb < nT; lb += (int64_t)NT * CB) {
            int32_t ii[CB];
            double dxv[CB], zv[CB];
            int yv[CB];
#pragma unroll
            for (int e = 0; e < CB; e++) {
                const int64_t li = lb + (int64_t)e * NT;
                ii[e] = li < nT ? (li == tid ? rr.i : Tl[li]) : -1;
            }
#pragma unroll
            for (int e = 0; e < CB; e++) {
                const int64_t li = lb + (int64_t)e * NT;
                dxv[e] = 0.0;
                zv[e] = 0.0;
                yv[e] = 1;
                if (ii[e] >= 0) {
                    // the heavy-row fold may have produced dx for the register row: take dxg then
                    const bool reg = li == tid && rr.has_dx;
                    dxv[e] = reg ? rr.dx : ldcg(&a.dxg[ii[e]]);
                    if (qacc >= 0) {
                        zv[e] = li == tid ? rr.zi : ldcg(&a.z[ii[e]]);
                        yv[e] = li == tid ? rr.yi : (int)a.y[ii[e]];
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < CB; e++) {
                const int32_t i = ii[e];
                if (i < 0) continue;
                if (qacc >= 0) {
                    const double zn = zv[e] + alpha_acc * dxv[e];
                    a.z[i] = zn;
                    const double2 cfo = a.loss == LOSS_SQ ? ldcg(&a.coef[i]) : make_double2(0.0, 0.0);
                    a.coef[i] = coef_next(a.loss, cfo, zn, alpha_acc * dxv[e], yv[e]);
                }
                a.cnt[i] = 0;
                if (a.debug) {
                    a.dbg_dx[i] = dxv[e];
                    a.dbg_mark[i] = 1;
                }
            }
        }
        for (int64_t wi = wb + tid; wi < we; wi += NT) a.bits[wi] = 0u;
        if (qacc >= 0) {
            for (int64_t kb = pb0 + tid; kb < pb1; kb += (int64_t)NT * CB) {
                int32_t jj[CB];
                double wv[CB], dv[CB];
#pragma unroll
                for (int e = 0; e < CB; e++) {
                    const int64_t kk = kb + (int64_t)e * NT;
                    jj[e] = kk < pb1 ? (kk == sh.kk ? sh.j : __ldg(&a.order[kk])) : -1;
                }
#pragma unroll
                for (int e = 0; e < CB; e++) {
                    const int64_t kk = kb + (int64_t)e * NT;
                    wv[e] = 0.0;
                    dv[e] = 0.0;
                    if (jj[e] >= 0) {
                        wv[e] = kk == sh.kk ? sh.wj : ldcg(&a.w[jj[e]]);
                        dv[e] = kk == sh.kk ? sh.d : ldcg(&a.dk[kk - k0]);
                    }
                }
#pragma unroll
                for (int e = 0; e < CB; e++)
                    if (jj[e] >= 0) a.w[jj[e]] = wv[e] + alpha_acc * dv[e];
            }
        }
        PROF_MARK(6);
        if (c == 0 && tid == 0) {
            double F = sm.F;
            if (qacc >= 0) F = F + ws.lhs;
            sm.F = F;
            *a.F = F;
            if (bad) atomicMax(a.status, 3);
            a.info[0] = (double)qacc;
            a.info[1] = alpha_acc;
            a.info[2] = ws.Delta;
            a.info[3] = ws.lhs;
            a.info[4] = ws.rhs;
            a.info[5] = F;
            a.info[7] = ws.nT_tot;
            const int64_t gstep = a.trace_off + t;
            if (gstep < a.trace_cap) {
                if (a.q_trace) a.q_trace[gstep] = qacc;
                if (a.F_trace) a.F_trace[gstep] = F;
            }
            sm.cnt[0] += 1;
            sm.cnt[1] += qacc < 0 ? 1 : 0;
            sm.cnt[2] += (int64_t)ws.nT_tot;
            sm.cnt[3] += Pt;
        }
        sy.arrive();
        // the next step's heavy plan, while the barrier completes
        if (warp == NW - 1 && k1 < a.ntot) heavy_plan_warp(a, k1, min(k1 + a.P, a.ntot), c, G, lane, &sm.plan[(t + 1) & 1]);
        sy.wait();
        PROF_MARK(7);
        if (bad) break;
    }
    if (c == 0 && tid == 0) {
        a.counters[0] += sm.cnt[0];
        a.counters[1] += sm.cnt[1];
        a.counters[3] += sm.cnt[2];
        a.counters[4] += sm.cnt[3];
    }
    if (prof)
        for (int i = 0; i < 16; i++) a.prof[i] += sm.pacc[i];
#undef PROF_MARK
}

// ------------------------------------------------------------------------------------
// a6 and state (re)initialisation
// ------------------------------------------------------------------------------------
// z_i = sum_j w_j x_ij over row i in ascending column order, then the cached factors.
__global__ void k_set_z(int64_t s, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                        const float *__restrict__ csr_val, const int8_t *__restrict__ y, const double *__restrict__ w,
                        int loss, double *z, double2 *coef, int zero, const double *__restrict__ t)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
        double zi = 0.0;
        if (!zero)
            for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; p++) zi += w[col_idx[p]] * (double)csr_val[p];
        z[i] = zi;
        coef[i] = loss == LOSS_SQ ? make_double2(2.0 * (zi - t[i]), 2.0) : coef_of(loss, zi, y[i]);
    }
}

// F = c sum_i phi(y_i z_i) + sum_j |w_j|, fixed two-level order: tile b of each array
constexpr int OBJ_NB = 256;
__device__ __forceinline__ void obj_block_partial(int64_t s, int64_t n, const double *__restrict__ z,
                                                  const int8_t *__restrict__ y, const double *__restrict__ w, int loss,
                                                  double *partial, const double *__restrict__ t)
{
    const int b = blockIdx.x;
    const int64_t zs0 = (int64_t)b * s / OBJ_NB, zs1 = (int64_t)(b + 1) * s / OBJ_NB;
    const int64_t ws0 = (int64_t)b * n / OBJ_NB, ws1 = (int64_t)(b + 1) * n / OBJ_NB;
    double ls = 0.0, l1 = 0.0, l2 = 0.0;
    for (int64_t i = zs0 + threadIdx.x; i < zs1; i += blockDim.x) {
        if (loss == LOSS_SQ) {
            const double r = t[i] - z[i];
            ls += r * r;
        } else {
            ls += phi_of(loss, (double)y[i] * z[i]);
        }
    }
    for (int64_t j = ws0 + threadIdx.x; j < ws1; j += blockDim.x) {
        l1 += fabs(w[j]);
        l2 += w[j] * w[j];
    }
    ls = warp_sum(ls);
    l1 = warp_sum(l1);
    l2 = warp_sum(l2);
    __shared__ double sh[3][32];
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = ls;
        sh[1][threadIdx.x >> 5] = l1;
        sh[2][threadIdx.x >> 5] = l2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (int w2 = 0; w2 < (int)(blockDim.x >> 5); w2++) {
            a0 += sh[0][w2];
            a1 += sh[1][w2];
            a2 += sh[2][w2];
        }
        partial[3 * b] = a0;
        partial[3 * b + 1] = a1;
        partial[3 * b + 2] = a2;
    }
}

// obj_block_partial's arithmetic for block b by a group of OBJ_NB consecutive threads (gt = thread
// in the group, gw = warp in the group, wsum = the group's OBJ_NB/32 x 3 scratch): the same per-thread
// strides, warp sums and warp order, so the partials equal k_obj's bit for bit
__device__ __forceinline__ void obj_group_partial(int b, int gt, int gw, int64_t s, int64_t n,
                                                  const double *__restrict__ z, const int8_t *__restrict__ y,
                                                  const double *__restrict__ w, int loss, const double *__restrict__ t,
                                                  double (*wsum)[3], double *partial, bool write)
{
    // (write == false: a group without a block this round; it only joins the barriers)
    const int64_t zs0 = write ? (int64_t)b * s / OBJ_NB : 0, zs1 = write ? (int64_t)(b + 1) * s / OBJ_NB : 0;
    const int64_t ws0 = write ? (int64_t)b * n / OBJ_NB : 0, ws1 = write ? (int64_t)(b + 1) * n / OBJ_NB : 0;
    double ls = 0.0, l1 = 0.0, l2 = 0.0;
    for (int64_t i = zs0 + gt; i < zs1; i += OBJ_NB) {
        if (loss == LOSS_SQ) {
            const double r = t[i] - __ldcg(&z[i]);
            ls += r * r;
        } else {
            ls += phi_of(loss, (double)y[i] * __ldcg(&z[i]));
        }
    }
    for (int64_t j = ws0 + gt; j < ws1; j += OBJ_NB) {
        const double wj = __ldcg(&w[j]);
        l1 += fabs(wj);
        l2 += wj * wj;
    }
    ls = warp_sum(ls);
    l1 = warp_sum(l1);
    l2 = warp_sum(l2);
    if ((gt & 31) == 0) {
        wsum[gw][0] = ls;
        wsum[gw][1] = l1;
        wsum[gw][2] = l2;
    }
    __syncthreads();
    if (gt == 0 && write) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (int w2 = 0; w2 < OBJ_NB / 32; w2++) {
            a0 += wsum[w2][0];
            a1 += wsum[w2][1];
            a2 += wsum[w2][2];
        }
        partial[3 * b] = a0;
        partial[3 * b + 1] = a1;
        partial[3 * b + 2] = a2;
    }
    __syncthreads();
}

__global__ void k_obj_partial(int64_t s, int64_t n, const double *__restrict__ z, const int8_t *__restrict__ y,
                              const double *__restrict__ w, int loss, double *partial, const double *__restrict__ t)
{
    obj_block_partial(s, n, z, y, w, loss, partial, t);
}

// F = c sum phi + ||w||_1 + (mu/2)||w||^2 (Eq.1 + the elastic-net term of Z25)
// stop (nullable): the solve's device-side stop test at this outer boundary -- the Eq.14 gap
// (F - F*)/F* <= eps (eps > 0), a non-finite F, or a raised status -- so that step launches the
// host queued ahead exit at once (the host takes the same decision from the read-back F)
__device__ __forceinline__ void obj_final_body(const double *partial, double c, double mu, double *F,
                                               double *F_copy, double eps, double fstar, const int *status, int *stop)
{
    __shared__ double sh[3][OBJ_NB];
    const int t = threadIdx.x;
    sh[0][t] = __ldcg(&partial[3 * t]);
    sh[1][t] = __ldcg(&partial[3 * t + 1]);
    sh[2][t] = __ldcg(&partial[3 * t + 2]);
    __syncthreads();
    for (int o = OBJ_NB / 2; o > 0; o >>= 1) {
        if (t < o) {
            sh[0][t] += sh[0][t + o];
            sh[1][t] += sh[1][t + o];
            sh[2][t] += sh[2][t + o];
        }
        __syncthreads();
    }
    if (t == 0) {
        const double Fv = c * sh[0][0] + sh[1][0] + 0.5 * mu * sh[2][0];
        *F = Fv;
        if (F_copy) *F_copy = Fv;
        if (stop && (!isfinite(Fv) || ldcg(status) != 0 || (eps > 0 && (Fv - fstar) / fstar <= eps))) *stop = 1;
    }
}

__global__ void k_obj_final(const double *__restrict__ partial, double c, double mu, double *F, double *F_copy,
                            double eps, double fstar, const int *status, int *stop)
{
    obj_final_body(partial, c, mu, F, F_copy, eps, fstar, status, stop);
}

// The solve's starting state of the read-back block (status, err_what, stop and ticket are
// consecutive ints; err_idx starts at the largest value for atomicMin) and the grid barrier
__global__ void k_solve_init(int *status4, long long *err_idx, int64_t *counters, unsigned long long *bar)
{
    const int t = threadIdx.x;
    if (t < 4) status4[t] = 0;
    if (t < 8) counters[t] = 0;
    if (t == 0) {
        *err_idx = 0x7f7f7f7f7f7f7f7fLL;
        *bar = 0ull;
    }
}

// The solve's outer boundary in one launch (OBJ_NB blocks of OBJ_NB threads): the block partials,
// then the last block to finish (ticket) sums them in the fixed order of k_obj_final, takes the
// stop test, re-arms the step kernels' grid barrier and the ticket, and copies the read-back block
// (F, status, counters, ...) straight into mapped pinned host memory -- no copy-engine work between
// two step launches.
struct ObjBoundary {
    double c, mu, eps, fstar;
    double *F;
    double *F_copy;                     // nullable
    const int *status;
    int *stop;
    unsigned *ticket;
    unsigned long long *bar;
    const unsigned long long *mirror;   // device block (8-byte words)
    unsigned long long *mirror_host;    // mapped pinned host block (nullable: no copy)
    int mirror_words;
    // optional: the next outer iteration's partition (k_perm's output) when nothing else of the
    // list build is needed (the dense kernel)
    int perm;
    uint64_t seed;
    int64_t k_next, n, s;
    const int64_t *col_ptr;
    int heavy_len;
    int32_t *order, *flag, *fflag;
    int4 *colinfo;
};
__global__ void __launch_bounds__(OBJ_NB) k_obj(int64_t s, int64_t n, const double *__restrict__ z,
                                                const int8_t *__restrict__ y, const double *__restrict__ w, int loss,
                                                double *partial, const double *__restrict__ t, ObjBoundary o)
{
    if (o.stop && ldcg(o.stop)) return;   // queued after the outer iteration that ended the solve (grid-uniform)
    if (o.perm) perm_positions(o.seed, o.k_next, o.n, o.s, o.col_ptr, o.heavy_len, o.order, o.flag, o.fflag, o.colinfo);
    obj_block_partial(s, n, z, y, w, loss, partial, t);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(o.ticket, 1u) == (unsigned)(OBJ_NB - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    obj_final_body(partial, o.c, o.mu, o.F, o.F_copy, o.eps, o.fstar, o.status, o.stop);
    __syncthreads();
    if (threadIdx.x == 0) {
        *o.ticket = 0u;
        *o.bar = 0ull;
    }
    if (o.mirror_host) {
        __threadfence();
        __syncthreads();
        for (int e = threadIdx.x; e < o.mirror_words; e += blockDim.x) o.mirror_host[e] = __ldcg(&o.mirror[e]);
        __threadfence_system();
    }
}

// status 1 + first index of a non-finite value (squared-loss targets)
__global__ void k_check_finite(const double *__restrict__ t, int64_t s, int *status, long long *err_idx)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(t[i])) {
            atomicMax(status, 1);
            atomicMin(err_idx, (long long)i);
        }
}

// is p the first offset of a segment of ptr[0..m] (ptr nondecreasing)?  (binary search)
__device__ __forceinline__ bool seg_start(const int64_t *__restrict__ ptr, int64_t m, int64_t p)
{
    int64_t lo = 0, hi = m;   // first k with ptr[k] >= p
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ptr[mid] < p) lo = mid + 1; else hi = mid;
    }
    return lo <= m && ptr[lo] == p;
}

// Input validation: code 1 + first offending index.  The pointer arrays a thread
// per entry; the nonzeros flat over the whole array (coalesced): an index not above its
// predecessor is an error unless it starts a segment (binary search in the pointer array) -- a
// thread or warp per column had left config 5's 1.96M-nonzero column to one of them (0.36 s).
__global__ void k_validate(int64_t s, int64_t n, int64_t nnz, const int64_t *__restrict__ col_ptr,
                           const int32_t *__restrict__ row_idx, const float *__restrict__ val,
                           const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                           const float *__restrict__ csr_val, const int8_t *__restrict__ y,
                           int *status, long long *err_idx, int *err_what)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    auto fail = [&](int what, int64_t idx) {
        atomicMax(status, 1);
        if (atomicMin(err_idx, (long long)idx) > (long long)idx) atomicExch(err_what, what);
    };
    bool cbad = false, rbad = false;   // this thread saw a broken pointer array (flat checks then stop)
    for (int64_t j = t0; j < n; j += stride) {
        const int64_t a0 = col_ptr[j], a1 = col_ptr[j + 1];
        if (j == 0 && a0 != 0) fail(1, 0);
        if (j == n - 1 && a1 != nnz) fail(2, j);
        if (a1 < a0 || a0 < 0 || a1 > nnz) {
            fail(3, j);
            cbad = true;
        }
    }
    for (int64_t i = t0; row_ptr && i < s; i += stride) {   // (row_ptr == NULL: the CSC alone)
        const int64_t a0 = row_ptr[i], a1 = row_ptr[i + 1];
        if (i == 0 && a0 != 0) fail(7, 0);
        if (i == s - 1 && a1 != nnz) fail(8, i);
        if (a1 < a0 || a0 < 0 || a1 > nnz) {
            fail(9, i);
            rbad = true;
        }
        if (y && y[i] != 1 && y[i] != -1) fail(13, i);   // labels unused by the squared loss
    }
    if (cbad || rbad) return;
    for (int64_t p = t0; p < nnz; p += stride) {
        const int32_t r = row_idx[p];
        if (r < 0 || r >= s) fail(4, p);
        if (p > 0 && r <= row_idx[p - 1] && !seg_start(col_ptr, n, p)) fail(5, p);
        if (!isfinite(val[p])) fail(6, p);
        if (row_ptr) {
            const int32_t cidx = col_idx[p];
            if (cidx < 0 || cidx >= n) fail(10, p);
            if (p > 0 && cidx <= col_idx[p - 1] && !seg_start(row_ptr, s, p)) fail(11, p);
            if (!isfinite(csr_val[p])) fail(12, p);
        }
    }
}

// CSR/CSC consistency: every CSR nonzero (i, j, v) must be found in column j by binary search
// (check == 0: a CSR the library built from this CSC itself -- found, values not compared).  The
// search also gives the sparse kernel's map cslot[CSC offset] = CSR offset of the same nonzero.
// Runs after k_validate on the same stream: if that refused the arrays (indices may point anywhere)
// this kernel does nothing.
__global__ void k_validate_transpose(int64_t s, const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ row_idx,
                                     const float *__restrict__ val, const int64_t *__restrict__ row_ptr,
                                     const int32_t *__restrict__ col_idx, const float *__restrict__ csr_val,
                                     int check, uint32_t *cslot, int *status, long long *err_idx, int *err_what)
{
    if (ldcg(status)) return;
    // one warp per row, lanes over its nonzeros: the binary searches of a row run side by side
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = gw; i < s; i += nw) {
        for (int64_t p = row_ptr[i] + lane; p < row_ptr[i + 1]; p += 32) {
            const int32_t j = col_idx[p];
            int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (row_idx[mid] < i) lo = mid + 1; else hi = mid;
            }
            if (lo >= col_ptr[j + 1] || row_idx[lo] != i || (check && val[lo] != csr_val[p])) {
                atomicMax(status, 1);
                if (atomicMin(err_idx, (long long)p) > (long long)p) atomicExch(err_what, 14);
            } else {
                cslot[lo] = (uint32_t)p;
            }
        }
    }
}

// per-column nnz total of the CSC must equal the CSR count (cheap necessary condition)
__global__ void k_debug_touched_clear(uint8_t *mark, int64_t s)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) mark[i] = 0;
}

}  // namespace pcdn
