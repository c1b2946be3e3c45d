// pcdn_resident.cuh -- the cluster-resident bundle-step kernel.
//
// Small bundle steps (the configured P of configs 1-3) are bound by the latency of the
// exchanges between phases, not by HBM.  This variant keeps ALL per-sample state
// in the distributed shared memory of one thread-block cluster for the whole launch (one launch =
// all b bundle steps of an outer iteration), and synchronises the steps with point-to-point
// DSMEM messages instead of cluster barriers: every `barrier.cluster.arrive.release` costs a
// GPU-scope memory drain (MEMBAR.ALL.GPU + ERRBAR in SASS), while `st.async` stores that
// complete a transaction count on the receiver's mbarrier need no fence at all.
//
//   CTA c of the G-CTA cluster (G = 2^lg <= 16) owns samples i = li*G + c:
//     zd[li] = (z_i, dx_i): retained w'x_i and the d'x_i of the LAST step (0 if
//     the sample was not touched), coef[li] = (G_i, H_i) (Eq.13 / App. A.2 factors), y[li].
//
//   phase A   warp per light column (split over all warps for heavy columns): coalesced
//             row-index/value loads from HBM; gather of (z_i, dx_i) from the owner's shared
//             memory and coef(z_i + alpha_prev dx_i) -- the previous step's commit applied on the
//             fly (the owner commits it lazily, below); g/h -> d (Eq.5) -> Delta term; if
//             d_j != 0 each nonzero sends the record (li, k, d_j x_ij) with st.async into this
//             CTA's fixed region of the owner's buffer.  Then one st.async per owner carries the
//             record count (mbarrier M0).
//   phase C   every CTA, locally: wait M0 (every producer has finished its gathers), commit the
//             previous step to its own samples (z += alpha_prev dx, coef, dx = 0), wait M1 (the
//             records: expected bytes = 16 x the counts), link each record into its sample's
//             list (one atomicExch), fold each list in ascending bundle position k (registers;
//             long lists by a warp) -> d'x_i (a3), deterministic, no float atomics; per-sample
//             loss changes for a window of Armijo candidates (Eq.12, a4) plus the L1 term and
//             Delta over the CTA's own bundle positions -> one partial row, sent with st.async to
//             every CTA (M2); every CTA sums the G rows in the same fixed order and takes the
//             same decision (first q with LHS <= sigma alpha Delta).
//   commit    w_B in HBM, F (a5); z/coef of the touched samples are committed lazily by their
//             owners at the next step (and at the end of the launch).
//
// Records that do not fit a producer's region spill to the owner's HBM overflow region sized
// by the nonzeros of the owner's samples (an upper bound on what a step can send it), so every
// step size is handled; z and coef are written back to HBM at the end of the launch.
#pragma once
#include <cooperative_groups.h>

#include "pcdn_kernels.cuh"

// the window's decision taken by every warp from the partial rows (1), or by warp 0 and broadcast
// behind a CTA barrier (0).  profiles/r2c/ab_res: config 2 6.86 -> 6.75 us per step, config 3
// (P = 1024) 19.63 -> 19.23.  (The same change in the dense kernel measured 17.17 -> 17.21: not taken.)
#ifndef PCDN_RES_DECALL
#define PCDN_RES_DECALL 1
#endif

namespace pcdn {

namespace cgx = cooperative_groups;

constexpr int R_HB = 256;  // per-warp bitonic buffer for samples with many records in one step
constexpr int R_CPW = 8;   // own bundle positions per warp whose column results stay in smem
constexpr int R_WMAX = 16; // partial-row slots (WinLayout<QW>::W)
constexpr int R_RP = 4;    // own light columns per warp staged a step ahead
constexpr int R_NREG = 4;  // records of a sample folded in one thread's registers (more: a warp)
constexpr int R_TBW = 32 * NT / 32;   // touched-bitmap words (<= 32 owned samples per thread)

struct __align__(16) RRec {  // a record: sample (then: next record of the sample's list), k, value
    int32_t li;
    int32_t k;
    double v;
};

struct ResFixed {
    // mbarriers: M0 record counts, M1 records, M2/M3 line-search partial rows of even/odd
    // windows (two: a fast CTA's next-window row must not complete this window's phase)
    uint64_t mb[4];
    int64_t hst[NE_MAX + 1];
    double hg[NE_MAX][NW];
    double hh[NE_MAX][NW];
    double hd[NE_MAX];
    int64_t ce0, ce1;
    int64_t cross_e[2];
    double cross_d[2];
    HPart hpo[2];                // this CTA's partials of the columns crossing its range (DSMEM-read)
    int64_t cross_st[2], cross_en[2], cross_cs[2];
    int32_t cross_kk[2];
    double cross_w[2];
    int32_t hkk[NE_MAX], hj[NE_MAX];   // staged heavy-entry descriptors of a round
    int64_t hcs[NE_MAX];
    double hw[NE_MAX];
    HeavyPlan plan[2];           // heavy-column plan of this and the next step
    // the next step's first R_RP own light columns of every warp, staged while the CTA waits for
    // the line-search exchange: descriptor, w_j and the first 32 (row, value) pairs
    int4 stg_ci[NW][R_RP];
    double stg_w[NW][R_RP];
    int32_t stg_r[NW][R_RP][32];
    float stg_x[NW][R_RP][32];
    double red[NW][32];
    double fd[FMAX];             // the step's full columns: d_j and col_ptr[j] (dense_dx)
    int64_t fcp[FMAX];
    __align__(16) double part_in[2][16][R_WMAX];   // partial rows from every CTA, by window parity
    // the CTA's own bundle positions kk = k0 + c*NW + warp + m*G*NW, m < R_CPW: the column
    // results of phase A kept for the line search's L1 term and the w commit (slot m*NW + warp)
    // (double-buffered by step parity: the next step's phase A may write while the commit reads)
    int32_t colj[2][R_CPW * NW];
    int32_t colf[2][R_CPW * NW]; // 1 = light column computed by the slot's warp, 0 = heavy (HBM)
    double colw[2][R_CPW * NW];
    double cold[2][R_CPW * NW];
    double coldl[2][R_CPW * NW];
    unsigned long long scan_w[NW];
    int64_t ovf_base[16];        // HBM overflow base of every CTA of the cluster
    int64_t own_nnz;
    int sendcnt[16];             // records this CTA sent to each owner in the current step
    uint32_t recvcnt[16];        // records each producer CTA sent to this CTA (st.async, M0)
    int spilled;                 // this CTA wrote overflow records to HBM in the current step
    int nlong;                   // samples whose list is longer than R_NREG (queued in lq)
    int ntl[2];                  // touched owned samples of the step, by step parity
    uint32_t tb[R_TBW];          // owned samples that received a record in the current step
    int stage_n;                 // HBM staging used by long lists in the current step
    int dec_q[2], dec_bad[2];    // the decision of the window, by window parity
    double dec_alpha[2], dec_lhs[2], dec_rhs[2], dec_Delta[2], dec_nT[2];
    double F;
    long long cnt[4];
    long long pacc[16];
    int32_t sk[NHW][R_HB];
    double sv[NHW][R_HB];
};

// byte layout of the dynamic shared memory of one CTA (identical in every CTA of the cluster)
struct ResLayout {
    int Bs, cap;
    size_t zd, coef, head, lq, y, tl, recin, total;
};

__host__ __device__ inline size_t r_align16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline ResLayout res_layout(int Bs, int cap)
{
    ResLayout L;
    L.Bs = Bs;
    L.cap = cap;
    size_t o = r_align16(sizeof(ResFixed));
    L.zd = o;   o = r_align16(o + sizeof(double2) * Bs);
    L.coef = o; o = r_align16(o + sizeof(double2) * Bs);
    L.head = o; o = r_align16(o + sizeof(int32_t) * Bs);
    L.lq = o;   o = r_align16(o + sizeof(int32_t) * Bs);
    L.y = o;    o = r_align16(o + 2 * (size_t)Bs + 4);   // label bitmap of ALL samples (s <= 16 Bs)
    L.tl = o;   o = r_align16(o + 2 * sizeof(uint16_t) * Bs);   // touched lists, by step parity
    L.recin = o; o = r_align16(o + sizeof(RRec) * cap);
    L.total = o;
    return L;
}
constexpr int R_BYTES_PER_RECORD = 16;

struct ResCtx {
    ResFixed *fx;
    double2 *zd, *coef;
    int32_t *head, *lq;
    uint32_t *ybits;   // bit i = (y_i > 0), every sample of the problem (constant per launch)
    uint16_t *tls;     // [2][Bs] touched owned samples (ascending li) of the step, by step parity
    RRec *recin;
    int lg, G, c, Bs, Bsc, cap, capP, per;
    int64_t my_ovf;
    double alpha_prev;   // the accepted step of the previous bundle step (0: none / null step)
    int cb;              // column-slot buffer of the current step (step parity)
    long long *tl;       // per-warp timeline slot of the current step (profiling mode 2), or null
};

// ---------------------------------------------------------------------------------------
// DSMEM / mbarrier primitives (sm_90+ PTX)
// ---------------------------------------------------------------------------------------
#ifdef PCDN_ALIGN_CHECK
#include <cstdio>
#define RCHK(p, al, site)                                                                          \
    do {                                                                                           \
        if (((uintptr_t)(p)) & ((al)-1)) {                                                         \
            printf("PCDN misaligned site %d ptr %p (cta %d tid %d)\n", site, (void *)(p), (int)blockIdx.x, (int)threadIdx.x); \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define RCHK(p, al, site) do {} while (0)
#endif
template <typename T>
__device__ __forceinline__ T *remote(T *p, int rank)
{
    T *r = cgx::this_cluster().map_shared_rank(p, (unsigned)rank);
    RCHK(r, alignof(T), 1);
    return r;
}
__device__ __forceinline__ uint32_t s_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// 16-byte load from another CTA's shared memory by a shared::cluster address (mapa), without
// generic-address translation
__device__ __forceinline__ double2 ld_dsmem_f64x2(uint32_t raddr)
{
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(raddr) : "memory");
    return v;
}

__device__ __forceinline__ void st_async_u32(uint32_t raddr, uint32_t v, uint32_t rbar)
{
    RCHK(raddr, 4, 4);
    RCHK(rbar, 8, 5);
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];"
                 :: "r"(raddr), "r"(v), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double a0, double a1, uint32_t rbar)
{
    RCHK(raddr, 16, 2);
    RCHK(rbar, 8, 3);
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 :: "r"(raddr), "d"(a0), "d"(a1), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
// Wait for the phase with the given parity (acquire, cluster scope).  A phase that does not
// complete within ~4 s of SM clock means a broken protocol: trap instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    uint32_t done;
    const long long t0 = clock64();
    do {
        asm volatile("{\n\t.reg .pred P;\n\t"
                     "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, P;\n\t}"
                     : "=r"(done) : "r"(bar), "r"(parity) : "memory");
        if (!done && clock64() - t0 > 8000000000LL) __trap();
    } while (!done);
}
// orders this CTA's shared-memory writes before a later cluster-scope signal (MEMBAR.CTA only)
__device__ __forceinline__ void fence_smem_release_cluster()
{
    asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ int res_ybit(const ResCtx &R, int32_t i) { return (R.ybits[i >> 5] >> (i & 31)) & 1u ? 1 : -1; }
__device__ __forceinline__ int res_y(const ResCtx &R, int li) { return res_ybit(R, li * R.G + R.c); }

// coef of sample i after the previous step: from the owner's (z_i, dx_i) and alpha_prev; a
// sample the previous step did not touch has dx_i = 0 and its stored coef is used as is
__device__ __forceinline__ double2 res_coef(const StepArgs &a, const ResCtx &R, int32_t i)
{
    const int owner = i & (R.G - 1);
    const int li = i >> R.lg;
    const double2 zd = ld_dsmem_f64x2(mapa_u32(s_addr(&R.zd[li]), owner));
    const double2 cf = ld_dsmem_f64x2(mapa_u32(s_addr(&R.coef[li]), owner));
    const int yi = res_ybit(R, i);   // local bitmap: no dependent L2 load for a touched sample
    if (zd.y == 0.0) return cf;
    return coef_next(a.loss, cf, zd.x + R.alpha_prev * zd.y, R.alpha_prev * zd.y, yi);
}

// SCDN (Alg.2; synchronous reading Z27): feature j's own 1-D Armijo step
// (Eq.6 with d = d_j e_j) from the step's start state, by the warp that owns the column.  Per
// candidate alpha = beta^q: the column's loss change (the owner state re-gathered per chunk of 32
// nonzeros, the previous step applied on the fly), warp-summed in a fixed order, plus the
// separable terms.  Returns alpha_j (0: no candidate passes, a null update).
__device__ double res_scdn_alpha(const StepArgs &a, const ResCtx &R, int64_t p0, int64_t p1, const int32_t *srow,
                                 const float *sx, double d, double wj, double delta, int lane)
{
    double alpha = 1.0;
    for (int q = 0; q <= a.qmax; q++) {
        double chg = 0.0;
        for (int64_t pb = p0; pb < p1; pb += 32) {
            const int64_t p = pb + lane;
            if (p < p1) {
                const bool st = srow && pb == p0;
                const int32_t i = st ? srow[lane] : __ldg(&a.row_idx[p]);
                const double x = (double)(st ? sx[lane] : __ldg(&a.val[p]));
                const int owner = i & (R.G - 1), li = i >> R.lg;
                const double2 zd = ld_dsmem_f64x2(mapa_u32(s_addr(&R.zd[li]), owner));
                const double2 cf = ld_dsmem_f64x2(mapa_u32(s_addr(&R.coef[li]), owner));
                const int yi = res_ybit(R, i);
                const double zc = zd.x + R.alpha_prev * zd.y;
                const double2 cc = zd.y == 0.0 ? cf : coef_next(a.loss, cf, zc, R.alpha_prev * zd.y, yi);
                chg += loss_change(a.loss, zc, yi, cc.x, d * x, alpha);
            }
        }
        chg = warp_sum(chg);
        const double wn = wj + alpha * d;
        const double lhs = a.c * chg + fabs(wn) - fabs(wj) + a.mu * alpha * d * (wj + 0.5 * alpha * d);
        if (lhs <= a.sigma * alpha * delta) return alpha;
        alpha *= a.beta;
    }
    return 0.0;
}

// Send the records (sample i, bundle position k, d_k x_ik) of the warp's valid lanes to their
// owners.  Every producer CTA p has a fixed region [p*capP, (p+1)*capP) of each owner's record
// buffer; the slot comes from a LOCAL shared-memory counter per owner (one atomic per group of
// lanes with the same owner), the record travels by st.async and completes 16 bytes on the
// owner's M1.  Records beyond the region go to the owner's HBM overflow (global atomic slot;
// rare).  All 32 lanes must call.
__device__ __forceinline__ void res_emit_warp(const StepArgs &a, const ResCtx &R, bool valid, int32_t i, int32_t k,
                                              double v, int lane)
{
    const int owner = valid ? (i & (R.G - 1)) : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, owner);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (valid && lane == leader) base = atomicAdd(&R.fx->sendcnt[owner], __popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!valid) return;
    const int slot = base + __popc(grp & ((1u << lane) - 1u));
    RRec r;
    r.li = i >> R.lg;
    r.k = k;
    r.v = v;
    const double2 raw = *reinterpret_cast<const double2 *>(&r);
    if (slot < R.capP) {
        st_async_f64x2(mapa_u32(s_addr(&R.recin[R.c * R.capP + slot]), owner), raw.x, raw.y,
                       mapa_u32(s_addr(&R.fx->mb[1]), owner));
    } else {
        const int gs = atomicAdd(&a.ovf_cnt[owner], 1);
        __stcg(reinterpret_cast<double2 *>(&a.rec[R.fx->ovf_base[owner] + gs]), raw);
        R.fx->spilled = 1;
    }
}

__device__ __forceinline__ void res_col_gh(const StepArgs &a, const ResCtx &R, int64_t p0, int64_t p1, int lane,
                                           double &gs, double &hs)
{
    double g = 0.0, h = 0.0;
#pragma unroll 4
    for (int64_t p = p0 + lane; p < p1; p += 32) {
        const int32_t i = __ldg(&a.row_idx[p]);
        const double x = (double)__ldg(&a.val[p]);
        const double2 cf = res_coef(a, R, i);
        g += x * cf.x;
        h += (x * x) * cf.y;
    }
    gs = warp_sum(g);
    hs = warp_sum(h);
}

__device__ __forceinline__ void res_col_scatter(const StepArgs &a, const ResCtx &R, int64_t p0, int64_t p1, int lane,
                                                int32_t kpos, double d)
{
    for (int64_t pb = p0; pb < p1; pb += 32) {
        const int64_t p = pb + lane;
        const bool ok = p < p1;
        const int32_t i = ok ? __ldg(&a.row_idx[p]) : 0;
        const double v = ok ? d * (double)__ldg(&a.val[p]) : 0.0;
        res_emit_warp(a, R, ok, i, kpos, v, lane);
    }
}

// a received record by slot index: the shared buffer below cap, the CTA's HBM overflow above
__device__ __forceinline__ RRec res_rec(const StepArgs &a, const ResCtx &R, int phys)
{
    double2 raw;
    RCHK(&R.recin[phys], 16, 6);
    if (phys < R.cap) raw = *reinterpret_cast<const double2 *>(&R.recin[phys]);
    else raw = __ldcg(reinterpret_cast<const double2 *>(&a.rec[R.my_ovf + (phys - R.cap)]));
    return *reinterpret_cast<const RRec *>(&raw);
}

// Fold of one long list (> R_NREG records) by a warp.  Lane 0 walks the list into HBM staging
// (the CTA's rec2 region); <= R_HB records are bitonic-sorted by k in shared memory and summed
// by lane-contiguous partials combined in a fixed tree; longer lists by repeated warp-wide
// minimum extraction.  The k of one sample's records are distinct (one record per column).
__device__ double res_fold_long(const StepArgs &a, const ResCtx &R, int h, int lane, int32_t *sk, double *sv)
{
    int n = 0;
    long long base = 0;
    RRec *stage = reinterpret_cast<RRec *>(a.rec2);
    if (lane == 0) {
        for (int p = h; p >= 0; p = res_rec(a, R, p).li) n++;
        base = R.my_ovf + atomicAdd(&R.fx->stage_n, n);
        int t = 0;
        for (int p = h; p >= 0;) {
            const RRec r = res_rec(a, R, p);
            __stcg(reinterpret_cast<double2 *>(&stage[base + t]), *reinterpret_cast<const double2 *>(&r));
            t++;
            p = r.li;
        }
    }
    n = __shfl_sync(0xffffffffu, n, 0);
    base = __shfl_sync(0xffffffffu, base, 0);
    __syncwarp();
    const RRec *seg = stage + base;
    auto ld = [&](int r, int32_t &k, double &v) {
        const double2 raw = __ldcg(reinterpret_cast<const double2 *>(&seg[r]));
        k = (int32_t)(__double_as_longlong(raw.x) >> 32);
        v = raw.y;
    };
    if (n <= R_HB) {
        int npow = 32;
        while (npow < n) npow <<= 1;
        for (int r = lane; r < npow; r += 32) {
            if (r < n) {
                ld(r, sk[r], sv[r]);
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
        const int chunk = (n + 31) / 32;
        double s = 0.0;
        for (int r = lane * chunk; r < min(n, (lane + 1) * chunk); r++) s += sv[r];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_down_sync(0xffffffffu, s, o);
            if ((lane & (2 * o - 1)) == 0) s += t;
        }
        __syncwarp();
        return __shfl_sync(0xffffffffu, s, 0);
    }
    double dx = 0.0;
    int last = -1;
    for (int t = 0; t < n; t++) {
        int best = 0x7fffffff;
        double bv = 0.0;
        for (int r = lane; r < n; r += 32) {
            int32_t k;
            double v;
            ld(r, k, v);
            if (k > last && k < best) {
                best = k;
                bv = v;
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

// per-warp timeline point (profiling mode 2)
#define RTL(R, pt)                                                    \
    do {                                                              \
        if ((R).tl && (threadIdx.x & 31) == 0) (R).tl[pt] = clock64(); \
    } while (0)

struct ResProf {   // profiling mode: CTA 0 thread 0 accumulates clock64 cycles per phase
    bool on;
    long long t;
    __device__ __forceinline__ void start() { if (on) t = clock64(); }
    __device__ __forceinline__ void mark(ResFixed &fx, int i)
    {
        if (on) {
            const long long now = clock64();
            fx.pacc[i] += now - t;
            t = now;
        }
    }
};

// Commit the previous step to this CTA's own samples (lazily: every producer has finished
// gathering them): z += alpha_prev dx (Alg.4 l.5 with additive retained z), coef, dx = 0.  A
// sample the previous step did not touch has dx = 0 (a no-op, as is a touched one whose dx
// cancelled to 0).  Used at the end of a launch; inside the step loop the commit is fused into
// the first fold pass of the next step.
__device__ __forceinline__ void res_lazy_commit(const StepArgs &a, const ResCtx &R, int tid)
{
    for (int r = 0; r < R.per; r++) {
        const int li = tid + r * NT;
        if (li >= R.Bsc) break;
        const double2 zd = R.zd[li];
        if (zd.y == 0.0) continue;
        const double zn = zd.x + R.alpha_prev * zd.y;
        R.zd[li] = make_double2(zn, 0.0);
        R.coef[li] = coef_next(a.loss, R.coef[li], zn, R.alpha_prev * zd.y, res_y(R, li));
    }
}

// Stage the first R_RP own light columns of the step [kb, ke) for this warp (its own slots only,
// so no CTA-level synchronisation): all descriptor loads first, then all data loads, then stores.
// w_j may be read early: the bundles of a launch are disjoint.
__device__ __forceinline__ void res_stage_cols(const StepArgs &a, ResFixed &fx, int64_t kb, int64_t ke, int64_t gw,
                                               int64_t GN, int warp, int lane)
{
    int4 ci[R_RP];
#pragma unroll
    for (int m = 0; m < R_RP; m++) {
        const int64_t kk = kb + gw + (int64_t)m * GN;
        ci[m] = kk < ke ? __ldg(&a.colinfo[kk]) : make_int4(0, -1, 0, 0);
    }
    int32_t r[R_RP];
    float x[R_RP];
    double w[R_RP];
#pragma unroll
    for (int m = 0; m < R_RP; m++) {
        const int len = ci[m].y;
        const bool light = len >= 0 && len <= a.heavy_len;
        r[m] = 0;
        x[m] = 0.f;
        w[m] = 0.0;
        if (light && lane < len) {
            const int64_t p = colinfo_p0(ci[m]) + lane;
            r[m] = __ldg(&a.row_idx[p]);
            x[m] = __ldg(&a.val[p]);
        }
        if (light && lane == 0) w[m] = ldcg(&a.w[ci[m].x]);
    }
#pragma unroll
    for (int m = 0; m < R_RP; m++) {
        if (lane == 0) {
            fx.stg_ci[warp][m] = ci[m];
            fx.stg_w[warp][m] = w[m];
        }
        fx.stg_r[warp][m][lane] = r[m];
        fx.stg_x[warp][m][lane] = x[m];
    }
    __syncwarp();
}

// L2 prefetch of everything res_stage_cols will load for the next step [kb, ke) of this CTA (the
// descriptors, the row / value lines and w_j of the NW x R_RP staged columns), issued by one warp
// during the fold, where the upper warps idle when the step touches fewer samples than threads:
// the staging after the partial-row send then hits L2 instead of HBM.
__device__ __forceinline__ void res_l2_prefetch_next(const StepArgs &a, int64_t kb, int64_t ke, int c, int G, int lane)
{
    const int64_t GN = (int64_t)G * NW;
#pragma unroll
    for (int e = 0; e < (NW * R_RP + 31) / 32; e++) {
        const int idx = lane + 32 * e, w = idx % NW, m = idx / NW;
        const int64_t kk = kb + (int64_t)c * NW + w + (int64_t)m * GN;
        if (m < R_RP && kk < ke) {
            const int4 ci = __ldg(&a.colinfo[kk]);
            if (ci.y > 0 && ci.y <= a.heavy_len) {
                const int64_t p0 = colinfo_p0(ci), p1 = p0 + ci.y - 1;
                prefetch_l2(&a.row_idx[p0]);
                prefetch_l2(&a.row_idx[p1]);
                prefetch_l2(&a.val[p0]);
                prefetch_l2(&a.val[p1]);
                prefetch_l2(&a.w[ci.x]);
            }
        }
    }
}

// The owner state of the next step's first staged column, gathered while the current step's
// decision is taken (valid from the M2 arrival of window 0 to the next step's M0: no owner writes
// its samples in between)
struct Pref {
    double2 zd, cf;
    int y;
    bool ok;
};

// One Armijo window over candidates q0 .. q0+NQ-1 (Eq.6 with Eq.12 from retained quantities):
// per-sample loss changes over this CTA's touched samples (window 0 also folds d'x_i), the L1
// term and Delta over the CTA's own bundle positions, a fixed-order CTA partial row, sent to
// every CTA of the cluster (st.async, M2); each CTA sums the G rows in the same fixed order and
// takes the same decision.
template <int NQ>
__device__ __forceinline__ void res_window(const StepArgs &a, const ResCtx &R, WinState &ws, int64_t k0, int64_t k1,
                                          int tid, int lane, int warp, ResProf &pr, int wcount, const DenseInfo &di,
                                          int64_t kn0, int64_t kn1, Pref &pf)
{
    using LY = WinLayout<NQ>;
    constexpr int W = LY::W;
    ResFixed &fx = *R.fx;
    double alpha0 = 1.0;
    for (int q = 0; q < ws.q0; q++) alpha0 *= a.beta;
    double acc[W];
#pragma unroll
    for (int q = 0; q < W; q++) acc[q] = 0.0;
    int ntouch = 0;
    unsigned longmask = 0;   // owned samples (bit r) whose list is longer than R_NREG
    // the step's touched owned samples (ascending li; every owned sample when a full column moved):
    // thread tid takes entries tid, tid + NT, ...  The previous step is already committed.
    const uint16_t *tl = R.tls + (size_t)R.cb * R.Bs;
    const int nT = fx.ntl[R.cb];
    if (ws.win == 0) {
        unsigned tm = 0;
        for (int r = 0;; r++) {
            const int e = tid + r * NT;
            if (e >= nT) break;
            const int li = tl[e];
            const double2 zd = R.zd[li];
            const int h = R.head[li];
            tm |= 1u << r;
            ntouch++;
            // full columns first (bundle order), then the records (ascending k): a fixed order
            const double dxd = di.any ? dense_dx(a, fx.fd, fx.fcp, di, k0, (int64_t)li * R.G + R.c) : 0.0;
            double dx;
            RRec rc;
            if (h < 0) {
                dx = 0.0;
            } else if ((rc = res_rec(a, R, h)).li < 0) {   // one record: the common case
                dx = rc.v;
                R.head[li] = -1;
            } else {
                // up to R_NREG records: gather, then add in ascending k (selection in registers)
                int kk[R_NREG];
                double vv[R_NREG];
                kk[0] = rc.k;
                vv[0] = rc.v;
                int ni = 1, p = rc.li;
#pragma unroll
                for (int e2 = 1; e2 < R_NREG; e2++) {
                    kk[e2] = 0x7fffffff;
                    vv[e2] = 0.0;
                    if (p >= 0) {
                        rc = res_rec(a, R, p);
                        kk[e2] = rc.k;
                        vv[e2] = rc.v;
                        p = rc.li;
                        ni++;
                    }
                }
                if (p >= 0) {   // long list: folded by a warp after the CTA reduction below
                    longmask |= 1u << r;
                    R.zd[li] = make_double2(zd.x, dxd);
                    R.lq[atomicAdd(&fx.nlong, 1)] = li;
                    continue;
                }
                R.head[li] = -1;
                dx = 0.0;
                int last = -1;
#pragma unroll 1
                for (int t = 0; t < ni; t++) {   // not unrolled: a small hot instruction footprint
                    int best = 0x7fffffff;
                    double bv = 0.0;
#pragma unroll
                    for (int e2 = 0; e2 < R_NREG; e2++) {
                        const bool take = kk[e2] > last && kk[e2] < best;
                        best = take ? kk[e2] : best;
                        bv = take ? vv[e2] : bv;
                    }
                    last = best;
                    dx += bv;
                }
                if (last == 0x7fffffff) atomicMax(a.status, 6);   // a repeated position: internal error
            }
            dx = dxd + dx;
            R.zd[li] = make_double2(zd.x, dx);
            if (a.debug) {
                const int64_t i = (int64_t)li * R.G + R.c;
                a.dbg_dx[i] = dx;
                a.dbg_mark[i] = 1;
            }
            const double cg = R.coef[li].x;
            const int yi = res_y(R, li);
            double al = alpha0;
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                acc[q] += loss_change(a.loss, zd.x, yi, cg, dx, al);
                al *= a.beta;
            }
        }
        ws.tmask = tm;
    } else {
        for (int r = 0; r < 32; r++) {
            if (!((ws.tmask >> r) & 1u)) continue;
            const int li = tl[tid + r * NT];
            ntouch++;
            const double2 zd = R.zd[li];
            const double cg = R.coef[li].x;
            const int yi = res_y(R, li);
            double al = alpha0;
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                acc[q] += loss_change(a.loss, zd.x, yi, cg, zd.y, al);
                al *= a.beta;
            }
        }
    }
    // L1 part of Eq.12 and Delta over this CTA's own bundle positions (monotone in s2)
    for (int s2 = tid;; s2 += NT) {
        const int m = s2 / NW, wq = s2 - m * NW;
        const int64_t kk = k0 + (int64_t)R.c * NW + wq + (int64_t)m * R.G * NW;
        if (kk >= k1) break;
        double wj, d, dl;
        if (m < R_CPW && fx.colf[R.cb][s2]) {
            wj = fx.colw[R.cb][s2];
            d = fx.cold[R.cb][s2];
            dl = fx.coldl[R.cb][s2];
        } else {
            wj = ldcg(&a.w[__ldg(&a.order[kk])]);
            d = ldcg(&a.dk[kk - k0]);
            dl = ldcg(&a.deltak[kk - k0]);
        }
        double al = alpha0;
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            acc[NQ + q] += fabs(wj + al * d) - fabs(wj) + a.mu * al * d * (wj + 0.5 * al * d);
            al *= a.beta;
        }
        acc[LY::DELTA] += dl;
    }
    acc[LY::NTOUCH] = (double)ntouch;
    pr.mark(fx, 3);
    if (ws.win == 0) RTL(R, 8);
    if (ws.win == 0 && kn0 < kn1 && warp == NW - 1) res_l2_prefetch_next(a, kn0, kn1, R.c, R.G, lane);
    constexpr int SPL = 32 / W;
    {
        const double tot = xreduce<W>(acc, lane);
        if ((lane % SPL) == 0) fx.red[warp][lane / SPL] = tot;
    }
    __syncthreads();
    if (ws.win == 0) RTL(R, 9);
    if (ws.win == 0 && fx.nlong > 0) {
        // rare: samples with more than R_NREG records in this step.  Warps fold their lists, the
        // owning threads add their loss changes, and the per-warp rows get a second fixed-order
        // contribution (the structure depends only on the data, so results stay deterministic).
        const int nl = fx.nlong;
        if (warp < NHW) {
            for (int e = warp; e < nl; e += NHW) {
                const int li = R.lq[e];
                const double dxr = res_fold_long(a, R, R.head[li], lane, fx.sk[warp], fx.sv[warp]);
                if (lane == 0) {
                    R.zd[li].y = R.zd[li].y + dxr;   // dense part + records
                    R.head[li] = -1;
                    if (a.debug) {
                        const int64_t i = (int64_t)li * R.G + R.c;
                        a.dbg_dx[i] = R.zd[li].y;
                        a.dbg_mark[i] = 1;
                    }
                }
            }
        }
        __syncthreads();
        double acc2[W];
#pragma unroll
        for (int q = 0; q < W; q++) acc2[q] = 0.0;
        for (int r = 0; r < 32; r++) {   // each owner thread, in its own fixed order
            if (!((longmask >> r) & 1u)) continue;
            const int li = tl[tid + r * NT];
            const double2 zd = R.zd[li];
            const double cg = R.coef[li].x;
            const int yi = res_y(R, li);
            double al = alpha0;
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                acc2[q] += loss_change(a.loss, zd.x, yi, cg, zd.y, al);
                al *= a.beta;
            }
        }
        const double tot2 = xreduce<W>(acc2, lane);
        if ((lane % SPL) == 0) fx.red[warp][lane / SPL] += tot2;
        __syncthreads();
    }
    const int buf = wcount & 1;
    const uint32_t mb2 = s_addr(&fx.mb[2 + buf]);
    if (warp == 0) {
        // this CTA's partial row -> part_in[buf][c][*] of every CTA (st.async, M2)
        double sv = 0.0;
        if (lane < W) {
#pragma unroll
            for (int w2 = 0; w2 < NW; w2++) sv += fx.red[w2][lane];
        }
        fence_smem_release_cluster();   // zd (dx, lazy commit) must be visible to the gathers
        constexpr int HW = W / 2;
        for (int base = 0; base < R.G * HW; base += 32) {
            const int idx = base + lane;
            const int q = idx % HW;
            const double v0 = __shfl_sync(0xffffffffu, sv, 2 * q);
            const double v1 = __shfl_sync(0xffffffffu, sv, 2 * q + 1);
            if (idx < R.G * HW) {
                const int dst = idx / HW;
                st_async_f64x2(mapa_u32(s_addr(&fx.part_in[buf][R.c][2 * q]), dst), v0, v1, mapa_u32(mb2, dst));
            }
        }
        if (lane == 0) mbar_arrive_tx(mb2, (uint32_t)(8 * W * R.G));
    }
    // while the partial rows travel: stage the next step's own light columns (window 0 only)
    if (ws.win == 0 && kn0 < kn1) res_stage_cols(a, fx, kn0, kn1, (int64_t)R.c * NW + warp, (int64_t)R.G * NW, warp, lane);
    if (ws.win == 0) RTL(R, 10);
    mbar_wait(mb2, (uint32_t)((wcount >> 1) & 1));
    if (ws.win == 0) RTL(R, 11);
    // every fold of this step is done (all partial rows arrived): gather the owner state of the
    // next step's first staged column now, overlapped with the decision below (warp 0, which takes
    // the decision, gathers after it: its shared-memory reads must not queue behind remote loads)
    auto prefetch = [&]() {
        if (ws.win == 0 && kn0 < kn1) {
            const int len = fx.stg_ci[warp][0].y;
            pf.ok = len >= 0 && len <= a.heavy_len;
            if (pf.ok && lane < len) {
                const int32_t i = fx.stg_r[warp][0][lane];
                const int owner = i & (R.G - 1), li = i >> R.lg;
                pf.zd = ld_dsmem_f64x2(mapa_u32(s_addr(&R.zd[li]), owner));
                pf.cf = ld_dsmem_f64x2(mapa_u32(s_addr(&R.coef[li]), owner));
                pf.y = res_ybit(R, i);
            }
        }
    };
#if PCDN_RES_DECALL
    pr.mark(fx, 4);
    // every warp: the G partial rows (local now), the same fixed-order sums and the same decision
    // (identical in every warp of every CTA: no broadcast, no CTA barrier), then the gather of the
    // next step's first staged column (after the decision: its shared-memory reads must not queue
    // behind remote loads).  part_in[buf] is refilled only after every CTA has received this CTA's
    // next row, which its warps contribute to after this point.
    {
        double tot = 0.0;
        if (lane < W) {
            double v[16];
#pragma unroll
            for (int r = 0; r < 16; r++) v[r] = r < R.G ? fx.part_in[buf][r][lane] : 0.0;
#pragma unroll
            for (int r = 0; r < 16; r++) tot += v[r];
        }
        const double Dl = __shfl_sync(0xffffffffu, tot, LY::DELTA);
        const double nTt = __shfl_sync(0xffffffffu, tot, LY::NTOUCH);
        int qa = -1, badl = 0;
        double al = alpha0, la = 0.0, ra = 0.0, alpha_a = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            const double Ls = __shfl_sync(0xffffffffu, tot, q);
            const double L1 = __shfl_sync(0xffffffffu, tot, NQ + q);
            if (qa < 0 && !badl) {
                const double lhs = L1 + a.c * Ls;
                const double rhs = a.sigma * al * Dl;
                if (!isfinite(lhs) || (!a.scdn && !isfinite(Dl))) {
                    badl = 1;
                } else if (a.scdn || lhs <= rhs) {   // SCDN takes the combined step as it is (Z27)
                    qa = ws.q0 + q;
                    alpha_a = al;
                    la = lhs;
                    ra = rhs;
                }
                al *= a.beta;
            }
        }
        ws.qacc = qa;
        ws.bad = badl;
        ws.alpha = alpha_a;
        ws.lhs = la;
        ws.rhs = ra;
        ws.Delta = Dl;
        ws.nT_tot = nTt;
    }
    prefetch();
#else
    if (warp != 0) prefetch();
    pr.mark(fx, 4);
    // warp 0: the G partial rows (local now), fixed-order tree, decision; broadcast in the CTA
    // (every CTA computes the identical decision)
    if (warp == 0) {
        // lane l < W sums slot l over the G rows in row order (independent loads, one add chain:
        // shorter than a shuffle tree's dependent levels)
        double tot = 0.0;
        if (lane < W) {
            double v[16];
#pragma unroll
            for (int r = 0; r < 16; r++) v[r] = r < R.G ? fx.part_in[buf][r][lane] : 0.0;
#pragma unroll
            for (int r = 0; r < 16; r++) tot += v[r];
        }
        const double Dl = __shfl_sync(0xffffffffu, tot, LY::DELTA);
        const double nTt = __shfl_sync(0xffffffffu, tot, LY::NTOUCH);
        int qa = -1, badl = 0;
        double al = alpha0, la = 0.0, ra = 0.0, alpha_a = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            const double Ls = __shfl_sync(0xffffffffu, tot, q);
            const double L1 = __shfl_sync(0xffffffffu, tot, NQ + q);
            if (qa < 0 && !badl) {
                const double lhs = L1 + a.c * Ls;
                const double rhs = a.sigma * al * Dl;
                if (!isfinite(lhs) || (!a.scdn && !isfinite(Dl))) {
                    badl = 1;
                } else if (a.scdn || lhs <= rhs) {   // SCDN takes the combined step as it is (Z27)
                    qa = ws.q0 + q;
                    alpha_a = al;
                    la = lhs;
                    ra = rhs;
                }
                al *= a.beta;
            }
        }
        if (lane == 0) {
            fx.dec_q[buf] = qa;
            fx.dec_bad[buf] = badl;
            fx.dec_alpha[buf] = alpha_a;
            fx.dec_lhs[buf] = la;
            fx.dec_rhs[buf] = ra;
            fx.dec_Delta[buf] = Dl;
            fx.dec_nT[buf] = nTt;
        }
        prefetch();
    }
    __syncthreads();   // dec_*[buf] is rewritten two windows later, after two more syncs
    ws.qacc = fx.dec_q[buf];
    ws.bad = fx.dec_bad[buf];
    ws.alpha = fx.dec_alpha[buf];
    ws.lhs = fx.dec_lhs[buf];
    ws.rhs = fx.dec_rhs[buf];
    ws.Delta = fx.dec_Delta[buf];
    ws.nT_tot = fx.dec_nT[buf];
#endif
    if (ws.win == 0) RTL(R, 12);
    ws.win++;
    pr.mark(fx, 5);
}

template <int LOSS, bool SCDN>
__global__ void __launch_bounds__(NT, 1) k_step_res(StepArgs a)
{
    if (a.stop && ldcg(a.stop)) return;   // the solve already ended (queued ahead; grid-uniform)
    a.loss = LOSS;   // a compile-time loss: the other loss's code is dead (smaller instruction footprint)
    a.scdn = SCDN;   // likewise the SCDN baseline's per-feature line search
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;   // one cluster = the whole grid
    ResCtx R;
    {
        // array offsets come from the kernel parameters (constant bank): cheap to rematerialize
        R.fx = reinterpret_cast<ResFixed *>(smem_raw);
        R.zd = reinterpret_cast<double2 *>(smem_raw + a.res_off[0]);
        R.coef = reinterpret_cast<double2 *>(smem_raw + a.res_off[1]);
        R.head = reinterpret_cast<int32_t *>(smem_raw + a.res_off[2]);
        R.lq = reinterpret_cast<int32_t *>(smem_raw + a.res_off[3]);
        R.ybits = reinterpret_cast<uint32_t *>(smem_raw + a.res_off[4]);
        R.tls = reinterpret_cast<uint16_t *>(smem_raw + a.res_off[6]);
        R.recin = reinterpret_cast<RRec *>(smem_raw + a.res_off[5]);
        R.lg = a.res_lg;
        R.G = G;
        R.c = c;
        R.Bs = a.res_Bs;
        R.cap = a.res_cap;
        R.capP = a.res_cap / G;
        R.Bsc = (int)((a.s - c + G - 1) / G);   // samples owned by this CTA
        R.per = (R.Bsc + NT - 1) / NT;          // owned samples per thread (interleaved)
        R.alpha_prev = 0.0;
        R.tl = nullptr;
        R.cb = 0;
    }
    ResFixed &fx = *R.fx;
    RCHK(R.zd, 16, 7);
    RCHK(R.coef, 16, 8);
    RCHK(R.recin, 16, 9);
    RCHK(&fx.part_in[0][0][0], 16, 10);
    const int64_t GN = (int64_t)G * NW;
    const int64_t gw = (int64_t)c * NW + warp;
    const uint32_t mb0 = s_addr(&fx.mb[0]), mb1 = s_addr(&fx.mb[1]);

    // ---------------- prologue: owned per-sample state into shared memory, mbarriers --------
    long long own = 0;
    for (int li = tid; li < R.Bsc; li += NT) {
        const int64_t i = (int64_t)li * G + c;
        R.zd[li] = make_double2(ldcg(&a.z[i]), 0.0);
        R.coef[li] = ldcg(&a.coef[i]);
        R.head[li] = -1;
        own += __ldg(&a.row_ptr[i + 1]) - __ldg(&a.row_ptr[i]);
    }
    // label bitmap: 8 words (256 samples) per warp and round, all loads in flight together
    for (int64_t wb = (int64_t)warp * 256; wb < a.s; wb += 256 * NW) {
        int8_t v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int64_t i = wb + u * 32 + lane;
            v[u] = i < a.s ? a.y[i] : (int8_t)0;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const unsigned m = __ballot_sync(0xffffffffu, v[u] > 0);
            if (lane == 0 && wb + u * 32 < a.s) R.ybits[(wb >> 5) + u] = m;
        }
    }
    own = warp_sum(own);
    if (lane == 0) fx.scan_w[warp] = (unsigned long long)own;
    if (tid < 16) fx.pacc[tid] = 0;
    for (int w = tid; w < R_TBW; w += NT) fx.tb[w] = 0u;
    if (tid < 16) {
        fx.sendcnt[tid] = 0;
        fx.recvcnt[tid] = 0;
    }
    if (tid == 0) {
        for (int b = 0; b < 4; b++) mbar_init(s_addr(&fx.mb[b]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fx.nlong = 0;
        fx.stage_n = 0;
        fx.spilled = 0;
        fx.ntl[0] = fx.ntl[1] = 0;
        fx.F = ldcg(a.F);
        for (int i = 0; i < 4; i++) fx.cnt[i] = 0;
    }
    __syncthreads();
    if (tid == 0) {
        long long t = 0;
        for (int w2 = 0; w2 < NW; w2++) t += (long long)fx.scan_w[w2];
        fx.own_nnz = t;
    }
    cluster_sync_all();   // every CTA's state and mbarriers are initialised
    if (warp == 0) {
        const long long mine = lane < G ? (long long)*remote(&fx.own_nnz, lane) : 0;
        long long incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane < G) fx.ovf_base[lane] = incl - mine;
    }
    if (warp == 1) heavy_plan_warp(a, 0, min(a.P, a.ntot), c, G, lane, &fx.plan[0]);
    __syncthreads();
    R.my_ovf = fx.ovf_base[c];

    ResProf pr;
    pr.on = PCDN_PROFILE && a.prof != nullptr && c == 0 && tid == 0;
    pr.t = 0;
    const bool prof = pr.on;
#define PROF_MARK(i) pr.mark(fx, i)
    int prev_q = 0;
    Pref pf;
    pf.ok = false;
    int wcount = 0;            // windows so far in this launch (M2 phase parity)
    uint32_t ph = 0;           // bit 0: M0 parity, bit 1: M1 parity
    res_stage_cols(a, fx, 0, min(a.P, a.ntot), gw, GN, warp, lane);
    for (int64_t t = 0; t < a.nsteps; t++) {
        pr.start();
        R.cb = (int)(t & 1);
        R.tl = (PCDN_PROFILE && a.tl && c == 0 && t < TL_STEPS) ? a.tl + (t * NW + warp) * TL_PTS : nullptr;
        RTL(R, 0);
        const int64_t k0 = t * a.P;
        const int64_t k1 = min(k0 + a.P, a.ntot);
        const int64_t Pt = k1 - k0;
        const int64_t kn1 = min(k1 + a.P, a.ntot);

        // ---------------- phase A: light columns, one warp per column (a1, a2, a3) --------
        {
            int m = 0;
            for (int64_t kk = k0 + gw; kk < k1; kk += GN, m++) {
                const bool stg = m < R_RP;   // staged during the previous step (res_stage_cols)
                const int4 ci = stg ? fx.stg_ci[warp][m] : __ldg(&a.colinfo[kk]);
                const int32_t j = ci.x, len = ci.y;
                const int64_t p0 = colinfo_p0(ci);
                const int slot = m * NW + warp;
                if (len > a.heavy_len) {
                    if (lane == 0 && m < R_CPW) fx.colf[R.cb][slot] = 0;
                    continue;
                }
                const int64_t p1 = p0 + len;
                double gs, hs;
                {
                    double g = 0.0, h = 0.0;
                    int64_t pr0 = p0;
                    if (stg) {
                        if (lane < len) {
                            const double x = (double)fx.stg_x[warp][m][lane];
                            double2 cf;
                            if (m == 0 && pf.ok) {   // gathered during the previous step's decision
                                cf = pf.zd.y == 0.0 ? pf.cf
                                                    : coef_next(a.loss, pf.cf, pf.zd.x + R.alpha_prev * pf.zd.y,
                                                                R.alpha_prev * pf.zd.y, pf.y);
                            } else {
                                cf = res_coef(a, R, fx.stg_r[warp][m][lane]);
                            }
                            g += x * cf.x;
                            h += (x * x) * cf.y;
                        }
                        pr0 = p0 + 32;
                    }
#pragma unroll 4
                    for (int64_t p = pr0 + lane; p < p1; p += 32) {
                        const int32_t i = __ldg(&a.row_idx[p]);
                        const double x = (double)__ldg(&a.val[p]);
                        const double2 cf = res_coef(a, R, i);
                        g += x * cf.x;
                        h += (x * x) * cf.y;
                    }
                    gs = warp_sum(g);
                    hs = warp_sum(h);
                }
                const double wj = stg ? fx.stg_w[warp][m] : ldcg(&a.w[j]);
                Dir r = finish_feature(a, gs, hs, wj);
                if (a.scdn && r.d != 0.0)   // SCDN: the feature's own 1-D step replaces d_j (Z27)
                    r.d *= res_scdn_alpha(a, R, p0, p1, stg ? fx.stg_r[warp][m] : nullptr,
                                          stg ? fx.stg_x[warp][m] : nullptr, r.d, wj, r.delta, lane);
                if (lane == 0) {
                    if (m >= R_CPW || a.d_out || len == a.s) {
                        a.dk[kk - k0] = r.d;
                        a.deltak[kk - k0] = r.delta;
                        if (len == a.s) fx.spilled = 1;   // read by other CTAs: fence before the counts
                    }
                    if (a.g_out) {
                        a.g_out[kk - k0] = r.g;
                        a.h_out[kk - k0] = r.h;
                    }
                    if (a.d_out) a.d_out[kk - k0] = r.d;
                    if (m < R_CPW) {
                        fx.colf[R.cb][slot] = 1;
                        fx.colj[R.cb][slot] = j;
                        fx.colw[R.cb][slot] = wj;
                        fx.cold[R.cb][slot] = r.d;
                        fx.coldl[R.cb][slot] = r.delta;
                    }
                }
                if (r.d != 0.0 && len != a.s) {   // full columns are folded from CSC (dense_dx)
                    if (stg) {
                        const bool ok = lane < len;
                        res_emit_warp(a, R, ok, fx.stg_r[warp][m][lane], (int32_t)(kk - k0),
                                      ok ? r.d * (double)fx.stg_x[warp][m][lane] : 0.0, lane);
                        res_col_scatter(a, R, p0 + 32, p1, lane, (int32_t)(kk - k0), r.d);
                    } else {
                        res_col_scatter(a, R, p0, p1, lane, (int32_t)(kk - k0), r.d);
                    }
                }
            }
        }

        pf.ok = false;   // consumed (re-gathered by this step's first window for the next step)
        RTL(R, 1);
        PROF_MARK(8);
        // ---------------- phase A': heavy columns, nnz-balanced over all warps -----------
        const HeavyPlan hpl = fx.plan[t & 1];   // computed a step ahead (see the count exchange)
        const int64_t e_lo = hpl.e_lo, e_hi = hpl.e_hi;
        if (a.scdn && e_hi > e_lo && tid == 0) atomicMax(a.status, 7);   // SCDN needs warp-owned columns
        if (e_hi > e_lo) {
            const int64_t hb0 = hpl.hb0, NH = hpl.NH;
            const int64_t lo_c = (int64_t)c * NH / G, hi_c = (int64_t)(c + 1) * NH / G;
            if (tid == 0) fx.cross_e[0] = fx.cross_e[1] = -1;
            PROF_MARK(9);
            const int64_t ce0 = hpl.ce0, ce1 = hpl.ce1;
            const int64_t a_w = lo_c + (int64_t)warp * (hi_c - lo_c) / NW;
            const int64_t b_w = lo_c + (int64_t)(warp + 1) * (hi_c - lo_c) / NW;
            for (int64_t rb = ce0; rb < ce1; rb += NE_MAX) {
                const int ne = (int)min((int64_t)NE_MAX, ce1 - rb);
                // entry offsets and descriptors (position, j, col_ptr[j]) and w_j, one round trip
                for (int i = tid; i <= ne; i += NT) {
                    fx.hst[i] = __ldg(&a.hstart[rb + i]) - hb0;
                    if (i < ne) {
                        const int4 hd = __ldg(&a.hdesc[rb + i]);
                        fx.hkk[i] = hd.x;
                        fx.hj[i] = hd.y;
                        fx.hcs[i] = colinfo_p0(hd);
                        fx.hw[i] = ldcg(&a.w[hd.y]);
                    }
                }
                for (int i = tid; i < ne * NW; i += NT) {
                    fx.hg[i / NW][i % NW] = 0.0;
                    fx.hh[i / NW][i % NW] = 0.0;
                }
                __syncthreads();
                for (int le = 0; le < ne; le++) {
                    const int64_t st = fx.hst[le], en = fx.hst[le + 1];
                    if (en <= a_w) continue;
                    if (st >= b_w) break;
                    const int64_t s0 = max(a_w, st), s1 = min(b_w, en);
                    const int64_t cs = fx.hcs[le];
                    double gs, hs;
                    res_col_gh(a, R, cs + (s0 - st), cs + (s1 - st), lane, gs, hs);
                    if (lane == 0) {
                        fx.hg[le][warp] = gs;
                        fx.hh[le][warp] = hs;
                    }
                }
                __syncthreads();
                for (int le = tid; le < ne; le += NT) {
                    double gs = 0.0, hs = 0.0;
                    for (int w2 = 0; w2 < NW; w2++) {
                        gs += fx.hg[le][w2];
                        hs += fx.hh[le][w2];
                    }
                    const int64_t st = fx.hst[le], en = fx.hst[le + 1];
                    const int64_t e = rb + le;
                    if (st >= lo_c && en <= hi_c) {
                        const int32_t kk = fx.hkk[le];
                        const Dir r = finish_feature(a, gs, hs, fx.hw[le]);
                        fx.hd[le] = r.d;
                        a.dk[kk - k0] = r.d;
                        a.deltak[kk - k0] = r.delta;
                        if (a.g_out) {
                            a.g_out[kk - k0] = r.g;
                            a.h_out[kk - k0] = r.h;
                        }
                        if (a.d_out) a.d_out[kk - k0] = r.d;
                    } else {
                        const int slot = st < lo_c ? 0 : 1;
                        HPart hp;
                        hp.e = e;
                        hp.g = gs;
                        hp.h = hs;
                        hp.pad = 0.0;
                        fx.hpo[slot] = hp;
                        fx.cross_e[slot] = e;
                        fx.cross_st[slot] = st;
                        fx.cross_en[slot] = en;
                        fx.cross_kk[slot] = fx.hkk[le];
                        fx.cross_cs[slot] = fx.hcs[le];
                        fx.cross_w[slot] = fx.hw[le];
                        fx.hd[le] = 0.0;
                    }
                }
                __syncthreads();
                for (int le = 0; le < ne; le++) {
                    const int64_t st = fx.hst[le], en = fx.hst[le + 1];
                    if (en <= a_w) continue;
                    if (st >= b_w) break;
                    if (!(st >= lo_c && en <= hi_c)) continue;
                    const double d = fx.hd[le];
                    if (d == 0.0 || en - st == a.s) continue;   // full columns: dense_dx
                    const int64_t s0 = max(a_w, st), s1 = min(b_w, en);
                    const int64_t cs = fx.hcs[le];
                    res_col_scatter(a, R, cs + (s0 - st), cs + (s1 - st), lane, fx.hkk[le] - (int32_t)k0, d);
                }
                __syncthreads();
            }
            PROF_MARK(10);
            // the crossing partials live in shared memory: a relaxed cluster barrier after a
            // shared-memory-only release fence (no GPU-scope drain) makes them readable
            fence_smem_release_cluster();
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
            PROF_MARK(11);
            if (warp < 2) {   // one warp per crossing column, lanes over the CTA partials
                const int64_t e = fx.cross_e[warp];
                if (lane == 0) fx.cross_d[warp] = 0.0;
                if (e >= 0) {
                    const int64_t st = fx.cross_st[warp], en = fx.cross_en[warp];
                    const int clo = cta_of(st, NH, G), chi = cta_of(en - 1, NH, G);
                    double gs = 0.0, hs = 0.0;
                    for (int c2 = clo + lane; c2 <= chi; c2 += 32) {
                        if ((int64_t)c2 * NH / G == (int64_t)(c2 + 1) * NH / G) continue;  // empty range
                        const HPart hp = *remote(&fx.hpo[c2 == clo ? 1 : 0], c2);
                        if (hp.e != e) atomicMax(a.status, 4);  // internal consistency check
                        gs += hp.g;
                        hs += hp.h;
                    }
                    gs = warp_sum(gs);
                    hs = warp_sum(hs);
                    if (lane == 0) {
                        const int32_t kk = fx.cross_kk[warp];
                        const Dir r = finish_feature(a, gs, hs, fx.cross_w[warp]);
                        fx.cross_d[warp] = r.d;
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
                const int64_t e = fx.cross_e[sl];
                if (e < 0 || (sl == 1 && e == fx.cross_e[0])) continue;
                const double d = fx.cross_d[sl];
                if (d == 0.0) continue;
                const int64_t st = fx.cross_st[sl], en = fx.cross_en[sl];
                if (en <= a_w || st >= b_w || en - st == a.s) continue;
                const int64_t s0 = max(a_w, st), s1 = min(b_w, en);
                const int64_t cs = fx.cross_cs[sl];
                res_col_scatter(a, R, cs + (s0 - st), cs + (s1 - st), lane, fx.cross_kk[sl] - (int32_t)k0, d);
            }
        }
        // ---------------- record counts to every owner (st.async, M0) ----------------------
        RTL(R, 2);
        __syncthreads();   // every warp's records are sent and the counters are final
        if (tid < G) {
            // HBM data other CTAs read in this step (overflow records, heavy-column results,
            // dk/deltak of positions beyond R_CPW) is made visible before the count signal
            if (fx.spilled || e_hi > e_lo || Pt > GN * R_CPW) __threadfence();
            st_async_u32(mapa_u32(s_addr(&fx.recvcnt[c]), tid), (uint32_t)fx.sendcnt[tid], mapa_u32(mb0, tid));
            fx.sendcnt[tid] = 0;
        }
        __syncwarp();   // warp 0 (tid < G <= 16) has read fx.spilled before tid 0 resets it below
        if (tid == 0) mbar_arrive_tx(mb0, (uint32_t)(4 * G));
        // while the counts travel: the next step's heavy plan (one warp) and every warp's next
        // own light columns (descriptor, w_j, first 32 nonzeros) into shared memory
        if (k1 < a.ntot && warp == NW - 1) heavy_plan_warp(a, k1, kn1, c, G, lane, &fx.plan[(t + 1) & 1]);
        PROF_MARK(0);
        RTL(R, 3);
        mbar_wait(mb0, ph & 1u);
        RTL(R, 4);
        ph ^= 1u;
        PROF_MARK(1);
        // lazy commit of the previous step to its touched owned samples (every producer has
        // finished its gathers): z += alpha_prev dx, coef, dx = 0 -- while the records travel
        {
            const int pb = R.cb ^ 1;
            const uint16_t *tlp = R.tls + (size_t)pb * R.Bs;
            const int np = fx.ntl[pb];
            for (int e = tid; e < np; e += NT) {
                const int li = tlp[e];
                const double2 zd = R.zd[li];
                if (zd.y == 0.0) continue;
                const double zn = zd.x + R.alpha_prev * zd.y;
                R.zd[li] = make_double2(zn, 0.0);
                R.coef[li] = coef_next(a.loss, R.coef[li], zn, R.alpha_prev * zd.y, res_y(R, li));
            }
        }

        // ---------------- phase C1: lazy commit of the previous step, link the records --------
        RTL(R, 5);
        int n_ovf;
        {
            const int ex = lane < G ? max(0, (int)fx.recvcnt[lane] - R.capP) : 0;
            n_ovf = __reduce_add_sync(0xffffffffu, ex);
            const int nin = lane < G ? min((int)fx.recvcnt[lane], R.capP) : 0;
            const int tot_in = __reduce_add_sync(0xffffffffu, nin);
            if (tid == 0) mbar_arrive_tx(mb1, (uint32_t)(16 * tot_in));
        }
        // (no CTA barrier here: the lazy commit touches zd/coef, the links below touch head/recin;
        // the fold reads zd only after the compaction barrier)
        if (tid == 0) fx.spilled = 0;
        mbar_wait(mb1, (ph >> 1) & 1u);
        RTL(R, 6);
        ph ^= 2u;
        if (warp < G) {   // warp p links the records of producer region p
            const int np = min((int)fx.recvcnt[warp], R.capP);
            for (int r = lane; r < np; r += 32) {
                const int phys = warp * R.capP + r;
                const int li = R.recin[phys].li;
                const int old = atomicExch(&R.head[li], phys);
                R.recin[phys].li = old;
                if (old < 0) atomicOr(&fx.tb[li >> 5], 1u << (li & 31));   // first record: touched
            }
        }
        for (int o = tid; o < n_ovf; o += NT) {
            int32_t *lip = reinterpret_cast<int32_t *>(&a.rec[R.my_ovf + o]);
            const int li = __ldcg(lip);
            const int old = atomicExch(&R.head[li], R.cap + o);
            __stcg(lip, old);
            if (old < 0) atomicOr(&fx.tb[li >> 5], 1u << (li & 31));
        }
        if (tid == 0 && n_ovf) {
            a.ovf_cnt[c] = 0;
            __threadfence();   // the reset is visible before this CTA's partial row is sent
        }
        // the step's full columns (dense_dx): staged, and whether they touch every sample
        DenseInfo di;
        di.f_lo = hpl.f_lo;   // from the plan computed a step ahead
        di.nf = hpl.nf;
        di.any = false;
        {
            int any = 0;
            for (int64_t e = tid; e < di.nf; e += NT) {
                const int32_t kk = __ldg(&a.flist[di.f_lo + e]);
                const double d = ldcg(&a.dk[kk - k0]);
                if (e < FMAX) {
                    fx.fd[e] = d;
                    fx.fcp[e] = __ldg(&a.col_ptr[__ldg(&a.order[kk])]);
                }
                any |= d != 0.0;
            }
            di.any = __syncthreads_or(any) != 0;
        }
        RTL(R, 14);
        // the step's touched owned samples, ascending (a fixed thread assignment for the fold and
        // the line search): every owned sample when a full column moved, else the bitmap compacted
        // by a CTA-wide scan
        {
            uint16_t *tlc = R.tls + (size_t)R.cb * R.Bs;
            const int nwords = (R.Bsc + 31) >> 5;
            if (di.any) {
                for (int e = tid; e < R.Bsc; e += NT) tlc[e] = (uint16_t)e;
                for (int w = tid; w < nwords; w += NT) fx.tb[w] = 0u;
                if (tid == 0) fx.ntl[R.cb] = R.Bsc;
            } else {   // one bitmap word per thread (nwords <= R_TBW = NT): a CTA-wide scan
                const uint32_t m0 = tid < nwords ? fx.tb[tid] : 0u;
                const int cnt = __popc(m0);
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                if (lane == 31) fx.scan_w[warp] = (unsigned long long)incl;
                __syncthreads();
                const int sw = lane < NW ? (int)fx.scan_w[lane] : 0;
                const int off = __reduce_add_sync(0xffffffffu, lane < warp ? sw : 0);
                int pos = off + incl - cnt;
                uint32_t m = m0;
                while (m) {
                    const int b = __ffs(m) - 1;
                    m &= m - 1;
                    tlc[pos++] = (uint16_t)(tid * 32 + b);
                }
                if (tid < nwords) fx.tb[tid] = 0u;
                const int tot = __reduce_add_sync(0xffffffffu, sw);
                if (tid == 0) fx.ntl[R.cb] = tot;
            }
            RTL(R, 15);
            __syncthreads();
        }
        PROF_MARK(2);
        RTL(R, 7);

        // ---------------- phase C2+C3: fold d'x_i (a3) and the Armijo windows (a4) ----------
        WinState ws;
        ws.q0 = 0;
        ws.nq = prev_q <= 1 ? 2 : QW;
        ws.qacc = -1;
        ws.bad = 0;
        ws.win = 0;
        while (true) {
            if (ws.nq <= 2) res_window<2>(a, R, ws, k0, k1, tid, lane, warp, pr, wcount, di, k1, kn1, pf);
            else res_window<QW>(a, R, ws, k0, k1, tid, lane, warp, pr, wcount, di, k1, kn1, pf);
            wcount++;
            if (ws.qacc >= 0 || ws.bad) break;
            ws.q0 += ws.nq;
            if (ws.q0 > a.qmax) break;
            ws.nq = QW;
        }
        int qacc = ws.qacc;
        const bool bad = ws.bad != 0;
        if (qacc > a.qmax) qacc = -1;
        const double alpha_acc = qacc < 0 ? 0.0 : ws.alpha;
        prev_q = qacc < 0 ? QW : qacc;
        R.alpha_prev = alpha_acc;   // z/coef of the touched samples: committed lazily

        // ---------------- commit (a5): w_B, F ---------------------------------------------
        if (qacc >= 0) {
            for (int s2 = tid;; s2 += NT) {
                const int m = s2 / NW, wq = s2 - m * NW;
                const int64_t kk = k0 + (int64_t)c * NW + wq + (int64_t)m * GN;
                if (kk >= k1) break;
                if (m < R_CPW && fx.colf[R.cb][s2]) {
                    a.w[fx.colj[R.cb][s2]] = fx.colw[R.cb][s2] + alpha_acc * fx.cold[R.cb][s2];
                } else {
                    const int32_t j = __ldg(&a.order[kk]);
                    a.w[j] = ldcg(&a.w[j]) + alpha_acc * ldcg(&a.dk[kk - k0]);
                }
            }
        }
        if (tid == 0) {
            fx.nlong = 0;
            fx.stage_n = 0;
        }
        if (c == 0 && tid == 0) {
            double F = fx.F;
            if (qacc >= 0) F = F + ws.lhs;
            fx.F = F;
            if (bad || t == a.nsteps - 1) {   // the maintained F and the last step's info
                *a.F = F;
                if (bad) atomicMax(a.status, 3);
                a.info[0] = (double)qacc;
                a.info[1] = alpha_acc;
                a.info[2] = ws.Delta;
                a.info[3] = ws.lhs;
                a.info[4] = ws.rhs;
                a.info[5] = F;
                a.info[7] = ws.nT_tot;
            }
            const int64_t gstep = a.trace_off + t;
            if (gstep < a.trace_cap) {
                if (a.q_trace) a.q_trace[gstep] = qacc;
                if (a.F_trace) a.F_trace[gstep] = F;
            }
            fx.cnt[0] += 1;
            fx.cnt[1] += qacc < 0 ? 1 : 0;
            fx.cnt[2] += (int64_t)ws.nT_tot;
            fx.cnt[3] += Pt;
        }
        PROF_MARK(6);
        RTL(R, 13);
        if (bad) break;
    }
    // ---------------- epilogue: last lazy commit, owned per-sample state back to HBM -------
    res_lazy_commit(a, R, tid);
    __syncthreads();
    for (int li = tid; li < R.Bsc; li += NT) {
        const int64_t i = (int64_t)li * G + c;
        a.z[i] = R.zd[li].x;
        a.coef[i] = R.coef[li];
    }
    if (c == 0 && tid == 0) {
        a.counters[0] += fx.cnt[0];
        a.counters[1] += fx.cnt[1];
        a.counters[3] += fx.cnt[2];
        a.counters[4] += fx.cnt[3];
    }
    if (prof)
        for (int i = 0; i < 16; i++) a.prof[i] += fx.pacc[i];
#undef PROF_MARK
    cluster_sync_all();   // no CTA exits while another may still read its shared memory
}

// the instantiation for a context's loss and solver
inline const void *res_kernel(int loss, bool scdn)
{
    if (scdn)
        return loss == LOSS_LOGISTIC ? (const void *)k_step_res<LOSS_LOGISTIC, true>
               : loss == LOSS_L2SVM  ? (const void *)k_step_res<LOSS_L2SVM, true>
                                     : (const void *)k_step_res<LOSS_SQ, true>;
    return loss == LOSS_LOGISTIC ? (const void *)k_step_res<LOSS_LOGISTIC, false>
           : loss == LOSS_L2SVM  ? (const void *)k_step_res<LOSS_L2SVM, false>
                                 : (const void *)k_step_res<LOSS_SQ, false>;
}

}  // namespace pcdn
