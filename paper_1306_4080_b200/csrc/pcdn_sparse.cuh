// pcdn_sparse.cuh -- the HBM-state bundle-step kernel for large sparse problems (launch modes 1-2;
// config 5, kdda-shaped: s = 2*10^6 samples, n = 2*10^7 features, P = 4096).
//
// One persistent launch runs every bundle step of an outer iteration (Alg.3 l.5-11, PAPER.md:
// 168-178).  The per-sample state (z_i, the cached factors (G_i, H_i)) lives in HBM/L2.  Per step:
//
//   A   g_j, h_j (Eq.13; App. A.2), d_j (Eq.5)
//       and the Delta terms (Eq.7) for every bundle column, then one record d_j x_ij per nonzero of
//       a column with d_j != 0 (Alg.4 l.1): stored at the CSR offset of (i, j) --
//       a fixed slot, so no returning atomic and no per-sample record list -- plus a bit in the
//       written-slot bitmap and a bit in the touched-sample bitmap (fire-and-forget reductions).
//         short columns (<= SP_SHORT nonzeros): one lane, in row order;
//         medium columns (<= heavy_len): one warp;
//         heavy columns: nch chunks over nch warps; each publishes its partial (g, h) and bumps
//         the column's arrival counter, the last to arrive sums the partials in chunk order,
//         finishes the column and publishes d_j with the step's stamp; the chunk warps then wait
//         for it and scatter their records.  No grid barrier inside phase A.
//   [grid barrier]
//   C   row-block owners: the touched set T (bitmap, ascending), d'x_i = the sum of the sample's
//       written slots in CSR (ascending column) order -- a fixed order, no sort, no float atomics
//       -- then the loss changes of a window of Armijo candidates (Eq.12), the L1 term and Delta
//       over the CTA's bundle share -> one partial row
//   [grid barrier]
//   D   every CTA sums the partial rows in the same fixed order and takes the same decision
//       (Eq.6, first passing q, further windows, q_max -> null step, reading Z10), commits its
//       samples (z, factors) and its bundle share of w, clears its bitmaps
//   [grid barrier]
//
// Summation orders differ from the oracle's (reading Z21: any fixed order); decisions and T are
// compared bit-exact, floats with the condition-aware 1e-9 bar.
#pragma once
#include "pcdn_kernels.cuh"

namespace pcdn {

// L2 eviction priorities of this kernel's accesses (PTX .L2::cache_hint with a createpolicy
// policy).  PCDN_L2_STREAM: the once-per-outer-iteration streams (CSC row indices, values, CSR
// slots) and the records (dead after the fold); PCDN_L2_STATE: the per-sample state gathered at
// random every step (z, the cached factors, row pointers, bitmaps, d'x).  0 = plain accesses,
// 1 = evict_first, 2 = evict_last, 3 = evict_normal.  Config 5 (LR, P = 4096 / 10^5 / 10^6, one
// outer iteration; profiles/r2c/l2a_*, l2b_*): plain 21.47 / 86.2 / 506 us per step, streams
// evict_first 21.11 / 83.7, state evict_last 20.88 / 83.6, both 20.65 / 80.6 / 495 us; records
// evict_normal with both 20.86 / 82.8.
#ifndef PCDN_L2_STREAM
#define PCDN_L2_STREAM 1
#endif
#ifndef PCDN_L2_STATE
#define PCDN_L2_STATE 2
#endif
#ifndef PCDN_L2_REC
#define PCDN_L2_REC PCDN_L2_STREAM
#endif
template <int K>
__device__ __forceinline__ uint64_t l2pol()
{
    uint64_t p = 0;
    if (K == 1) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    if (K == 2) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    if (K == 3) asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// read-only streams (non-coherent path)
template <int K>
__device__ __forceinline__ int32_t ldro(const int32_t *p)
{
    if (K == 0) return __ldg(p);
    int32_t v;
    asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2pol<K>()));
    return v;
}
template <int K>
__device__ __forceinline__ uint32_t ldro(const uint32_t *p)
{
    if (K == 0) return __ldg(p);
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2pol<K>()));
    return v;
}
template <int K>
__device__ __forceinline__ float ldro(const float *p)
{
    if (K == 0) return __ldg(p);
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(l2pol<K>()));
    return v;
}
template <int K>
__device__ __forceinline__ int64_t ldro(const int64_t *p)
{
    if (K == 0) return __ldg((const long long *)p);
    int64_t v;
    asm("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(l2pol<K>()));
    return v;
}
// mutable state (L2-coherent .cg loads; volatile: never merged or moved across the kernel's barriers)
template <int K>
__device__ __forceinline__ double ldst(const double *p)
{
    if (K == 0) return __ldcg(p);
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2pol<K>()));
    return v;
}
template <int K>
__device__ __forceinline__ double2 ldst(const double2 *p)
{
    if (K == 0) return __ldcg(p);
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(l2pol<K>()));
    return v;
}
template <int K>
__device__ __forceinline__ uint32_t ldst(const uint32_t *p)
{
    if (K == 0) return __ldcg(p);
    uint32_t v;
    asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2pol<K>()));
    return v;
}
template <int K>
__device__ __forceinline__ void stst(double *p, double v)
{
    if (K == 0) { *p = v; return; }
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(l2pol<K>()) : "memory");
}
template <int K>
__device__ __forceinline__ void stst(double2 *p, double2 v)
{
    if (K == 0) { *p = v; return; }
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(l2pol<K>()) : "memory");
}
template <int K>
__device__ __forceinline__ void stcg_rec(double *p, double v)
{
    if (K == 0) { __stcg(p, v); return; }
    asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(l2pol<K>()) : "memory");
}
template <int K>
__device__ __forceinline__ void red_or(uint32_t *p, uint32_t v)
{
    if (K == 0) { atomicOr(p, v); return; }
    asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(l2pol<K>()) : "memory");
}
constexpr int SK = PCDN_L2_STREAM, TK = PCDN_L2_STATE, RK = PCDN_L2_REC;
// L2 prefetch (evict_last) of the next step's column descriptors and bundle positions after the
// first barrier (1 = on).  Config 5 LR (profiles/r2c/l2pf_*): P = 4096 20.65 -> 20.54 us per step,
// P = 10^5 80.5 -> 80.8; prefetching each light lane's next column rows / slots / values / w_j as
// well (between the decision barrier's arrive and wait) measured 20.77 / 82.0.
#ifndef PCDN_SP_L2PF
#define PCDN_SP_L2PF 1
#endif
// the window's decision taken by every thread from the totals (1) or by one thread and broadcast
// through shared memory behind two more CTA barriers (0).  Config 5 LR P = 4096
// (profiles/r2c/ab_c1/b_*): 20.55 -> 20.36 us per step.  (Deferring the line-search share's w_j
// load and the next step's plan to after the touched-set scan measured 20.63.)
#ifndef PCDN_SP_DECALL
#define PCDN_SP_DECALL 1
#endif
__device__ __forceinline__ void pf_l2_last(const void *p) { asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p)); }


// Profiling instrumentation (phase cycles of CTA 0 for pcdn_set_profile(ctx, 1); per-CTA phase
// sums for mode 2) is compiled in only with -DPCDN_PROFILE=1 (pcdn_kernels.cuh): even as untaken
// branches it cost the production kernel registers and ~5 us per config-5 step.

// CTA shape of the sparse kernel: 384 threads per SM (one CTA per SM) leave each thread up to 168
// registers -- at 512 threads the kernel's live state spilled (config 5: 25.7 us per step at 512,
// 25.5 at 256, 25.2 at 384)
#ifndef PCDN_SNT
#define PCDN_SNT 384
#endif
constexpr int SNT = PCDN_SNT;
constexpr int SNW = SNT / 32;

constexpr int SP_SHORT = 4;     // columns with <= SP_SHORT nonzeros are reduced by one lane
constexpr int SP_CH = 256;      // default heavy_len of the sparse kernel: longer columns go in chunks
constexpr int SP_FOLD = 4;      // record loads of one sample in flight together in the fold
constexpr int SP_CB = 4;        // samples / positions of a thread with their loads in flight together (commit)
constexpr int SP_MQ = 256;      // per-CTA queue of a step's medium columns (one warp each, after the lane sweep)
constexpr int SP_GT_ROWS = 160; // grids up to this many CTAs read every partial row in one batch of loads
static_assert(SP_CTA_MUL == SNW, "a heavy chunk is one warp-register range (32 * SP_WR) per warp of the CTA");

struct SpPlan {
    int64_t c0, c1;     // the step's chunks [c0, c1) of cdesc
    int64_t f_lo, nf;   // the step's full columns: entries [f_lo, f_lo + nf) of flist
};

struct SpSmem {
    SpPlan plan[2];   // this and the next step (by step parity), computed a step ahead
    double red[SNW][32];
    double tot[32];
    int64_t scan_w[SNW];
    int64_t nT;
    double F;
    long long cnt[4];
    long long pacc[16];
    long long cprof[16];   // profiling mode 2: this CTA's sums, copied out at the end of the launch
    int dec_q, dec_bad, dec_nospec;
    double dec_alpha, dec_lhs, dec_rhs, dec_Delta, dec_nT;
    int nmq;               // medium columns of this CTA in this step, queued by the lane sweep
    int4 mq[SP_MQ];        // their column descriptors ...
    int32_t mqk[SP_MQ];    // ... and bundle positions (relative to the step)
    double fd[FMAX];
    int64_t fcp[FMAX];
    double dxd[TSM];
    int64_t row_base;
    int32_t tl[TSM];
    double pv[SP_GT_ROWS * 16];   // the partial rows of every CTA (sp_grid_totals), up to SP_GT_ROWS CTAs
};

__device__ __forceinline__ int atom_add_acq_rel(int *p, int v)
{
    int old;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// record d_j x_ij of nonzero (i, j) at CSR offset `slot` (a3)
__device__ __forceinline__ void sp_emit(const StepArgs &a, int32_t i, uint32_t slot, double v)
{
    PCDN_CHECK(i >= 0 && i < a.s);
    PCDN_CHECK(slot >= (uint32_t)__ldg(&a.row_ptr[i]) && slot < (uint32_t)__ldg(&a.row_ptr[i + 1]));
    stcg_rec<RK>(&a.rv[slot], v);
    red_or<TK>(&a.sbits[slot >> 5], 1u << (slot & 31));
    red_or<TK>(&a.bits[i >> 5], 1u << (i & 31));
}

__device__ __forceinline__ void sp_store_dir(const StepArgs &a, int64_t k, const Dir &r)
{
    a.dk[k] = r.d;
    a.deltak[k] = r.delta;
    if (a.g_out) {
        a.g_out[k] = r.g;
        a.h_out[k] = r.h;
    }
    if (a.d_out) a.d_out[k] = r.d;
}

// warp: g/h over nonzeros [p0, p1) then, for d != 0, the records (a column of <= heavy_len or a chunk)
__device__ __forceinline__ void sp_scatter(const StepArgs &a, int64_t p0, int64_t p1, int lane, double d)
{
    constexpr int B = 4;
    for (int64_t pb = p0 + lane; pb < p1; pb += 32 * B) {
        int32_t ri[B];
        uint32_t sl[B];
        float xv[B];
#pragma unroll
        for (int e = 0; e < B; e++) {
            const int64_t p = pb + 32 * e;
            ri[e] = -1;
            if (p < p1) {
                ri[e] = ldro<SK>(&a.row_idx[p]);
                sl[e] = ldro<SK>(&a.cslot[p]);
                xv[e] = ldro<SK>(&a.val[p]);
            }
        }
#pragma unroll
        for (int e = 0; e < B; e++)
            if (ri[e] >= 0) sp_emit(a, ri[e], sl[e], d * (double)xv[e]);
    }
}

// A warp's range [p0, p1) of at most SP_WR nonzeros per lane, held in registers from the gather to
// the scatter: load (row, slot, value), gather the factors, reduce (lane order, fixed xor tree).
constexpr int SP_WR = 8;
struct WarpRange {
    int32_t ri[SP_WR];
    uint32_t sl[SP_WR];
    float xv[SP_WR];
};
__device__ __forceinline__ void sp_range_gh(const StepArgs &a, int64_t p0, int64_t p1, int lane, WarpRange &r,
                                            double &gs, double &hs)
{
#pragma unroll
    for (int e = 0; e < SP_WR; e++) {
        const int64_t p = p0 + lane + 32 * e;
        r.ri[e] = -1;
        r.sl[e] = 0;
        r.xv[e] = 0.f;
        if (p < p1) {
            r.ri[e] = ldro<SK>(&a.row_idx[p]);
            r.sl[e] = ldro<SK>(&a.cslot[p]);
            r.xv[e] = ldro<SK>(&a.val[p]);
        }
    }
    double2 cf[SP_WR];
#pragma unroll
    for (int e = 0; e < SP_WR; e++) cf[e] = r.ri[e] >= 0 ? ldst<TK>(&a.coef[r.ri[e]]) : make_double2(0.0, 0.0);
    double g = 0.0, h = 0.0;
#pragma unroll
    for (int e = 0; e < SP_WR; e++) {
        if (r.ri[e] >= 0) {
            const double x = (double)r.xv[e];
            g += x * cf[e].x;
            h += (x * x) * cf[e].y;
        }
    }
    gs = warp_sum(g);
    hs = warp_sum(h);
}
__device__ __forceinline__ void sp_range_scatter(const StepArgs &a, const WarpRange &r, double d)
{
#pragma unroll
    for (int e = 0; e < SP_WR; e++)
        if (r.ri[e] >= 0) sp_emit(a, r.ri[e], r.sl[e], d * (double)r.xv[e]);
}

// A medium column (SP_SHORT < length <= heavy_len) by one warp: g/h (Eq.13), d_j (Eq.5), the Delta
// term, and its records; k = the column's bundle position within the step
__device__ __forceinline__ void sp_medium_column(const StepArgs &a, const int4 ci, int64_t k, int lane)
{
    const int ml = ci.y;
    const int64_t p0 = colinfo_p0(ci), p1 = p0 + ml;
    const double wj = ldcg(&a.w[ci.x]);
    double gs, hs;
    if (ml <= 32 * SP_WR) {   // held in registers from the gather to the scatter
        WarpRange wr;
        sp_range_gh(a, p0, p1, lane, wr, gs, hs);
        const Dir r = finish_feature(a, gs, hs, wj);
        if (lane == 0) sp_store_dir(a, k, r);
        if (r.d != 0.0 && ml != a.s) sp_range_scatter(a, wr, r.d);
    } else {
        col_gh(a, p0, p1, lane, gs, hs);
        const Dir r = finish_feature(a, gs, hs, wj);
        if (lane == 0) sp_store_dir(a, k, r);
        if (r.d != 0.0 && ml != a.s) sp_scatter(a, p0, p1, lane, r.d);
    }
}

// fold of sample i's records: the written slots of its CSR segment [r0, r1), ascending.  The first
// three words of the segment's written-slot bitmap are loaded together (a row of <= 65 nonzeros
// needs no more), then up to SP_FOLD slots of a word at a time (static register indices), summed
// in slot order.
__device__ __forceinline__ double sp_fold_word(const StepArgs &a, int64_t wd, uint32_t m)
{
    PCDN_CHECK(wd >= 0 && wd <= (int64_t)(a.row_ptr[a.s] >> 5));
    double dx = 0.0;
    while (m) {
        uint32_t sl[SP_FOLD];
#pragma unroll
        for (int r = 0; r < SP_FOLD; r++) {
            sl[r] = m ? (uint32_t)(wd * 32 + __ffs(m) - 1) : 0xffffffffu;
            m &= m - 1;
        }
        double v[SP_FOLD];
#pragma unroll
        for (int r = 0; r < SP_FOLD; r++) v[r] = sl[r] != 0xffffffffu ? ldst<RK>(&a.rv[sl[r]]) : 0.0;
#pragma unroll
        for (int r = 0; r < SP_FOLD; r++)
            if (sl[r] != 0xffffffffu) dx += v[r];
    }
    return dx;
}
__device__ __forceinline__ uint32_t sp_word_mask(int64_t wd, int64_t r0, int64_t r1)
{
    uint32_t m = 0xffffffffu;
    if (wd == (r0 >> 5)) m &= 0xffffffffu << (r0 & 31);
    if (wd == ((r1 - 1) >> 5)) m &= 0xffffffffu >> (31 - ((r1 - 1) & 31));
    return m;
}
// Clear sample i's written-slot bits (its CSR segment [r0, r1)) before the decision's barrier (the
// speculative commit): a word shared with a neighbouring sample's segment -- which another thread,
// or another CTA at a block boundary, may not have folded yet -- loses only this sample's bits.
// (Clearing whole words here lost a neighbour's records whenever its fold ran later.)
__device__ __forceinline__ void sp_clear_own_slots(const StepArgs &a, int64_t r0, int64_t r1)
{
    if (r1 <= r0) return;
    for (int64_t wd = r0 >> 5; wd <= ((r1 - 1) >> 5); wd++) {
        const uint32_t m = sp_word_mask(wd, r0, r1);
        if (m == 0xffffffffu) a.sbits[wd] = 0u;
        else atomicAnd(&a.sbits[wd], ~m);
    }
}
__device__ __forceinline__ double sp_fold(const StepArgs &a, int64_t r0, int64_t r1)
{
    double dx = 0.0;
    if (r1 <= r0) return dx;
    const int64_t w0 = r0 >> 5, w1 = (r1 - 1) >> 5;
    uint32_t m3[3];
#pragma unroll
    for (int u = 0; u < 3; u++) m3[u] = w0 + u <= w1 ? ldst<TK>(&a.sbits[w0 + u]) & sp_word_mask(w0 + u, r0, r1) : 0u;
#pragma unroll
    for (int u = 0; u < 3; u++)
        if (m3[u]) dx += sp_fold_word(a, w0 + u, m3[u]);
    for (int64_t wd = w0 + 3; wd <= w1; wd++) {
        const uint32_t m = ldst<TK>(&a.sbits[wd]) & sp_word_mask(wd, r0, r1);
        if (m) dx += sp_fold_word(a, wd, m);
    }
    return dx;
}

// The full columns' d'x part of sample i in bundle order (a full column holds row i at offset i).
// Out of line (rare: a step with a full column); scalar arguments only, so that no copy of the
// kernel's StepArgs is made addressable.
__device__ __noinline__ double sp_dense_dx(const int32_t *__restrict__ flist, const double *dk,
                                          const int4 *__restrict__ colinfo, const float *__restrict__ val,
                                          const double *fd, const int64_t *fcp, int64_t f_lo, int64_t nf, int64_t k0,
                                          int64_t i)
{
    double dx = 0.0;
    for (int64_t e = 0; e < nf; e++) {
        double d;
        int64_t cp;
        if (e < FMAX) {
            d = fd[e];
            cp = fcp[e];
        } else {
            const int32_t kk = __ldg(&flist[f_lo + e]);
            d = ldcg(&dk[kk - k0]);
            cp = colinfo_p0(__ldg(&colinfo[kk]));
        }
        if (d != 0.0) dx += d * (double)__ldg(&val[cp + i]);
    }
    return dx;
}

// Totals of the G partial rows part[c2][0..W) in a fixed order, into tot[0..W) (valid for every
// thread after the call).  Up to SP_GT_ROWS CTAs: every thread loads its share of the G x W values
// in one batch (a single L2 round trip), then warp q sums slot q over the rows (lane-strided, a
// fixed xor tree).  Beyond: warp w sums rows w, w + SNW, ... and warp 0 the warp sums.  (Warp q
// loading slot q of every row itself, without the shared-memory staging and its CTA barrier,
// measured slower: config 5 LR P = 4096 20.37 -> 21.10 us per step, profiles/r2c/ab_gt.)
template <int W>
__device__ __forceinline__ void sp_grid_totals(const double *part, int G, double (*red)[32], double *tot, double *pv,
                                               int tid, int lane, int warp)
{
    if (G <= SP_GT_ROWS) {
        constexpr int K = (SP_GT_ROWS * W + SNT - 1) / SNT;   // values per thread
        double v[K];
#pragma unroll
        for (int e = 0; e < K; e++) {
            const int idx = tid + e * SNT;
            v[e] = idx < G * W ? ldcg(&part[(int64_t)(idx / W) * NPART + (idx % W)]) : 0.0;
        }
#pragma unroll
        for (int e = 0; e < K; e++) {
            const int idx = tid + e * SNT;
            if (idx < G * W) pv[idx] = v[e];
        }
        __syncthreads();
        for (int q = warp; q < W; q += SNW) {
            double x = 0.0;
            for (int r = lane; r < G; r += 32) x += pv[r * W + q];
            x = warp_sum(x);
            if (lane == 0) tot[q] = x;
        }
        __syncthreads();
        return;
    }
    double x = 0.0;
    if (lane < W) {
#pragma unroll 4
        for (int c2 = warp; c2 < G; c2 += SNW) x += ldcg(&part[(int64_t)c2 * NPART + lane]);
    }
    red[warp][lane] = x;
    __syncthreads();
    if (warp == 0 && lane < W) {
        double t = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < SNW; w2++) t += red[w2][lane];
        tot[lane] = t;
    }
    __syncthreads();
}


// One Armijo window over q0 .. q0+NQ-1 (Eq.6 with Eq.12 from retained quantities); window 0 also
// folds d'x_i.  Then the grid barrier and the decision taken identically by every CTA.
template <int NQ, int LOSS, class Sync>
__device__ __forceinline__ void sp_window(const StepArgs &a, SpSmem &sm, Sync &sy, WinState &ws, const int32_t *Tl,
                                          int64_t nT, int64_t k0, int64_t pb0, int64_t pb1, int G, int c, int tid,
                                          int lane, int warp, const ShareReg &sh, RowReg &rr, const DenseInfo &di,
                                          bool spec, double alpha_s, int64_t wb, int64_t we,
                                          bool prof, long long &tprev, long long *ctal, long long tstep)
{
    using LY = WinLayout<NQ>;
    constexpr int W = LY::W;
    double alpha0 = 1.0;
    for (int q = 0; q < ws.q0; q++) alpha0 *= a.beta;
    double acc[W];
#pragma unroll
    for (int q = 0; q < W; q++) acc[q] = 0.0;
    for (int64_t li = tid; li < nT; li += SNT) {
        const int32_t i = Tl[li];
        PCDN_CHECK(i >= 0 && i < a.s);
        // (the thread's first sample from registers after window 0: its z / G may already hold the
        // speculative commit)
        const bool rg = ws.win > 0 && li == tid;
        const double zi = rg ? rr.zi : ldst<TK>(&a.z[i]);
        const double cg = rg ? rr.cg : ldst<TK>(&a.coef[i]).x;
        const int yi = rg ? rr.yi : a.y[i];
        double dx;
        if (ws.win == 0) {
            const int64_t r0 = ldro<TK>(&a.row_ptr[i]), r1 = ldro<TK>(&a.row_ptr[i + 1]);
            dx = sp_fold(a, r0, r1);
            if (di.any) {   // full columns, from CSC in bundle order (then the records)
                const int64_t li2 = i - sm.row_base;
                dx = (nT <= TSM ? sm.dxd[li2] : sp_dense_dx(a.flist, a.dk, a.colinfo, a.val, sm.fd, sm.fcp, di.f_lo, di.nf, k0, i)) + dx;
            }
            stst<TK>(&a.dxg[i], dx);
            if (li == tid) {
                rr.i = i;
                rr.yi = yi;
                rr.zi = zi;
                rr.dx = dx;
                rr.has_dx = 1;
                rr.r0 = r0;
                rr.r1 = r1;
                rr.cg = cg;
            }
        } else {
            dx = li == tid ? rr.dx : ldst<TK>(&a.dxg[i]);
        }
        double al = alpha0;
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            acc[q] += loss_change(LOSS, zi, yi, cg, dx, al);
            al *= a.beta;
        }
    }
    // L1 part of Eq.12 and Delta over this CTA's share of the bundle (the thread's first position
    // from registers, the others in batches of SP_CB)
    if (sh.kk >= 0) {
        double al = alpha0;
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            acc[NQ + q] += fabs(sh.wj + al * sh.d) - fabs(sh.wj) + a.mu * al * sh.d * (sh.wj + 0.5 * al * sh.d);
            al *= a.beta;
        }
        acc[LY::DELTA] += sh.delta;
    }
    for (int64_t kb = pb0 + tid + SNT; kb < pb1; kb += (int64_t)SNT * SP_CB) {
        int32_t jj[SP_CB];
#pragma unroll
        for (int e = 0; e < SP_CB; e++) {
            const int64_t kk = kb + (int64_t)e * SNT;
            jj[e] = kk < pb1 ? __ldg(&a.order[kk]) : -1;
        }
        double wv[SP_CB], dv[SP_CB], tv[SP_CB];
#pragma unroll
        for (int e = 0; e < SP_CB; e++) {
            const int64_t kk = kb + (int64_t)e * SNT;
            wv[e] = dv[e] = tv[e] = 0.0;
            if (jj[e] >= 0) {
                wv[e] = ldcg(&a.w[jj[e]]);
                dv[e] = ldcg(&a.dk[kk - k0]);
                tv[e] = ldcg(&a.deltak[kk - k0]);
            }
        }
#pragma unroll
        for (int e = 0; e < SP_CB; e++) {
            if (jj[e] < 0) continue;
            double al = alpha0;
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                acc[NQ + q] += fabs(wv[e] + al * dv[e]) - fabs(wv[e]) + a.mu * al * dv[e] * (wv[e] + 0.5 * al * dv[e]);
                al *= a.beta;
            }
            acc[LY::DELTA] += tv[e];
        }
    }
    if (tid == 0) {
        acc[LY::NTOUCH] = (double)nT;
        acc[LY::NOSPEC] = spec ? 0.0 : 1.0;
    }
    // speculative commit (a5) with alpha_s = beta^{previous q}: this CTA's samples (one per thread,
    // in registers) and the clearing of its bitmaps, before the barrier -- the decision after it
    // confirms (no third barrier) or corrects it (the kernel redoes the commit from registers)
    if (spec && ws.win == 0) {
        if (rr.i >= 0) {
            const int32_t i = rr.i;
            const double zn = rr.zi + alpha_s * rr.dx;
            stst<TK>(&a.z[i], zn);
            stst<TK>(&a.coef[i], coef_next(LOSS, make_double2(rr.cg, 2.0), zn, alpha_s * rr.dx, rr.yi));
            sp_clear_own_slots(a, rr.r0, rr.r1);
        }
        for (int64_t wi = wb + tid; wi < we; wi += SNT) a.bits[wi] = 0u;
    }
    if (ctal && ws.win == 0) {   // profiling mode 2: this CTA's fold + line-search time
        __syncthreads();
        if (tid == 0) ctal[1] += clock64() - tstep;
    }
    constexpr int SPL = 32 / W;
    {
        const double tot = xreduce<W>(acc, lane);
        if ((lane % SPL) == 0) sm.red[warp][lane / SPL] = tot;
    }
    double *part = a.part + (int64_t)(ws.win & 1) * G * NPART;
    __syncthreads();
    if (warp == 0 && lane < W) {
        double s = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < SNW; w2++) s += sm.red[w2][lane];
        part[(int64_t)c * NPART + lane] = s;
    }
    if (prof) {
        const long long now = clock64();
        sm.pacc[3] += now - tprev;
        tprev = now;
    }
    sy.sync();
    if (prof) {
        const long long now = clock64();
        sm.pacc[4] += now - tprev;
        tprev = now;
    }
    sp_grid_totals<W>(part, G, sm.red, sm.tot, sm.pv, tid, lane, warp);
#if PCDN_SP_DECALL
    // every thread takes the decision itself from the totals (the same bits in every thread of
    // every CTA): no broadcast through shared memory and no further CTA barrier (sm.tot is next
    // written after the next window's first __syncthreads)
    {
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
        ws.qacc = qa;
        ws.bad = badl;
        ws.alpha = alpha_a;
        ws.lhs = la;
        ws.rhs = ra;
        ws.Delta = Dl;
        ws.nT_tot = sm.tot[LY::NTOUCH];
        ws.nospec = sm.tot[LY::NOSPEC] != 0.0;
        ws.win++;
    }
#else
    if (warp == 0 && lane == 0) {
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
        sm.dec_nospec = sm.tot[LY::NOSPEC] != 0.0;
    }
    __syncthreads();
    ws.qacc = sm.dec_q;
    ws.bad = sm.dec_bad;
    ws.alpha = sm.dec_alpha;
    ws.lhs = sm.dec_lhs;
    ws.rhs = sm.dec_rhs;
    ws.Delta = sm.dec_Delta;
    ws.nT_tot = sm.dec_nT;
    ws.nospec = sm.dec_nospec;
    ws.win++;
    __syncthreads();   // sm.dec_* / sm.red / sm.tot are reused by the next window
#endif
    if (prof) {
        const long long now = clock64();
        sm.pacc[5] += now - tprev;
        tprev = now;
    }
}

__device__ __forceinline__ void sp_plan(const StepArgs &a, int64_t k0, int64_t k1, SpPlan *out)
{
    SpPlan p;
    p.c0 = __ldg(&a.cpos[k0]);
    p.c1 = __ldg(&a.cpos[k1]);
    p.f_lo = __ldg(&a.fpos[k0]);
    p.nf = __ldg(&a.fpos[k1]) - p.f_lo;
    *out = p;
}

template <class Sync, int LOSS>
__global__ void __launch_bounds__(SNT, 1) k_step_sparse(StepArgs a)
{
    if (a.stop && ldcg(a.stop)) return;   // the solve already ended (queued ahead; grid-uniform)
    Sync sy(a.bar);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SpSmem &sm = *reinterpret_cast<SpSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t nwords = (a.s + 31) >> 5;
    const int64_t wb = (int64_t)c * nwords / G, we = (int64_t)(c + 1) * nwords / G;
    const int64_t row_base = wb * 32;
    if (tid == 0) sm.row_base = row_base;
    int prev_q = 0;
    int q_spec = 0;   // the speculative commit's q: the last accepted one (the dense kernel's rule)
    const int64_t pbs0 = (int64_t)c * a.P / G, pbs1 = (int64_t)(c + 1) * a.P / G;
    const int64_t gw = (int64_t)c * SNW + warp;

    long long tprev = 0;
    const bool prof = PCDN_PROFILE && a.prof != nullptr && c == 0 && tid == 0;
    if (tid < 16) sm.pacc[tid] = 0;
#define SP_MARK(i)                                \
    do {                                          \
        if (prof) {                               \
            const long long now_ = clock64();     \
            sm.pacc[i] += now_ - tprev;           \
            tprev = now_;                         \
        }                                         \
    } while (0)
    if (c == 0 && tid == 0) {
        sm.F = ldcg(a.F);
        for (int i = 0; i < 4; i++) sm.cnt[i] = 0;
    }
    long long *const ctal_out = (PCDN_PROFILE && a.tl && c < 256) ? a.tl + (int64_t)c * 16 : nullptr;   // profiling mode 2
    long long *const ctal = ctal_out ? sm.cprof : nullptr;   // per-CTA phase sums, in shared memory
    if (tid < 16) sm.cprof[tid] = 0;
    if (tid == 0) sm.nmq = 0;
    if (tid == 0 && a.nsteps > 0) sp_plan(a, 0, min(a.P, a.ntot), &sm.plan[0]);
    __syncthreads();
    long long tstep = 0;
    for (int64_t t = 0; t < a.nsteps; t++) {
        if (prof) tprev = clock64();
        if (ctal && tid == 0) tstep = clock64();
        const int64_t k0 = t * a.P;
        const int64_t k1 = min(k0 + a.P, a.ntot);
        const int64_t Pt = k1 - k0;
        const unsigned long long stamp = a.stamp0 + (unsigned long long)t + 1ull;
        const SpPlan pl = sm.plan[t & 1];

        // ---------------- phase A: short and medium columns (a1, a2, a3) ----------------------
        // The step's heavy-column chunks go to the top GH CTAs (one chunk per CTA at a time, all
        // 16 warps), the short and medium columns to the warps of the others.
        const int64_t C0 = pl.c0, NCH = pl.c1 - pl.c0;
        const int GH = NCH > 0 ? (int)max((int64_t)1, min((int64_t)(G / 2), NCH)) : 0;
        const int GL = max(1, G - GH);
        if (c < GL) {
            const int64_t NWL = (int64_t)GL * SNW;
            const int cw = (int)min((int64_t)32, max((int64_t)1, (Pt + NWL - 1) / NWL));
            for (int64_t ch = gw;; ch += NWL) {
                const int64_t kb = k0 + ch * cw;
                if (kb >= k1) break;
                const int64_t kk = kb + lane;
                // profiling mode 2, thread 0 of the CTA: cycles from the start of its lane column until
                // the descriptor, the rows / w_j, the gathered factors have arrived and the emits are
                // issued (slots 4-7, cumulative; slot 8 counts its lane columns).  The volatile
                // shared-memory write of a loaded value stalls until the load has returned.
                const long long tq0 = (ctal && tid == 0) ? clock64() : 0;
#define SP_PROBE(slot, dep)                                                       \
    do {                                                                          \
        if (ctal && tid == 0) {                                                   \
            *reinterpret_cast<volatile long long *>(&sm.cprof[15]) = (long long)(dep); \
            ctal[slot] += clock64() - tq0;                                        \
        }                                                                         \
    } while (0)
                const int4 ci = (lane < cw && kk < k1) ? __ldg(&a.colinfo[kk]) : make_int4(0, -1, 0, 0);
                const int len = ci.y;
                PCDN_CHECK(len < 0 || (ci.x >= 0 && ci.x < a.n && colinfo_p0(ci) + len <= a.col_ptr[a.n]));
                if (len >= 0 && len <= SP_SHORT && len <= a.heavy_len) {
                    const int32_t j = ci.x;
                    const int64_t p0 = colinfo_p0(ci);
                    int32_t ri[SP_SHORT];
                    uint32_t sl[SP_SHORT];
                    float xv[SP_SHORT];
#pragma unroll
                    for (int e = 0; e < SP_SHORT; e++) {
                        ri[e] = 0;
                        sl[e] = 0;
                        xv[e] = 0.f;
                        if (e < len) {
                            ri[e] = ldro<SK>(&a.row_idx[p0 + e]);
                            sl[e] = ldro<SK>(&a.cslot[p0 + e]);
                            xv[e] = ldro<SK>(&a.val[p0 + e]);
                        }
                    }
                    const double wj = ldcg(&a.w[j]);
                    SP_PROBE(4, len);
                    SP_PROBE(5, ri[0] + (long long)__float_as_int(xv[0]) + (long long)sl[0] + __double_as_longlong(wj));
                    double2 cf[SP_SHORT];
#pragma unroll
                    for (int e = 0; e < SP_SHORT; e++) cf[e] = e < len ? ldst<TK>(&a.coef[ri[e]]) : make_double2(0.0, 0.0);
                    SP_PROBE(6, __double_as_longlong(cf[0].x) + __double_as_longlong(cf[len > 1 ? 1 : 0].y));
                    double g = 0.0, h = 0.0;
#pragma unroll
                    for (int e = 0; e < SP_SHORT; e++) {
                        if (e < len) {
                            const double x = (double)xv[e];
                            g += x * cf[e].x;
                            h += (x * x) * cf[e].y;
                        }
                    }
                    const Dir r = finish_feature(a, g, h, wj);
                    sp_store_dir(a, kk - k0, r);
                    if (r.d != 0.0 && len != a.s) {   // full columns are folded from CSC (dense_dx)
#pragma unroll
                        for (int e = 0; e < SP_SHORT; e++)
                            if (e < len) sp_emit(a, ri[e], sl[e], r.d * (double)xv[e]);
                    }
                    SP_PROBE(7, __double_as_longlong(r.d));
                    if (ctal && tid == 0) ctal[8] += 1;
                }
#undef SP_PROBE
                // medium columns go to the CTA's queue (a warp each below), so that no warp reduces
                // two of them one after the other; beyond the queue the warp takes them itself
                unsigned med = __ballot_sync(0xffffffffu, len > SP_SHORT && len <= a.heavy_len);
                if (med) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&sm.nmq, __popc(med));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    const int slot = base + __popc(med & ((1u << lane) - 1u));
                    if (((med >> lane) & 1u) && slot < SP_MQ) {
                        sm.mq[slot] = ci;
                        sm.mqk[slot] = (int32_t)(kk - k0);
                    }
                    med &= __ballot_sync(0xffffffffu, ((med >> lane) & 1u) && slot >= SP_MQ);
                }
                while (med) {
                    const int src = __ffs(med) - 1;
                    med &= med - 1;
                    const int4 cm = make_int4(__shfl_sync(0xffffffffu, ci.x, src), __shfl_sync(0xffffffffu, ci.y, src),
                                              __shfl_sync(0xffffffffu, ci.z, src), __shfl_sync(0xffffffffu, ci.w, src));
                    sp_medium_column(a, cm, kb + src - k0, lane);
                }
            }
        }
        __syncthreads();
        if (ctal && tid == 0) ctal[9] += clock64() - tstep;   // profiling mode 2: lane sweep done (all warps)
        for (int q = warp; q < min(sm.nmq, SP_MQ); q += SNW) sp_medium_column(a, sm.mq[q], sm.mqk[q], lane);
        if (ctal) {   // profiling mode 2: medium columns done; the CTA's medium-column count
            __syncthreads();
            if (tid == 0) {
                ctal[10] += clock64() - tstep;
                ctal[12] += sm.nmq;
            }
        }
        SP_MARK(8);

        // ---------------- phase A, heavy columns: one chunk per CTA at a time (A1) ------------------
        // The CTA's warps split the chunk's nonzeros evenly, their partials are added in warp
        // order.  A one-chunk column is finished and scattered at once; a longer one publishes the
        // chunk's partial and bumps the column's arrival counter -- the last chunk to arrive sums
        // the partials in chunk order, finishes the column and publishes d_j with the step's stamp
        // (A2 below scatters the other chunks).  Every partial is published before any CTA waits,
        // so no wait can block a partial another column needs.
        const bool heavy_cta = c >= G - GH;
        if (heavy_cta) {
            for (int64_t q = G - 1 - c; q < NCH; q += GH) {
                const ChunkDesc cd = chunk_decode(__ldg(&a.cdesc[C0 + q]));
                PCDN_CHECK(cd.e >= 0 && cd.e < a.n && cd.c < cd.nch && cd.nch >= 1 && cd.nch <= SP_NCHMAX);
                PCDN_CHECK(cd.pb >= 0 && cd.len >= 1 && cd.pb + cd.len <= a.col_ptr[a.n]);
                const int64_t w0 = cd.pb + (int64_t)warp * cd.len / SNW, w1 = cd.pb + (int64_t)(warp + 1) * cd.len / SNW;
                // the column's position, feature and w_j, loaded beside the gather (warp 0 finishes)
                int4 hd = make_int4(0, 0, 0, 0);
                double wj = 0.0;
                if (warp == 0) {
                    hd = __ldg(&a.hdesc[cd.e]);   // (position, j, col_ptr[j])
                    wj = ldcg(&a.w[hd.y]);
                }
                const bool inreg = w1 - w0 <= 32 * SP_WR;   // this warp's share held in registers
                WarpRange wr;
                double gs, hs;
                if (inreg) sp_range_gh(a, w0, w1, lane, wr, gs, hs);
                else col_gh(a, w0, w1, lane, gs, hs);
                if (lane == 0) {
                    sm.red[warp][0] = gs;
                    sm.red[warp][1] = hs;
                }
                __syncthreads();
                if (warp == 0) {
                    double g = 0.0, h = 0.0;
#pragma unroll
                    for (int w2 = 0; w2 < SNW; w2++) {
                        g += sm.red[w2][0];
                        h += sm.red[w2][1];
                    }
                    int fin = cd.nch == 1;
                    if (!fin) {
                        if (lane == 0) {
                            __stcg(&a.cpart[q], make_double2(g, h));
                            const int old = atom_add_acq_rel(&a.ccnt[cd.e], 1);
                            PCDN_CHECK(old >= 0 && old < cd.nch);   // arrivals of this step only
                            fin = old == cd.nch - 1;
                        }
                        fin = __shfl_sync(0xffffffffu, fin, 0);
                        __syncwarp();
                        if (fin) {   // the last chunk: the column's partials in chunk order, a fixed tree
                            if (lane == 0) a.ccnt[cd.e] = 0;   // re-armed: the entry recurs only in a later launch
                            g = 0.0;
                            h = 0.0;
                            const int64_t qb = q - cd.c;
                            for (int u = lane; u < cd.nch; u += 32) {
                                const double2 v = __ldcg(&a.cpart[qb + u]);
                                g += v.x;
                                h += v.y;
                            }
                            g = warp_sum(g);
                            h = warp_sum(h);
                        }
                    }
                    if (fin) {
                        const Dir r = finish_feature(a, g, h, wj);
                        PCDN_CHECK(hd.x >= k0 && hd.x < k1);
                        if (lane == 0) {
                            sp_store_dir(a, hd.x - k0, r);
                            if (cd.nch > 1) {
                                __stcg(&a.dflag[cd.e].d, r.d);
                                st_release(&a.dflag[cd.e].stamp, stamp);
                            }
                            sm.tot[0] = r.d;
                        }
                    }
                }
                __syncthreads();
                if (cd.nch == 1) {
                    const double d = sm.tot[0];
                    if (d != 0.0 && !cd.full) {
                        if (inreg) sp_range_scatter(a, wr, d);
                        else sp_scatter(a, w0, w1, lane, d);
                    }
                }
                __syncthreads();   // sm.red / sm.tot reused by the next chunk
            }
        }
        SP_MARK(9);
        if (ctal) {   // profiling mode 2: heavy chunks reduced (A1)
            __syncthreads();
            if (tid == 0) ctal[11] += clock64() - tstep;
        }
        // ---------------- phase A, heavy columns: records once d_j is published (A2) --------------
        if (heavy_cta) {
            for (int64_t q = G - 1 - c; q < NCH; q += GH) {
                const ChunkDesc cd = chunk_decode(__ldg(&a.cdesc[C0 + q]));
                if (cd.nch == 1 || cd.full) continue;
                if (tid == 0) {
                    const long long t0 = clock64();
                    while (ld_acquire(&a.dflag[cd.e].stamp) != stamp) {
                        if (clock64() - t0 > 8000000000LL) __trap();   // a broken protocol: fail, do not hang
                        __nanosleep(32);
                    }
                    sm.tot[0] = __ldcg(&a.dflag[cd.e].d);
                }
                __syncthreads();
                const double d = sm.tot[0];
                const int64_t w0 = cd.pb + (int64_t)warp * cd.len / SNW, w1 = cd.pb + (int64_t)(warp + 1) * cd.len / SNW;
                if (d != 0.0) sp_scatter(a, w0, w1, lane, d);
                __syncthreads();
            }
        }
        SP_MARK(0);
        if (ctal) {   // profiling mode 2: this CTA's phase-A time (all its warps done)
            __syncthreads();
            if (tid == 0) ctal[0] += clock64() - tstep;
        }
        sy.sync();
        SP_MARK(1);
        if (tid == 0) sm.nmq = 0;   // every warp left the medium-column queue before the barrier
        if (ctal && tid == 0) tstep = clock64();
        // the next step's plan (read after this step's decision)
        if (tid == SNT - 1 && k1 < a.ntot) sp_plan(a, k1, min(k1 + a.P, a.ntot), &sm.plan[(t + 1) & 1]);
        if (PCDN_SP_L2PF && k1 < a.ntot) {   // the next step's descriptors and positions into L2
            const int64_t n1 = min(k1 + a.P, a.ntot);
            const int64_t gt = (int64_t)c * SNT + tid, lines = ((n1 - k1) * 16 + 127) / 128;
            if (gt < lines) pf_l2_last(reinterpret_cast<const char *>(&a.colinfo[k1]) + 128 * gt);
            else if (gt - lines < ((n1 - k1) * 4 + 127) / 128)
                pf_l2_last(reinterpret_cast<const char *>(&a.order[k1]) + 128 * (gt - lines));
        }

        const bool fullP = Pt == a.P;
        const int64_t pb0 = k0 + (fullP ? pbs0 : (int64_t)c * Pt / G);
        const int64_t pb1 = k0 + (fullP ? pbs1 : (int64_t)(c + 1) * Pt / G);
        ShareReg sh;
        sh.kk = -1;
        if (pb0 + tid < pb1) {   // loads issued here, consumed by the line search
            sh.kk = pb0 + tid;
            sh.j = __ldg(&a.order[sh.kk]);
            sh.wj = ldcg(&a.w[sh.j]);
            sh.d = ldcg(&a.dk[sh.kk - k0]);
            sh.delta = ldcg(&a.deltak[sh.kk - k0]);
        }
        RowReg rr;
        rr.i = -1;
        rr.has_dx = 0;

        // ---------------- the step's full columns (dense_dx) ------------------------------------
        DenseInfo di;
        di.f_lo = pl.f_lo;
        di.nf = pl.nf;
        di.any = false;
        if (di.nf > 0) {
            int any = 0;
            for (int64_t e = tid; e < di.nf; e += SNT) {
                const int32_t kk = __ldg(&a.flist[di.f_lo + e]);
                const double d = ldcg(&a.dk[kk - k0]);
                if (e < FMAX) {
                    sm.fd[e] = d;
                    sm.fcp[e] = colinfo_p0(__ldg(&a.colinfo[kk]));   // (a.val's offset of the column)
                }
                any |= d != 0.0;
            }
            di.any = __syncthreads_or(any) != 0;
        }

        // ---------------- phase C1: touched set of this CTA's row block -------------------------
        if (di.any) {   // a full column with d_j != 0 touches every sample (reading Z8)
            const int64_t nrows = min(a.s, we * 32) - row_base;
            int32_t *Tw = nrows <= TSM ? sm.tl : a.tlist + row_base;
            for (int64_t li = tid; li < nrows; li += SNT) Tw[li] = (int32_t)(row_base + li);
            if (tid == 0) sm.nT = nrows > 0 ? nrows : 0;
            __syncthreads();
        } else {
            const int64_t nwc = we - wb;
            const int64_t wpt = (nwc + SNT - 1) / SNT;
            const int64_t w0 = wb + (int64_t)tid * wpt, w1 = min(we, w0 + wpt);
            uint32_t wv[WREG];
            unsigned cntb = 0;
#pragma unroll
            for (int r = 0; r < WREG; r++) {
                wv[r] = (w0 + r < w1) ? ldst<TK>(&a.bits[w0 + r]) : 0u;
                cntb += __popc(wv[r]);
            }
            for (int64_t wi = w0 + WREG; wi < w1; wi++) cntb += __popc(ldst<TK>(&a.bits[wi]));
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
            const unsigned sw = lane < SNW ? (unsigned)sm.scan_w[lane] : 0u;
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
                    uint32_t m = ldst<TK>(&a.bits[wi]);
                    while (m) {
                        const int b = __ffs(m) - 1;
                        m &= m - 1;
                        Tw[pos++] = (int32_t)(wi * 32 + b);
                    }
                }
            }
            if (tid == 0) sm.nT = total;
            __syncthreads();
        }
        const int64_t nT = sm.nT;
        const int32_t *Tl = nT <= TSM ? sm.tl : a.tlist + row_base;
        if (di.any && nT <= TSM) {
            // the full columns' d'x part of every row of the block, (row, column chunk) per thread so
            // that a column's loads are coalesced over rows; chunk partials added in chunk order
            const int R = (int)nT;
            const int C = R >= SNT ? 1 : (int)min((int64_t)(SNT / max(R, 1)), di.nf);
            double *dpart = &sm.red[0][0];   // SNW*32 = SNT doubles
            for (int r0 = 0; r0 < R; r0 += SNT) {
                const int tt = tid;
                if (C == 1) {
                    if (r0 + tt < R) sm.dxd[r0 + tt] = sp_dense_dx(a.flist, a.dk, a.colinfo, a.val, sm.fd, sm.fcp, di.f_lo, di.nf, k0,
                                                                       row_base + r0 + tt);
                } else if (tt < R * C) {
                    const int r = tt % R, chn = tt / R;
                    const int64_t e0 = (int64_t)chn * di.nf / C, e1 = (int64_t)(chn + 1) * di.nf / C;
                    const int64_t i = row_base + r;
                    double part = 0.0;
                    for (int64_t e = e0; e < e1; e++) {
                        double d;
                        int64_t cp;
                        if (e < FMAX) {
                            d = sm.fd[e];
                            cp = sm.fcp[e];
                        } else {
                            const int32_t kk = __ldg(&a.flist[di.f_lo + e]);
                            d = ldcg(&a.dk[kk - k0]);
                            cp = colinfo_p0(__ldg(&a.colinfo[kk]));
                        }
                        if (d != 0.0) part += d * (double)__ldg(&a.val[cp + i]);
                    }
                    dpart[tt] = part;
                }
            }
            if (C > 1) {
                __syncthreads();
                for (int r = tid; r < R; r += SNT) {
                    double x = 0.0;
                    for (int chn = 0; chn < C; chn++) x += dpart[chn * R + r];
                    sm.dxd[r] = x;
                }
            }
            __syncthreads();
        }
        SP_MARK(2);
        if (ctal && tid == 0) {
            ctal[2] += nT;
            ctal[3] += clock64() - tstep;
        }

        // ---------------- phase C2+C3: fold d'x_i (a3) and the Armijo windows (a4) --------------
        WinState ws;
        ws.q0 = 0;
        // the first window: one candidate after a step that accepted q = 0 (almost every step at the
        // configured P: the second candidate's loss changes would sit on every step's critical path),
        // two after q = 1, six otherwise
        ws.nq = prev_q == 0 ? 1 : prev_q <= 1 ? 2 : QW;
        ws.qacc = -1;
        ws.bad = 0;
        ws.win = 0;
        ws.nospec = 0;
        // speculative commit (a5) before the decision's barrier: one touched sample per thread, no
        // full column (then T is the whole block)
        const bool spec = nT <= SNT && !di.any;
        double alpha_s = 1.0;
        for (int q = 0; q < q_spec; q++) alpha_s *= a.beta;
        while (true) {
            if (ws.nq == 1)
                sp_window<1, LOSS>(a, sm, sy, ws, Tl, nT, k0, pb0, pb1, G, c, tid, lane, warp, sh, rr, di, spec, alpha_s,
                                   wb, we, prof, tprev, ctal, tstep);
            else if (ws.nq <= 2)
                sp_window<2, LOSS>(a, sm, sy, ws, Tl, nT, k0, pb0, pb1, G, c, tid, lane, warp, sh, rr, di, spec, alpha_s,
                                   wb, we, prof, tprev, ctal, tstep);
            else
                sp_window<QW, LOSS>(a, sm, sy, ws, Tl, nT, k0, pb0, pb1, G, c, tid, lane, warp, sh, rr, di, spec, alpha_s,
                                    wb, we, prof, tprev, ctal, tstep);
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
        // the speculation hit: every CTA that could speculate did, with the accepted q -- then no
        // third barrier (the w commit below reads registers only: P <= SNT * G)
        const bool hit = !bad && qacc >= 0 && qacc == q_spec;
        const bool skip3 = hit && !ws.nospec && a.P <= (int64_t)SNT * G;
        if (qacc >= 0) q_spec = qacc;
        if (spec) {
            // correct a missed speculation from registers (alpha_acc = 0: the state before the step)
            if (!hit && rr.i >= 0) {
                const double zn = rr.zi + alpha_acc * rr.dx;
                stst<TK>(&a.z[rr.i], zn);
                stst<TK>(&a.coef[rr.i], coef_next(LOSS, make_double2(rr.cg, 2.0), zn, alpha_acc * rr.dx, rr.yi));
            }
            if (a.debug && rr.i >= 0) {
                a.dbg_dx[rr.i] = rr.dx;
                a.dbg_mark[rr.i] = 1;
            }
        } else {   // the commit (a5) of a CTA that could not speculate
            // ---------------- commit (a5): this CTA's samples and bundle share; clear the bitmaps -----
            // (every fold of the step finished before the decision's barrier, so the written-slot words
            // can be cleared here even where two samples' segments share a word)
            // (the thread's first sample from registers; the others in batches of SP_CB, all loads in
            // flight together)
            if (rr.i >= 0) {
                const int32_t i = rr.i;
                if (qacc >= 0) {
                    const double zn = rr.zi + alpha_acc * rr.dx;
                    stst<TK>(&a.z[i], zn);
                    const double2 cfo = LOSS == LOSS_SQ ? ldst<TK>(&a.coef[i]) : make_double2(0.0, 0.0);
                    stst<TK>(&a.coef[i], coef_next(LOSS, cfo, zn, alpha_acc * rr.dx, rr.yi));
                }
                if (rr.r1 > rr.r0)
                    for (int64_t wd = rr.r0 >> 5; wd <= ((rr.r1 - 1) >> 5); wd++) a.sbits[wd] = 0u;
                if (a.debug) {
                    a.dbg_dx[i] = rr.dx;
                    a.dbg_mark[i] = 1;
                }
            }
            for (int64_t lb = tid + SNT; lb < nT; lb += (int64_t)SNT * SP_CB) {
                int32_t ii[SP_CB];
                double dxv[SP_CB], zv[SP_CB];
                double2 cfo[SP_CB];
                int64_t ra[SP_CB], rb[SP_CB];
                int yv[SP_CB];
    #pragma unroll
                for (int e = 0; e < SP_CB; e++) {
                    const int64_t li = lb + (int64_t)e * SNT;
                    ii[e] = li < nT ? Tl[li] : -1;
                }
    #pragma unroll
                for (int e = 0; e < SP_CB; e++) {
                    dxv[e] = zv[e] = 0.0;
                    cfo[e] = make_double2(0.0, 0.0);
                    ra[e] = rb[e] = 0;
                    yv[e] = 1;
                    if (ii[e] >= 0) {
                        dxv[e] = ldst<TK>(&a.dxg[ii[e]]);
                        ra[e] = ldro<TK>(&a.row_ptr[ii[e]]);
                        rb[e] = ldro<TK>(&a.row_ptr[ii[e] + 1]);
                        if (qacc >= 0) {
                            zv[e] = ldst<TK>(&a.z[ii[e]]);
                            yv[e] = (int)a.y[ii[e]];
                            if (LOSS == LOSS_SQ) cfo[e] = ldst<TK>(&a.coef[ii[e]]);
                        }
                    }
                }
    #pragma unroll
                for (int e = 0; e < SP_CB; e++) {
                    const int32_t i = ii[e];
                    if (i < 0) continue;
                    if (qacc >= 0) {
                        const double zn = zv[e] + alpha_acc * dxv[e];
                        stst<TK>(&a.z[i], zn);
                        stst<TK>(&a.coef[i], coef_next(LOSS, cfo[e], zn, alpha_acc * dxv[e], yv[e]));
                    }
                    if (rb[e] > ra[e])
                        for (int64_t wd = ra[e] >> 5; wd <= ((rb[e] - 1) >> 5); wd++) a.sbits[wd] = 0u;
                    if (a.debug) {
                        a.dbg_dx[i] = dxv[e];
                        a.dbg_mark[i] = 1;
                    }
                }
            }
            for (int64_t wi = wb + tid; wi < we; wi += SNT) a.bits[wi] = 0u;
        }
        if (qacc >= 0) {
            for (int64_t kb = pb0 + tid; kb < pb1; kb += (int64_t)SNT * SP_CB) {
                int32_t jj[SP_CB];
                double wv[SP_CB], dv[SP_CB];
#pragma unroll
                for (int e = 0; e < SP_CB; e++) {
                    const int64_t kk = kb + (int64_t)e * SNT;
                    jj[e] = kk < pb1 ? (kk == sh.kk ? sh.j : __ldg(&a.order[kk])) : -1;
                }
#pragma unroll
                for (int e = 0; e < SP_CB; e++) {
                    const int64_t kk = kb + (int64_t)e * SNT;
                    wv[e] = dv[e] = 0.0;
                    if (jj[e] >= 0) {
                        wv[e] = kk == sh.kk ? sh.wj : ldcg(&a.w[jj[e]]);
                        dv[e] = kk == sh.kk ? sh.d : ldcg(&a.dk[kk - k0]);
                    }
                }
#pragma unroll
                for (int e = 0; e < SP_CB; e++)
                    if (jj[e] >= 0) a.w[jj[e]] = wv[e] + alpha_acc * dv[e];
            }
        }
        SP_MARK(6);
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
        if (!skip3) sy.sync();
        else __syncthreads();   // (sm.plan, written after the first barrier, before its use)
        SP_MARK(7);
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
    if (ctal_out && tid < 16) ctal_out[tid] += sm.cprof[tid];
#undef SP_MARK
}

}  // namespace pcdn
