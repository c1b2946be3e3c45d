// pcdn_dense.cuh -- the bundle-step kernel for fully dense problems (every column holds a nonzero
// in every row; config 4, gisette-like), SURVEY.md 8(a) rows a1..a5.
//
// A dense bundle step is a pair of skinny dense products (g = X_B^T G, h = (X_B o X_B)^T H, then
// d'x = X_B d), so the step is laid out by ROW BLOCKS instead of records:
//   CTA c of the cooperative grid owns rows [r0, r1): z, coef and d'x of those rows live in its
//   shared memory for the whole launch (one launch = all bundle steps of an outer iteration), and
//   X_B restricted to those rows (the step's TILE, x_ij at col_ptr[j] + i: no row indices) is
//   copied into shared memory by cp.async one step AHEAD, while the current step computes.
//   G  every thread takes bundle columns: partial g/h over the CTA's rows in row order (from the
//      tile) -> part_gh[c][pos]                                                   [grid barrier B1]
//   R  (the previous step's decision, below)
//   D  column pos is finished by CTA pos mod G: one warp sums the G partials (lanes, fixed tree),
//      Eq.5 -> d_j, Delta term; dk/deltak in HBM                                  [grid barrier B2]
//   X  d'x of the CTA's rows in bundle order from the tile (row, column chunk) threads, chunks
//      added in chunk order
//   LS loss changes of the CTA's rows for a window of Armijo candidates, the L1 term and Delta of
//      its finished columns -> part_ls[c]
//   Speculative commit: the decision needs one more grid-wide exchange.  Instead of a third barrier
//   per step, every CTA continues with the NEXT step's G phase using coef(z + alpha_s d'x) for the
//   likely step alpha_s = beta^{q of the previous step}; the next B1 then also publishes the line-search
//   partials, and right after it (R) every CTA sums them in the same fixed order, takes the same
//   decision (first q with LHS <= sigma alpha Delta, Eq.6 with Eq.12) and commits z, w_B, F.  When
//   the accepted alpha differs from alpha_s (or further windows are needed), coef is recomputed from
//   the committed z and the G phase is redone (one extra barrier): the arithmetic of every accepted
//   step is exactly that of the sequential algorithm.
// Every sample is touched when some d_j != 0 (reading Z8): T = all rows.
// With a.n_outer > 1 the launch runs the whole solve: at each outer boundary every CTA recomputes F
// from (z, w) with k_obj's arithmetic, takes the Eq.14 stop test, and the grid writes the next
// partition (so order / colinfo are read through L2, never the non-coherent path).
#pragma once
#include "pcdn_kernels.cuh"
#include "pcdn_resident.cuh"   // mbarrier primitives

namespace pcdn {

constexpr int D_RMAX = 512;    // rows per CTA kept in shared memory
constexpr int D_PMAX = 2048;   // bundle columns whose d_j is staged per step
constexpr int D_OWN = 32;      // finished columns per CTA per step kept for L1 / commit

struct DenseFixed {
    uint64_t tmb[2];           // tile-buffer mbarriers
    double z[D_RMAX];          // committed z of the CTA's rows
    double dx[D_RMAX];         // d'x of the current (or just decided) step
    double2 coef[2][D_RMAX];   // [cc]: coef at the committed z; [cc ^ 1]: speculative coef
    int8_t y[D_RMAX];
    double dcol[D_PMAX];
    double dpart[NT];
    double red[NW][32];
    double tot[32];
    // columns finished by this CTA in the step (phase D): position, j, w_j, d_j, Delta term
    int32_t okk[D_OWN], oj[D_OWN];
    double ow[D_OWN], od[D_OWN], odl[D_OWN];
    int dec_q, dec_bad;
    double dec_alpha, dec_lhs, dec_rhs, dec_Delta;
    double F;
    long long cnt[4];
    long long pacc[16];
};

__host__ __device__ inline size_t dense_fixed_bytes() { return (sizeof(DenseFixed) + 127) & ~(size_t)127; }

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint32_t mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(s_addr(dst)), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

// X_B of the step restricted to rows [r0, r0 + R) -> tile [pos][r] (column stride Rs), by the TMA
// engine: one 1-D bulk copy per column (16-byte aligned: row blocks start at multiples of 4 rows
// and s % 4 == 0), completing R*4 bytes each on the buffer's mbarrier.  The generic-proxy reads of
// the buffer (two steps back) are ordered before the async-proxy writes by the proxy fence.
// Columns [pa, pb) of the step are issued by this call; the part with pa == 0 also posts the whole
// step's byte count on the mbarrier.
__device__ __forceinline__ void dense_prefetch(const StepArgs &a, float *tile, uint32_t mbar, int64_t k0, int Pt,
                                               int64_t r0, int R, int Rs, int tid, int64_t p0_first, int pa, int pb)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0 && pa == 0) mbar_arrive_tx(mbar, (uint32_t)Pt * (uint32_t)R * 4u);
    if (R > 0) {
        for (int pos = tid; pos < Pt; pos += NT) {
            if (pos < pa || pos >= pb) continue;
            // the first descriptor of each thread was loaded early (p0_first): no dependent load here
            const int64_t cp = (pos == tid ? p0_first : colinfo_p0(__ldcg(&a.colinfo[k0 + pos]))) + r0;
            bulk_g2s(tile + (int64_t)pos * Rs, a.val + cp, (uint32_t)R * 4u, mbar);
        }
    }
}

// G: partial g/h of the CTA's rows for every bundle column, rows in order (from the tile, or from
// HBM with 16-byte loads once aligned when the tile does not fit: the same sums either way)
__device__ __forceinline__ void dense_gphase(const StepArgs &a, const float *tile, const double2 *coef, int64_t k0,
                                             int Pt, int64_t r0, int R, int Rs, int c, double *part_gh, int tid)
{
    for (int pos = tid; pos < Pt; pos += NT) {
        double g = 0.0, h = 0.0;
        if (tile) {   // R % 4 == 0; 16-byte reads, conflict-free for Rs / 4 odd
            const float4 *tp = reinterpret_cast<const float4 *>(tile + (int64_t)pos * Rs);
#pragma unroll 2
            for (int r4 = 0; r4 < (R >> 2); r4++) {
                const float4 v = tp[r4];
                const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const double x = (double)xv[e];
                    const double2 cf = coef[4 * r4 + e];
                    g += x * cf.x;
                    h += (x * x) * cf.y;
                }
            }
        } else {
            const float *xp = a.val + colinfo_p0(__ldcg(&a.colinfo[k0 + pos])) + r0;
            const int head = min(R, (int)((4 - (((uintptr_t)xp >> 2) & 3)) & 3));
            int r = 0;
            for (; r < head; r++) {
                const double x = (double)__ldg(xp + r);
                const double2 cf = coef[r];
                g += x * cf.x;
                h += (x * x) * cf.y;
            }
#pragma unroll 4
            for (; r + 4 <= R; r += 4) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(xp + r));
                const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const double x = (double)xv[e];
                    const double2 cf = coef[r + e];
                    g += x * cf.x;
                    h += (x * x) * cf.y;
                }
            }
            for (; r < R; r++) {
                const double x = (double)__ldg(xp + r);
                const double2 cf = coef[r];
                g += x * cf.x;
                h += (x * x) * cf.y;
            }
        }
        __stcg(reinterpret_cast<double2 *>(&part_gh[((int64_t)c * a.P + pos) * 2]), make_double2(g, h));
    }
}

// One Armijo window [q0, q0 + nq) of the current step: loss changes of the CTA's rows (from the
// committed z, its coef and d'x), L1 term and Delta of its finished columns -> this CTA's row of
// the window's partial buffer.  No barrier here: the caller publishes the row with the next one.
template <int LOSS>
__device__ __forceinline__ void dense_ls_partial(const StepArgs &a, DenseFixed &sm, const double2 *coefc, int q0,
                                                 int nq, bool dense_any, int R, int nown, int64_t k0, int c, int G,
                                                 double *part, int tid, int lane, int warp, double2 *spec = nullptr,
                                                 double alpha_s = 0.0)
{
    double alpha0 = 1.0;
    for (int q = 0; q < q0; q++) alpha0 *= a.beta;
    constexpr int W = WinLayout<QW>::W;   // 16 slots: Ls[0,6) L1[6,12) Delta
    double acc[W];
#pragma unroll
    for (int q = 0; q < W; q++) acc[q] = 0.0;
    if (dense_any) {   // one (row, candidate) pair per thread: the transcendental latency once
        for (int idx = tid; idx < R * nq; idx += NT) {
            const int q = idx / R, r = idx - q * R;
            double al = alpha0;
            for (int qq = 0; qq < q; qq++) al *= a.beta;   // the decision's alpha of candidate q
            const double v = loss_change(LOSS, sm.z[r], sm.y[r], coefc[r].x, sm.dx[r], al);
#pragma unroll
            for (int qq = 0; qq < QW; qq++)
                if (qq == q) acc[qq] += v;
        }
        // the speculative coef for the next step's G phase, by the threads after the pairs
        if (spec) {
            for (int r = tid - ((R * nq) % NT); r < R; r += NT)
                if (r >= 0) spec[r] = coef_next(LOSS, coefc[r], __fma_rn(alpha_s, sm.dx[r], sm.z[r]), alpha_s * sm.dx[r], sm.y[r]);
        }
    }
    for (int m = tid; m < nown; m += NT) {
        double wj, d, dl;
        if (m < D_OWN) {
            wj = sm.ow[m];
            d = sm.od[m];
            dl = sm.odl[m];
        } else {   // beyond the staged slots: from HBM
            const int pos = c + G * m;
            wj = ldcg(&a.w[__ldcg(&a.order[k0 + pos])]);
            d = ldcg(&a.dk[pos]);
            dl = ldcg(&a.deltak[pos]);
        }
        double al = alpha0;
        for (int q = 0; q < nq; q++) {
#pragma unroll
            for (int qq = 0; qq < QW; qq++)
                if (qq == q) acc[QW + qq] += fabs(wj + al * d) - fabs(wj) + a.mu * al * d * (wj + 0.5 * al * d);
            al *= a.beta;
        }
        acc[2 * QW] += dl;
    }
    constexpr int SPL = 32 / W;
    {
        const double tt = xreduce<W>(acc, lane);
        if ((lane % SPL) == 0) sm.red[warp][lane / SPL] = tt;
    }
    __syncthreads();
    if (warp == 0 && lane < W) {
        double s = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < NW; w2++) s += sm.red[w2][lane];
        part[(int64_t)c * NPART + lane] = s;
    }
}

// After the barrier that published a window: every CTA sums the G rows in the same fixed order and
// takes the same decision; returns through sm.dec_* (valid after the trailing __syncthreads).
__device__ __forceinline__ void dense_decide(const StepArgs &a, DenseFixed &sm, const double *part, int q0, int nq,
                                             int G, int lane, int warp)
{
    constexpr int W = WinLayout<QW>::W;
    grid_totals<W>(part, G, sm.red, sm.tot, lane, warp);
    if (warp == 0 && lane == 0) {
        double alpha0 = 1.0;
        for (int q = 0; q < q0; q++) alpha0 *= a.beta;
        const double D = sm.tot[2 * QW];
        int qa = -1, bl = 0;
        double al = alpha0, la = 0.0, ra = 0.0, aa = 0.0;
        for (int q = 0; q < nq; q++) {
            const double lhs = sm.tot[QW + q] + a.c * sm.tot[q];
            const double rhs = a.sigma * al * D;
            if (!isfinite(lhs) || !isfinite(D)) {
                bl = 1;
                break;
            }
            if (lhs <= rhs) {
                qa = q0 + q;
                aa = al;
                la = lhs;
                ra = rhs;
                break;
            }
            al *= a.beta;
        }
        sm.dec_q = qa;
        sm.dec_bad = bl;
        sm.dec_alpha = aa;
        sm.dec_lhs = la;
        sm.dec_rhs = ra;
        sm.dec_Delta = D;
    }
    __syncthreads();
}

// The outer boundary of a whole-solve launch (a6): F from scratch over (z, w) -- k_obj's blocks and
// tree, bit for bit -- the Eq.14 stop test, and the next outer iteration's partition into the other
// half of order / colinfo.
template <int LOSS>
__device__ __forceinline__ bool dense_boundary(const StepArgs &a, DenseFixed &sm, GridSync &sy, int64_t r0, int R, int G,
                                               int c, int tid, int oi)
{
    for (int r = tid; r < R; r += NT) a.z[r0 + r] = sm.z[r];
    sy.sync();   // z of every row and the w commits of the last step
    const bool more = oi + 1 < a.n_outer;
    if (more) {
        const int64_t kn = (int64_t)((oi + 1) & 1) * a.n;
        // from the last CTA down: the objective blocks below start at CTA 0, so the two run side by side
        perm_positions(a.seed, a.outer0 + oi + 1, a.n, a.s, a.col_ptr, a.heavy_len,
                       const_cast<int32_t *>(a.order) + kn, a.pflag, a.pfflag, const_cast<int4 *>(a.colinfo) + kn,
                       (int64_t)(G - 1 - c) * NT + tid, (int64_t)G * NT);
    }
    const int h = tid / OBJ_NB, gt = tid % OBJ_NB;
    double(*wsum)[3] = reinterpret_cast<double(*)[3]>(&sm.red[0][0] + h * 3 * (OBJ_NB / 32));
    for (int rb = 0; rb < OBJ_NB; rb += 2 * G) {
        const int b = rb + 2 * c + h;
        obj_group_partial(b, gt, gt >> 5, a.s, a.n, a.z, a.y, a.w, LOSS, a.t, wsum, a.objp, b < OBJ_NB);
    }
    sy.sync();   // the partials (and the next partition)
    double *sh = sm.dcol;   // [3][OBJ_NB]: k_obj_final's tree, in every CTA
    if (tid < OBJ_NB) {
        sh[tid] = __ldcg(&a.objp[3 * tid]);
        sh[OBJ_NB + tid] = __ldcg(&a.objp[3 * tid + 1]);
        sh[2 * OBJ_NB + tid] = __ldcg(&a.objp[3 * tid + 2]);
    }
    __syncthreads();
    for (int o = OBJ_NB / 2; o > 0; o >>= 1) {
        if (tid < o) {
            sh[tid] += sh[tid + o];
            sh[OBJ_NB + tid] += sh[OBJ_NB + tid + o];
            sh[2 * OBJ_NB + tid] += sh[2 * OBJ_NB + tid + o];
        }
        __syncthreads();
    }
    const double Fv = a.c * sh[0] + sh[OBJ_NB] + 0.5 * a.mu * sh[2 * OBJ_NB];
    const bool stop = !more || !isfinite(Fv) || (a.eps_stop > 0 && (Fv - a.fstar) / a.fstar <= a.eps_stop);
    if (tid == 0) sm.F = Fv;
    if (c == 0 && tid == 0) {
        *a.F = Fv;
        *a.outers_done = oi + 1;
        if (!isfinite(Fv)) atomicMax(a.status, 3);
    }
    __syncthreads();   // sh (dcol) is reused by the next step
    return stop;
}

template <int LOSS>
__global__ void __launch_bounds__(NT, 1) k_step_dense(StepArgs a)
{
    if (a.stop && ldcg(a.stop)) return;   // the solve already ended (queued ahead; grid-uniform)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DenseFixed &sm = *reinterpret_cast<DenseFixed *>(smem_raw);
    float *tiles = reinterpret_cast<float *>(smem_raw + dense_fixed_bytes());
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    GridSync sy(a.bar);
    // row blocks start at multiples of 4 rows when s % 4 == 0 and val is 16-byte aligned, so every
    // column's block is one aligned bulk copy
    const bool al4 = (a.s % 4 == 0) && (((uintptr_t)a.val & 15) == 0);
    const int64_t r0 = al4 ? 4 * ((int64_t)c * (a.s / 4) / G) : (int64_t)c * a.s / G;
    const int64_t r1 = al4 ? 4 * ((int64_t)(c + 1) * (a.s / 4) / G) : (int64_t)(c + 1) * a.s / G;
    const int R = (int)(r1 - r0);
    const int Rmax = al4 ? (int)(4 * ((a.s / 4 + G - 1) / G)) : (int)((a.s + G - 1) / G);
    const int Rs = ((Rmax + 3) & ~3) | 4;   // tile column stride: 16-byte multiple, Rs / 4 odd
    double *part_gh = a.part_gh;   // [G][P][2]
    double *part_ls = a.part;      // [2][G][NPART]
    // the tile of every step of the launch fits (Pt <= P): copied a step ahead by the TMA engine
    const bool use_tile = al4 && (int64_t)Rs * a.P <= (int64_t)a.dense_tcap;
    uint64_t *tmb = sm.tmb;

    // ---------------- prologue: own rows into shared memory, the first tile ------------------
    int cc = 0;   // coef[cc] = coef at the committed z
    for (int r = tid; r < R; r += NT) {
        sm.z[r] = ldcg(&a.z[r0 + r]);
        sm.coef[0][r] = ldcg(&a.coef[r0 + r]);
        sm.y[r] = a.y[r0 + r];
        sm.dx[r] = 0.0;
    }
    if (tid < 16) sm.pacc[tid] = 0;
    if (tid == 0) {
        sm.F = ldcg(a.F);
        for (int i = 0; i < 4; i++) sm.cnt[i] = 0;
    }
    if (tid == 0) {
        mbar_init(s_addr(&tmb[0]), 1);
        mbar_init(s_addr(&tmb[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    bool inflight = false;   // a tile copy was issued and not yet waited for (for step inflight_t)
    int64_t inflight_t = 0;
    long long tprev = 0;
    const bool prof = PCDN_PROFILE && a.prof != nullptr && c == 0 && tid == 0;
#define DPROF(i)                                 \
    do {                                         \
        if (prof) {                              \
            const long long now_ = clock64();    \
            sm.pacc[i] += now_ - tprev;          \
            tprev = now_;                        \
        }                                        \
    } while (0)
    int prev_q = 0, wcount = 0;
    // the step waiting for its decision (published by the next barrier)
    bool pend = false, pend_any = false, bad = false;
    int pend_q0 = 0, pend_nq = 0, pend_nown = 0;
    int64_t pend_k0 = 0, pend_t = 0;   // pend_t: step index within the launch
    bool pend_last = false;            // the pending step is its outer iteration's last
    int pend_Pt = 0;
    double alpha_s = 1.0;

    // Decide the pending step (its first window was published by the barrier just passed), commit
    // it; returns true when the G phase that used the speculative coef must be redone.
    auto resolve = [&]() -> bool {
        int q0 = pend_q0, nq = pend_nq;
        int qacc = -1;
        double alpha_acc = 0.0, lhs_acc = 0.0, rhs_acc = 0.0, Dl = 0.0;
        while (true) {
            dense_decide(a, sm, part_ls + (int64_t)((wcount - 1) & 1) * G * NPART, q0, nq, G, lane, warp);
            qacc = sm.dec_q;
            bad = bad || sm.dec_bad != 0;
            alpha_acc = sm.dec_alpha;
            lhs_acc = sm.dec_lhs;
            rhs_acc = sm.dec_rhs;
            Dl = sm.dec_Delta;
            __syncthreads();   // sm.dec_* / sm.red / sm.tot are reused
            if (qacc >= 0 || bad) break;
            q0 += nq;
            if (q0 > a.qmax) break;
            nq = QW;
            // a further window of the pending step, from the committed state (coef[cc])
            dense_ls_partial<LOSS>(a, sm, sm.coef[cc], q0, nq, pend_any, R, pend_nown, pend_k0, c, G,
                                   part_ls + (int64_t)(wcount & 1) * G * NPART, tid, lane, warp);
            wcount++;
            sy.sync();
        }
        DPROF(13);
        if (qacc > a.qmax) qacc = -1;
        if (qacc < 0) alpha_acc = 0.0;
        prev_q = qacc < 0 ? QW : qacc;
        // commit z (and coef): the speculative coef is exactly coef(z_new) when alpha_acc == alpha_s
        const bool hit = !pend_any || alpha_acc == alpha_s;
        if (pend_any) {
            for (int r = tid; r < R; r += NT) {
                const double zn = __fma_rn(alpha_acc, sm.dx[r], sm.z[r]);   // the same rounding as the speculation
                sm.z[r] = zn;
                if (!hit) sm.coef[cc ^ 1][r] = coef_next(LOSS, sm.coef[cc][r], zn, alpha_acc * sm.dx[r], sm.y[r]);
            }
            cc ^= 1;
            if (a.debug) {
                for (int r = tid; r < R; r += NT) {
                    a.dbg_dx[r0 + r] = sm.dx[r];
                    a.dbg_mark[r0 + r] = 1;
                }
            }
        }
        if (qacc >= 0) {
            for (int m = tid; m < pend_nown; m += NT) {
                if (m < D_OWN) {
                    a.w[sm.oj[m]] = sm.ow[m] + alpha_acc * sm.od[m];
                } else {
                    const int pos = c + G * m;
                    const int32_t j = __ldcg(&a.order[pend_k0 + pos]);
                    a.w[j] = ldcg(&a.w[j]) + alpha_acc * ldcg(&a.dk[pos]);
                }
            }
        }
        DPROF(14);
        if (c == 0 && tid == 0) {
            double F = sm.F;
            if (qacc >= 0) F = F + lhs_acc;
            sm.F = F;
            if (bad || pend_last) {
                *a.F = F;
                if (bad) atomicMax(a.status, 3);
                a.info[0] = (double)qacc;
                a.info[1] = alpha_acc;
                a.info[2] = Dl;
                a.info[3] = lhs_acc;
                a.info[4] = rhs_acc;
                a.info[5] = F;
                a.info[7] = pend_any ? (double)a.s : 0.0;
            }
            const int64_t gstep = a.trace_off + pend_t;
            if (gstep < a.trace_cap) {
                if (a.q_trace) a.q_trace[gstep] = qacc;
                if (a.F_trace) a.F_trace[gstep] = F;
            }
            sm.cnt[0] += 1;
            sm.cnt[1] += qacc < 0 ? 1 : 0;
            sm.cnt[2] += pend_any ? a.s : 0;
            sm.cnt[3] += pend_Pt;
        }
        __syncthreads();   // committed z / coef / own columns before their reuse
        pend = false;
        return !hit;
    };

    // outer iterations of this launch (one unless a.n_outer > 1: then positions of outer oi sit at
    // [kb, kb + ntot) of order / colinfo, and steps are numbered T = T0 + t across the launch for
    // the tile buffers' mbarrier phases and the traces)
    for (int oi = 0;; oi++) {
    const int64_t kb = (int64_t)(oi & 1) * a.n;
    const int64_t T0 = (int64_t)oi * a.nsteps;
    if (use_tile && a.nsteps > 0) {
        const int P0 = (int)min(a.P, a.ntot);
        dense_prefetch(a, tiles + (size_t)(T0 & 1) * (size_t)a.dense_tcap, s_addr(&tmb[T0 & 1]), kb, P0, r0, R, Rs, tid,
                       tid < P0 ? colinfo_p0(__ldcg(&a.colinfo[kb + tid])) : 0, 0, P0);
        inflight = true;
        inflight_t = T0;
    }
    for (int64_t t = 0; t < a.nsteps; t++) {
        if (prof) tprev = clock64();
        const int64_t T = T0 + t;
        const int64_t k0 = kb + t * a.P;
        const int64_t k1 = min(k0 + a.P, kb + a.ntot);
        const int Pt = (int)(k1 - k0);
        float *tile = nullptr;
        // the next step's first tile descriptor of this thread, loaded now (used after the G phase)
        const int64_t kn1 = min(k1 + a.P, kb + a.ntot);
        const int64_t p0n = (use_tile && k1 + tid < kn1) ? colinfo_p0(__ldcg(&a.colinfo[k1 + tid])) : 0;
        if (use_tile) {
            tile = tiles + (size_t)(T & 1) * (size_t)a.dense_tcap;
            mbar_wait(s_addr(&tmb[T & 1]), (uint32_t)((T >> 1) & 1));   // this step's tile (issued a step ahead)
            inflight = false;
        }
        DPROF(8);

        // ---------------- G: partial g/h of the CTA's rows (speculative coef if pending) -----
        dense_gphase(a, tile, sm.coef[pend && pend_any ? cc ^ 1 : cc], k0, Pt, r0, R, Rs, c, part_gh, tid);
        DPROF(6);
        sy.arrive();   // B1: the g/h partials of this step and the line-search partials of the last
        DPROF(10);
        // the next step's tile, issued while the barrier completes (in the background of this
        // step's remaining phases)
        if (use_tile && t + 1 < a.nsteps) {
            dense_prefetch(a, tiles + (size_t)((T + 1) & 1) * (size_t)a.dense_tcap, s_addr(&tmb[(T + 1) & 1]), k1,
                           (int)(kn1 - k1), r0, R, Rs, tid, p0n, 0, (int)(kn1 - k1));
            inflight = true;
            inflight_t = T + 1;
        }
        DPROF(0);
        sy.wait();
        DPROF(1);
        // this warp's first column of phase D: its G partials are loaded now, summed after the
        // previous step's decision (the two L2 round trips overlap)
        const int pos_pre = c + G * warp;
        constexpr int PRE = 5;
        double2 pv[PRE];
        const bool pre = pos_pre < Pt && G <= 32 * PRE;
#pragma unroll
        for (int e = 0; e < PRE; e++) {
            const int c2 = lane + 32 * e;
            pv[e] = (pre && c2 < G) ? __ldcg(reinterpret_cast<const double2 *>(&part_gh[((int64_t)c2 * a.P + pos_pre) * 2]))
                                    : make_double2(0.0, 0.0);
        }
        bool redone = false;
        if (pend) {
            if (resolve()) {   // the speculation missed: redo G from the committed coef
                dense_gphase(a, tile, sm.coef[cc], k0, Pt, r0, R, Rs, c, part_gh, tid);
                sy.sync();
                redone = true;
            }
            if (bad) break;
        }
        DPROF(9);

        // ---------------- D: finish the columns owned by this CTA ---------------------------
        for (int pos = c + G * warp; pos < Pt; pos += G * NW) {
            double g = 0.0, h = 0.0;
            if (pos == pos_pre && pre && !redone) {   // the same lane sums in the same c2 order
#pragma unroll
                for (int e = 0; e < PRE; e++) {
                    g += pv[e].x;
                    h += pv[e].y;
                }
            } else {
                for (int c2 = lane; c2 < G; c2 += 32) {
                    const double2 v = __ldcg(reinterpret_cast<const double2 *>(&part_gh[((int64_t)c2 * a.P + pos) * 2]));
                    g += v.x;
                    h += v.y;
                }
            }
            g = warp_sum(g);
            h = warp_sum(h);
            if (lane == 0) {
                const int32_t j = __ldcg(&a.order[k0 + pos]);
                const double wj = ldcg(&a.w[j]);
                const Dir r = finish_feature(a, g, h, wj);
                a.dk[pos] = r.d;
                a.deltak[pos] = r.delta;
                if (a.g_out) {
                    a.g_out[pos] = r.g;
                    a.h_out[pos] = r.h;
                }
                if (a.d_out) a.d_out[pos] = r.d;
                const int slot = (pos - c) / G;   // this CTA's m-th column (m = warp + NW * round)
                if (slot < D_OWN) {
                    sm.okk[slot] = pos;
                    sm.oj[slot] = j;
                    sm.ow[slot] = wj;
                    sm.od[slot] = r.d;
                    sm.odl[slot] = r.delta;
                }
            }
        }
        DPROF(2);
        sy.sync();   // B2
        DPROF(3);

        // ---------------- X: d'x of the CTA's rows in bundle order --------------------------
        int any = 0;
        for (int pos = tid; pos < Pt; pos += NT) {
            const double d = ldcg(&a.dk[pos]);
            if (pos < D_PMAX) sm.dcol[pos] = d;
            any |= d != 0.0;
        }
        const bool dense_any = __syncthreads_or(any) != 0;
        DPROF(11);
        if (dense_any) {
            const int C = R >= NT ? 1 : (int)min(NT / max(R, 1), Pt);
            for (int rb = 0; rb < R; rb += NT) {
                if (C == 1) {
                    const int r = rb + tid;
                    if (r < R) {
                        double x = 0.0;
                        for (int pos = 0; pos < Pt; pos++) {
                            const double d = pos < D_PMAX ? sm.dcol[pos] : ldcg(&a.dk[pos]);
                            const double xv = tile ? (double)tile[(int64_t)pos * Rs + r]
                                                   : (double)__ldg(&a.val[colinfo_p0(__ldcg(&a.colinfo[k0 + pos])) + r0 + r]);
                            if (d != 0.0) x += d * xv;
                        }
                        sm.dx[r] = x;
                    }
                } else if (tid < R * C) {
                    const int r = tid % R, ch = tid / R;
                    const int e0 = (int)((int64_t)ch * Pt / C), e1 = (int)((int64_t)(ch + 1) * Pt / C);
                    // no branch on d_j == 0: its product is +-0 and leaves the sum unchanged, and
                    // branch-free iterations let the loads of several columns be in flight
                    double x = 0.0;
                    if (tile && e1 <= D_PMAX) {
#pragma unroll 8
                        for (int pos = e0; pos < e1; pos++) x += sm.dcol[pos] * (double)tile[(int64_t)pos * Rs + r];
                    } else {
                        for (int pos = e0; pos < e1; pos++) {
                            const double d = pos < D_PMAX ? sm.dcol[pos] : ldcg(&a.dk[pos]);
                            const double xv = tile ? (double)tile[(int64_t)pos * Rs + r]
                                                   : (double)__ldg(&a.val[colinfo_p0(__ldcg(&a.colinfo[k0 + pos])) + r0 + r]);
                            x += d * xv;
                        }
                    }
                    sm.dpart[tid] = x;
                }
            }
            DPROF(12);
            if (C > 1) {
                __syncthreads();
                for (int r = tid; r < R; r += NT) {
                    double x = 0.0;
                    for (int ch = 0; ch < C; ch++) x += sm.dpart[ch * R + r];
                    sm.dx[r] = x;
                }
            }
            __syncthreads();
        }
        DPROF(4);

        // ---------------- LS: the first Armijo window (Eq.6 with Eq.12), published by B1 -----
        const int nq = prev_q <= 1 ? 2 : QW;
        const int nown = max(0, (Pt - c + G - 1) / G);   // columns finished by this CTA
        // with the speculative coef for the next step's G phase: alpha_s = beta^{previous q} (inside
        // the window), computed from the same expression as the commit (bit-identical on a hit)
        alpha_s = 1.0;
        for (int q = 0; q < min(prev_q, nq - 1); q++) alpha_s *= a.beta;
        dense_ls_partial<LOSS>(a, sm, sm.coef[cc], 0, nq, dense_any, R, nown, k0, c, G,
                               part_ls + (int64_t)(wcount & 1) * G * NPART, tid, lane, warp, sm.coef[cc ^ 1], alpha_s);
        wcount++;
        pend = true;
        pend_any = dense_any;
        pend_q0 = 0;
        pend_nq = nq;
        pend_nown = nown;
        pend_k0 = k0;
        pend_t = T;
        pend_last = t == a.nsteps - 1;
        pend_Pt = Pt;
        __syncthreads();   // speculative coef complete before the next G phase reads it
        DPROF(5);
    }
    if (pend && !bad) {   // the last step of the outer iteration: publish and decide it
        sy.sync();
        resolve();
    }
    if (a.n_outer <= 0 || bad) break;   // one outer iteration per launch (the host takes a6)
    // ---------------- outer boundary (a6) inside the launch ------------------------------------
    if (dense_boundary<LOSS>(a, sm, sy, r0, R, G, c, tid, oi)) break;
    prev_q = 0;   // as a fresh launch
    }   // outer iterations
    if (inflight)   // nothing may still be landing in shared memory at exit (an early break)
        mbar_wait(s_addr(&tmb[inflight_t & 1]), (uint32_t)((inflight_t >> 1) & 1));
    // ---------------- epilogue: own rows back to HBM ----------------------------------------
    for (int r = tid; r < R; r += NT) {
        a.z[r0 + r] = sm.z[r];
        a.coef[r0 + r] = sm.coef[cc][r];
    }
    if (c == 0 && tid == 0) {
        a.counters[0] += sm.cnt[0];
        a.counters[1] += sm.cnt[1];
        a.counters[3] += sm.cnt[2];
        a.counters[4] += sm.cnt[3];
    }
    if (prof)
        for (int i = 0; i < 16; i++) a.prof[i] += sm.pacc[i];
#undef DPROF
}

}  // namespace pcdn
