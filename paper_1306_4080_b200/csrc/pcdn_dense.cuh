// pcdn_dense.cuh -- the bundle-step kernel for fully dense problems (every column holds a nonzero
// in every row; config 4, gisette-like), SURVEY.md 8(a) rows a1..a5.
//
// A dense bundle step is a pair of skinny dense products (g = X_B^T G, h = (X_B o X_B)^T H, then
// d'x = X_B d), so the step is laid out by ROW BLOCKS instead of records:
//   CTA c of the cooperative grid owns rows [r0, r1): z, coef and d'x of those rows live in its
//   shared memory for the whole launch (one launch = all bundle steps of an outer iteration).
//   G  every thread takes bundle columns; for each, the partial g/h over the CTA's rows in row
//      order (x_ij at col_ptr[j] + i: no row indices) -> part_gh[c][pos]         [grid barrier]
//   D  column pos is finished by CTA pos mod G: one warp sums the G partials (lanes, fixed tree),
//      Eq.5 -> d_j, Delta term; dk/deltak in HBM                                [grid barrier]
//   X  every CTA stages (d_j, col_ptr[j]) of the step and forms d'x_i of its rows in bundle order
//      split over (row, column chunk) threads, chunks added in chunk order (X_B re-read from L2)
//   LS loss changes of the CTA's rows for a window of candidates, the L1 term and Delta of its
//      finished columns -> part_ls[c]                                             [grid barrier]
//      every CTA sums the G rows in the same fixed order and takes the same decision
//   commit z/coef of its rows (shared memory), w_j of its finished columns, F.
// Every sample is touched when some d_j != 0 (reading Z8): T = all rows.
#pragma once
#include "pcdn_kernels.cuh"

namespace pcdn {

constexpr int D_RMAX = 1024;   // rows per CTA kept in shared memory
constexpr int D_PMAX = 2048;   // bundle columns staged per step (d_j, col_ptr[j])
constexpr int D_OWN = 32;      // finished columns per CTA per step kept for L1 / commit
constexpr int D_TILE = 24576;  // floats of the CTA's X_B tile kept from phase G for phase X (96 KB)

struct DenseSmem {
    double z[D_RMAX];
    double2 coef[D_RMAX];
    double dx[D_RMAX];
    int8_t y[D_RMAX];
    double dcol[D_PMAX];
    int64_t cp[D_PMAX];
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
    float tile[D_TILE];   // X_B restricted to the CTA's rows, column-major [pos][r] (when it fits)
};

__global__ void __launch_bounds__(NT, 1) k_step_dense(StepArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DenseSmem &sm = *reinterpret_cast<DenseSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    GridSync sy(a.bar);
    const int64_t r0 = (int64_t)c * a.s / G, r1 = (int64_t)(c + 1) * a.s / G;
    const int R = (int)(r1 - r0);
    double *part_gh = a.part_gh;   // [G][P][2]
    double *part_ls = a.part;      // [2][G][NPART]

    // ---------------- prologue: own rows into shared memory ----------------------------------
    for (int r = tid; r < R; r += NT) {
        sm.z[r] = ldcg(&a.z[r0 + r]);
        sm.coef[r] = ldcg(&a.coef[r0 + r]);
        sm.y[r] = a.y[r0 + r];
    }
    if (tid < 16) sm.pacc[tid] = 0;
    if (tid == 0) {
        sm.F = ldcg(a.F);
        for (int i = 0; i < 4; i++) sm.cnt[i] = 0;
    }
    __syncthreads();
    long long tprev = 0;
    const bool prof = a.prof != nullptr && c == 0 && tid == 0;
#define DPROF(i)                                 \
    do {                                         \
        if (prof) {                              \
            const long long now_ = clock64();    \
            sm.pacc[i] += now_ - tprev;          \
            tprev = now_;                        \
        }                                        \
    } while (0)
    int prev_q = 0, wcount = 0;
    for (int64_t t = 0; t < a.nsteps; t++) {
        if (prof) tprev = clock64();
        const int64_t k0 = t * a.P;
        const int64_t k1 = min(k0 + a.P, a.ntot);
        const int Pt = (int)(k1 - k0);

        // ---------------- G: partial g/h of the CTA's rows for every bundle column ----------
        const int Rp = R | 1;   // odd tile stride: a warp's 32 columns hit 32 different banks
        const bool use_tile = (int64_t)Rp * Pt <= D_TILE;   // keep X_B's rows for phase X
        for (int pos = tid; pos < Pt; pos += NT) {
            float *tp = use_tile ? sm.tile + (int64_t)pos * Rp : nullptr;
            const int64_t cp = colinfo_p0(__ldg(&a.colinfo[k0 + pos])) + r0;
            const float *xp = a.val + cp;
            double g = 0.0, h = 0.0;
            // rows in order; 16-byte loads once the address is aligned (same sums, fewer requests)
            const int head = min(R, (int)((4 - (((uintptr_t)xp >> 2) & 3)) & 3));
            int r = 0;
            for (; r < head; r++) {
                const float xf = __ldg(xp + r);
                if (tp) tp[r] = xf;
                const double x = (double)xf;
                const double2 cf = sm.coef[r];
                g += x * cf.x;
                h += (x * x) * cf.y;
            }
#pragma unroll 4
            for (; r + 4 <= R; r += 4) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(xp + r));
                const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    if (tp) tp[r + e] = xv[e];
                    const double x = (double)xv[e];
                    const double2 cf = sm.coef[r + e];
                    g += x * cf.x;
                    h += (x * x) * cf.y;
                }
            }
            for (; r < R; r++) {
                const float xf = __ldg(xp + r);
                if (tp) tp[r] = xf;
                const double x = (double)xf;
                const double2 cf = sm.coef[r];
                g += x * cf.x;
                h += (x * x) * cf.y;
            }
            __stcg(reinterpret_cast<double2 *>(&part_gh[((int64_t)c * a.P + pos) * 2]), make_double2(g, h));
        }
        DPROF(0);
        sy.sync();
        DPROF(1);

        // ---------------- D: finish the columns owned by this CTA ---------------------------
        for (int pos = c + G * warp; pos < Pt; pos += G * NW) {
            double g = 0.0, h = 0.0;
            for (int c2 = lane; c2 < G; c2 += 32) {
                const double2 v = __ldcg(reinterpret_cast<const double2 *>(&part_gh[((int64_t)c2 * a.P + pos) * 2]));
                g += v.x;
                h += v.y;
            }
            g = warp_sum(g);
            h = warp_sum(h);
            if (lane == 0) {
                const int32_t j = __ldg(&a.order[k0 + pos]);
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
        sy.sync();
        DPROF(3);

        // ---------------- X: d'x of the CTA's rows in bundle order --------------------------
        int any = 0;
        for (int pos = tid; pos < Pt; pos += NT) {
            const double d = ldcg(&a.dk[pos]);
            if (pos < D_PMAX) {
                sm.dcol[pos] = d;
                sm.cp[pos] = colinfo_p0(__ldg(&a.colinfo[k0 + pos])) + r0;
            }
            any |= d != 0.0;
        }
        const bool dense_any = __syncthreads_or(any) != 0;
        if (dense_any) {
            const int C = R >= NT ? 1 : (int)min(NT / max(R, 1), Pt);
            for (int rb = 0; rb < R; rb += NT) {
                if (C == 1) {
                    const int r = rb + tid;
                    if (r < R) {
                        double x = 0.0;
                        for (int pos = 0; pos < Pt; pos++) {
                            const double d = pos < D_PMAX ? sm.dcol[pos] : ldcg(&a.dk[pos]);
                            const int64_t cp = pos < D_PMAX ? sm.cp[pos] : colinfo_p0(__ldg(&a.colinfo[k0 + pos])) + r0;
                            if (d != 0.0) x += d * (double)__ldg(&a.val[cp + r]);
                        }
                        sm.dx[r] = x;
                    }
                } else if (tid < R * C) {
                    const int r = tid % R, ch = tid / R;
                    const int e0 = (int)((int64_t)ch * Pt / C), e1 = (int)((int64_t)(ch + 1) * Pt / C);
                    // no branch on d_j == 0: its product is +-0 and leaves the sum unchanged, and
                    // branch-free iterations let the loads of several columns be in flight
                    double x = 0.0;
                    if (use_tile && e1 <= D_PMAX) {
#pragma unroll 8
                        for (int pos = e0; pos < e1; pos++) x += sm.dcol[pos] * (double)sm.tile[(int64_t)pos * Rp + r];
                    } else if (e1 <= D_PMAX) {
#pragma unroll 16
                        for (int pos = e0; pos < e1; pos++) x += sm.dcol[pos] * (double)__ldg(&a.val[sm.cp[pos] + r]);
                    } else {
                        for (int pos = e0; pos < e1; pos++) {
                            const double d = pos < D_PMAX ? sm.dcol[pos] : ldcg(&a.dk[pos]);
                            const int64_t cp = pos < D_PMAX ? sm.cp[pos] : colinfo_p0(__ldg(&a.colinfo[k0 + pos])) + r0;
                            x += d * (double)__ldg(&a.val[cp + r]);
                        }
                    }
                    sm.dpart[tid] = x;
                }
            }
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

        // ---------------- LS: Armijo windows (Eq.6 with Eq.12) ---------------------------------
        int q0 = 0, nq = prev_q <= 1 ? 2 : QW, qacc = -1, bad = 0;
        double alpha_acc = 0.0, lhs_acc = 0.0, rhs_acc = 0.0, Dl = 0.0;
        const int nown = max(0, (Pt - c + G - 1) / G);   // columns finished by this CTA
        while (true) {
            double alpha0 = 1.0;
            for (int q = 0; q < q0; q++) alpha0 *= a.beta;
            constexpr int W = WinLayout<QW>::W;   // 16 slots: Ls[0,6) L1[6,12) Delta
            double acc[W];
#pragma unroll
            for (int q = 0; q < W; q++) acc[q] = 0.0;
            if (dense_any) {
                for (int r = tid; r < R; r += NT) {
                    const double zi = sm.z[r], dxi = sm.dx[r];
                    const double cg = sm.coef[r].x;
                    const int yi = sm.y[r];
                    double al = alpha0;
                    for (int q = 0; q < nq; q++) {
#pragma unroll
                        for (int qq = 0; qq < QW; qq++)
                            if (qq == q) acc[qq] += loss_change(a.loss, zi, yi, cg, dxi, al);
                        al *= a.beta;
                    }
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
                    wj = ldcg(&a.w[__ldg(&a.order[k0 + pos])]);
                    d = ldcg(&a.dk[pos]);
                    dl = ldcg(&a.deltak[pos]);
                }
                double al = alpha0;
                for (int q = 0; q < nq; q++) {
#pragma unroll
                    for (int qq = 0; qq < QW; qq++)
                        if (qq == q) acc[QW + qq] += fabs(wj + al * d) - fabs(wj);
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
            double *part = part_ls + (int64_t)(wcount & 1) * G * NPART;
            if (warp == 0 && lane < W) {
                double s = 0.0;
#pragma unroll
                for (int w2 = 0; w2 < NW; w2++) s += sm.red[w2][lane];
                part[(int64_t)c * NPART + lane] = s;
            }
            DPROF(5);
            sy.sync();
            DPROF(6);
            grid_totals<W>(part, G, sm.red, sm.tot, lane, warp);
            if (warp == 0) {
                if (lane == 0) {
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
            }
            __syncthreads();
            qacc = sm.dec_q;
            bad = sm.dec_bad;
            alpha_acc = sm.dec_alpha;
            lhs_acc = sm.dec_lhs;
            rhs_acc = sm.dec_rhs;
            Dl = sm.dec_Delta;
            wcount++;
            __syncthreads();   // sm.dec_* / sm.red / sm.tot are reused
            if (qacc >= 0 || bad) break;
            q0 += nq;
            if (q0 > a.qmax) break;
            nq = QW;
        }
        if (qacc > a.qmax) qacc = -1;
        if (qacc < 0) alpha_acc = 0.0;
        prev_q = qacc < 0 ? QW : qacc;
        DPROF(7);

        // ---------------- commit (a5) ---------------------------------------------------------
        if (qacc >= 0 && dense_any) {
            for (int r = tid; r < R; r += NT) {
                const double zn = sm.z[r] + alpha_acc * sm.dx[r];
                sm.z[r] = zn;
                sm.coef[r] = coef_of(a.loss, zn, sm.y[r]);
            }
        }
        if (a.debug && dense_any) {
            for (int r = tid; r < R; r += NT) {
                a.dbg_dx[r0 + r] = sm.dx[r];
                a.dbg_mark[r0 + r] = 1;
            }
        }
        if (qacc >= 0) {
            for (int m = tid; m < nown; m += NT) {
                if (m < D_OWN) {
                    a.w[sm.oj[m]] = sm.ow[m] + alpha_acc * sm.od[m];
                } else {
                    const int pos = c + G * m;
                    const int32_t j = __ldg(&a.order[k0 + pos]);
                    a.w[j] = ldcg(&a.w[j]) + alpha_acc * ldcg(&a.dk[pos]);
                }
            }
        }
        if (c == 0 && tid == 0) {
            double F = sm.F;
            if (qacc >= 0) F = F + lhs_acc;
            sm.F = F;
            if (bad || t == a.nsteps - 1) {
                *a.F = F;
                if (bad) atomicMax(a.status, 3);
                a.info[0] = (double)qacc;
                a.info[1] = alpha_acc;
                a.info[2] = Dl;
                a.info[3] = lhs_acc;
                a.info[4] = rhs_acc;
                a.info[5] = F;
                a.info[7] = dense_any ? (double)a.s : 0.0;
            }
            const int64_t gstep = a.trace_off + t;
            if (gstep < a.trace_cap) {
                if (a.q_trace) a.q_trace[gstep] = qacc;
                if (a.F_trace) a.F_trace[gstep] = F;
            }
            sm.cnt[0] += 1;
            sm.cnt[1] += qacc < 0 ? 1 : 0;
            sm.cnt[2] += dense_any ? a.s : 0;
            sm.cnt[3] += Pt;
        }
        __syncthreads();
        if (bad) break;
    }
    // ---------------- epilogue: own rows back to HBM ----------------------------------------
    for (int r = tid; r < R; r += NT) {
        a.z[r0 + r] = sm.z[r];
        a.coef[r0 + r] = sm.coef[r];
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
