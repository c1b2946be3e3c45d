// pcdn_shard.cuh -- the sample-sharded bundle step.
//
// Each rank holds a row shard of X (its samples' CSC/CSR, z, y, cached factors); w and the
// partition stream are replicated.  One step is four phases, each a plain (non-persistent)
// kernel, with the cross-rank sums taken by the caller between them (host-driven collectives; the
// kernels never wait on another rank):
//   gh      local partial sums  sum_i x_ij G_i,  sum_i x_ij^2 H_i  per bundle position  -> [2P]
//           (caller: all-reduce, summed in rank order)
//   dir     d_j (Eq.5), Delta terms from the GLOBAL sums -- identical on every rank -- and the
//           (k, d_k x_ik) records of the local samples (per-sample CSR-offset segments)
//   ls      d'x_i of the local touched samples (records folded in ascending k) and the local loss
//           changes for a window of 6 candidates; rank 0 adds the L1 terms and Delta -> [13]
//           (caller: all-reduce, first q with LHS <= sigma alpha Delta)
//   commit  w_B += alpha d_B (every rank), z_T, factors of the local touched samples.
// Plain and deterministic (fixed reduction orders); not tuned: the single-GPU persistent kernels
// are the fast path, this one lets data larger than one GPU run with unchanged results.
#pragma once
#include "pcdn_kernels.cuh"

namespace pcdn {

constexpr int SH_NT = 256;
constexpr int SH_W = QW;     // candidates per line-search window
constexpr int SH_SHORT = 16; // records folded by one thread; longer lists by a warp (k_sh_ls_long)
constexpr int SH_LNT = 96;   // threads of k_sh_ls_long: 3 warps x an HB-record sort buffer (36 KB)

__global__ void k_sh_gh(StepArgs a, const int32_t *__restrict__ bundle, int64_t P, double *gh)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t kk = gw; kk < P; kk += nw) {
        const int32_t j = bundle[kk];
        double gs, hs;
        col_gh(a, a.col_ptr[j], a.col_ptr[j + 1], lane, gs, hs);
        if (lane == 0) {
            gh[2 * kk] = gs;
            gh[2 * kk + 1] = hs;
        }
    }
}

// d_j and the Delta term from the global sums, then the records of the local samples
__global__ void k_sh_dir(StepArgs a, const int32_t *__restrict__ bundle, int64_t P, const double *__restrict__ gh)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t kk = gw; kk < P; kk += nw) {
        const int32_t j = bundle[kk];
        const Dir r = finish_feature(a, gh[2 * kk], gh[2 * kk + 1], a.w[j]);
        if (lane == 0) {
            a.dk[kk] = r.d;
            a.deltak[kk] = r.delta;
        }
        if (r.d != 0.0) col_scatter(a, a.col_ptr[j], a.col_ptr[j + 1], lane, (int32_t)kk, r.d);
    }
}

// The records of sample i folded in ascending bundle position (any count: repeated minimum
// extraction over the segment, a plain O(n^2) walk)
__device__ __forceinline__ double sh_fold(const StepArgs &a, int64_t off, int ni)
{
    double dx = 0.0;
    int last = -1;
    for (int t = 0; t < ni; t++) {
        int best = 0x7fffffff;
        double bv = 0.0;
        for (int r = 0; r < ni; r++) {
            const double2 raw = __ldcg(reinterpret_cast<const double2 *>(&a.rec[off + r]));
            const int k = (int)(__double_as_longlong(raw.x) & 0xffffffffLL);
            if (k > last && k < best) {
                best = k;
                bv = raw.y;
            }
        }
        if (best == 0x7fffffff) atomicMax(a.status, 6);   // a repeated position: internal error
        last = best;
        dx += bv;
    }
    return dx;
}

// Loss changes of the local touched samples for candidates alpha_q = beta^(q0+q), q < SH_W, one
// partial row per block (threads in order, fixed trees).  first: fold d'x_i into dxg first.
__global__ void k_sh_ls(StepArgs a, int q0, int first, double *part)
{
    __shared__ double red[SH_W][SH_NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double alpha0 = 1.0;
    for (int q = 0; q < q0; q++) alpha0 *= a.beta;
    double acc[SH_W];
#pragma unroll
    for (int q = 0; q < SH_W; q++) acc[q] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.s; i += (int64_t)gridDim.x * blockDim.x) {
        const int ni = a.cnt[i];
        if (ni == 0 || ni > SH_SHORT) continue;   // long lists: k_sh_ls_long
        double dx;
        if (first) {
            dx = sh_fold(a, a.row_ptr[i], ni);
            a.dxg[i] = dx;
        } else {
            dx = a.dxg[i];
        }
        const double zi = a.z[i], cg = a.coef[i].x;
        const int yi = a.y[i];
        double al = alpha0;
#pragma unroll
        for (int q = 0; q < SH_W; q++) {
            acc[q] += loss_change(a.loss, zi, yi, cg, dx, al);
            al *= a.beta;
        }
    }
#pragma unroll
    for (int q = 0; q < SH_W; q++) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[q][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < SH_W) {
        double s = 0.0;
        for (int w2 = 0; w2 < SH_NT / 32; w2++) s += red[threadIdx.x][w2];
        part[(int64_t)blockIdx.x * SH_W + threadIdx.x] = s;
    }
}

// Samples with more than SH_SHORT records (dense rows): a warp each, bitonic sort by position in
// shared memory (fold_warp); their loss changes form further partial rows after k_sh_ls's.
__global__ void k_sh_ls_long(StepArgs a, int q0, int first, double *part)
{
    __shared__ int32_t sk[SH_LNT / 32][HB];
    __shared__ double sv[SH_LNT / 32][HB];
    __shared__ double red[SH_W][SH_LNT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double alpha0 = 1.0;
    for (int q = 0; q < q0; q++) alpha0 *= a.beta;
    double acc[SH_W];
#pragma unroll
    for (int q = 0; q < SH_W; q++) acc[q] = 0.0;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = gw; i < a.s; i += nw) {
        const int ni = a.cnt[i];
        if (ni <= SH_SHORT) continue;
        double dx;
        if (first) {
            dx = fold_warp(a, a.row_ptr[i], ni, sk[warp], sv[warp], lane);
            if (lane == 0) a.dxg[i] = dx;
        } else {
            dx = a.dxg[i];
        }
        if (lane == 0) {
            const double zi = a.z[i], cg = a.coef[i].x;
            const int yi = a.y[i];
            double al = alpha0;
#pragma unroll
            for (int q = 0; q < SH_W; q++) {
                acc[q] += loss_change(a.loss, zi, yi, cg, dx, al);
                al *= a.beta;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < SH_W; q++) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[q][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < SH_W) {
        double s = 0.0;
        for (int w2 = 0; w2 < SH_LNT / 32; w2++) s += red[threadIdx.x][w2];
        part[(int64_t)blockIdx.x * SH_W + threadIdx.x] = s;
    }
}

// out[0..6): the block rows summed in block order (local c-free loss changes); out[6..12): L1 +
// elastic terms of the bundle per candidate, out[12]: Delta -- only when with_l1 (one rank)
__global__ void k_sh_ls_final(StepArgs a, const int32_t *__restrict__ bundle, int64_t P, int q0, int nblocks,
                              const double *__restrict__ part, int with_l1, double *out)
{
    __shared__ double red[SH_W + 1][SH_NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < SH_W) {
        double s = 0.0;
        for (int b = 0; b < nblocks; b++) s += part[(int64_t)b * SH_W + threadIdx.x];
        out[threadIdx.x] = s;
    }
    double alpha0 = 1.0;
    for (int q = 0; q < q0; q++) alpha0 *= a.beta;
    double acc[SH_W + 1];
#pragma unroll
    for (int q = 0; q <= SH_W; q++) acc[q] = 0.0;
    if (with_l1) {
        for (int64_t kk = threadIdx.x; kk < P; kk += blockDim.x) {
            const double wj = a.w[bundle[kk]], d = a.dk[kk];
            double al = alpha0;
#pragma unroll
            for (int q = 0; q < SH_W; q++) {
                acc[q] += fabs(wj + al * d) - fabs(wj) + a.mu * al * d * (wj + 0.5 * al * d);
                al *= a.beta;
            }
            acc[SH_W] += a.deltak[kk];
        }
    }
#pragma unroll
    for (int q = 0; q <= SH_W; q++) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[q][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x <= SH_W) {
        double s = 0.0;
        for (int w2 = 0; w2 < (int)(blockDim.x >> 5); w2++) s += red[threadIdx.x][w2];
        out[SH_W + threadIdx.x] = s;
    }
}

// The Eq.6 decision of one window from the rank-summed totals tot[13] (tot[q]: c-free loss changes,
// tot[6+q]: separable terms, tot[12]: Delta) for candidates alpha = beta^(q0+q): the first q with
// LHS = tot[6+q] + c tot[q] <= sigma alpha Delta (alpha by repeated multiplication, reading Z11),
// candidates past q_max not taken (reading Z10).  dec[0] q (-1: none in this window), dec[1]
// next (1: run the window at q0 + 6), dec[2..6] alpha, LHS, RHS, Delta, the maintained F after
// the step.  Every rank holds the same totals, so every rank takes the same decision.
__global__ void k_sh_decide(StepArgs a, const double *__restrict__ tot, int q0, double *dec)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double Delta = tot[2 * SH_W];
    double al = 1.0;
    for (int q = 0; q < q0; q++) al *= a.beta;
    int qa = -1, bad = 0;
    double la = 0.0, ra = 0.0, alpha = 0.0;
    for (int q = 0; q < SH_W && q0 + q <= a.qmax; q++) {
        const double lhs = tot[SH_W + q] + a.c * tot[q];
        const double rhs = a.sigma * al * Delta;
        if (!isfinite(lhs) || !isfinite(Delta)) {
            bad = 1;
            break;
        }
        if (lhs <= rhs) {
            qa = q0 + q;
            alpha = al;
            la = lhs;
            ra = rhs;
            break;
        }
        al *= a.beta;
    }
    if (bad) atomicMax(a.status, 3);
    const double F = *a.F;
    dec[0] = (double)qa;
    dec[1] = (qa < 0 && !bad && q0 + SH_W <= a.qmax) ? 1.0 : 0.0;
    dec[2] = alpha;
    dec[3] = la;
    dec[4] = ra;
    dec[5] = Delta;
    dec[6] = qa >= 0 ? F + la : F;
}

// commit with the recorded decision (q < 0: a null step -- the records are only cleared) and the
// maintained F (reading Z23)
__global__ void k_sh_commit(StepArgs a, const int32_t *__restrict__ bundle, int64_t P, const double *__restrict__ dec)
{
    const double alpha = dec[0] >= 0.0 ? dec[2] : 0.0;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < a.s; i += nth) {
        if (a.cnt[i] == 0) continue;
        if (alpha != 0.0) {
            const double dx = a.dxg[i];
            const double zn = a.z[i] + alpha * dx;
            a.coef[i] = coef_next(a.loss, a.coef[i], zn, alpha * dx, a.y[i]);
            a.z[i] = zn;
        }
        a.cnt[i] = 0;
    }
    for (int64_t wi = tid; wi < (a.s + 31) / 32; wi += nth) a.bits[wi] = 0u;
    if (alpha != 0.0)
        for (int64_t kk = tid; kk < P; kk += nth) a.w[bundle[kk]] += alpha * a.dk[kk];
    if (tid == 0) *a.F = dec[6];
}

// F at an outer boundary: the rank-summed c sum_i phi_i plus the separable terms of the replicated
// w (||w||_1 + mu/2 ||w||^2, by k_obj_partial/k_obj_final over w alone into *F first)
__global__ void k_sh_add_loss(double *F, const double *__restrict__ loss_sum, double *F_copy)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const double v = loss_sum[0] + *F;
        *F = v;
        *F_copy = v;
    }
}

}  // namespace pcdn
