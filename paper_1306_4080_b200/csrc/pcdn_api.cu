// pcdn_api.cu -- C-ABI of the B200 PCDN hot path (declared in include/pcdn.h).
//
// Host side only marshals arguments, carves the caller's workspace and enqueues the kernels
// of pcdn_kernels.cuh on the context stream; every step of the path runs on the device.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/pcdn.h"
#include "pcdn_kernels.cuh"
#include "pcdn_resident.cuh"
#include "pcdn_dense.cuh"
#include "pcdn_shard.cuh"
#include "pcdn_sparse.cuh"

using namespace pcdn;

namespace {

constexpr int GMAX = 1024;
constexpr int DENSE_GMAX = 512;   // CTAs of the dense step kernel (<= 2 per SM on 148 SMs)
constexpr size_t ALIGN = 256;

inline size_t align_up(size_t x) { return (x + ALIGN - 1) & ~(ALIGN - 1); }

// chunk descriptors a list set can need: chunks hold >= SP_CHMIN nonzeros, one partial chunk per column
inline size_t chunk_capacity(int64_t n, int64_t nnz) { return (size_t)(nnz / SP_CHMIN + n + 1); }

// per-outer-iteration lists (partition, column descriptors, heavy / full column lists); two sets
// so that the lists of outer iteration k+1 can be built while the step kernel of k runs
struct Lists {
    size_t order, hdesc, flag, fflag, fpos, flist, tiles3, colinfo, hpos, hlist, hlen, hstart, tiles1, tiles2, nheavy;
    size_t lb, ticket;   // k_prep_lists: tile states (zeroed at create) and its ticket pair
    size_t cpos, cdesc, ccount;   // the sparse kernel's chunk lists (ccount: reference build only)
};

struct HostMirror {  // the readback block: device copy in the workspace, pinned host copy
    double F;
    double Fcopy;
    long long err_idx;
    int status;
    int err_what;
    int stop;   // set on the device at an outer boundary that ends the solve: later step launches exit
    unsigned ticket;   // k_obj's last-block ticket (zero between launches)
    int64_t counters[8];
    double info[8];
};

static_assert(sizeof(HostMirror) % 8 == 0, "k_obj copies the read-back block in 8-byte words");

struct Layout {
    size_t ydummy, w, z, coef, cnt, bits, rec, dxg, tlist, seen, dk, deltak, gk, hk, part, hpart, counters, info, F, Fcopy,
        status, err_idx, err_what, stop, ticket, mirror, bar, objp, prof, tl, dbg_dx, dbg_mark, rec2, rslot, ovf_cnt, part_gh,
        cslot, sbits, ccnt, dflag, cpart, total;
    Lists ls[2];
};

Layout make_layout(int64_t s, int64_t n, int64_t nnz)
{
    Layout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + (bytes ? bytes : 1));
        return o;
    };
    const int64_t nw = (s + 31) / 32;
    const int64_t ntile = (n + 1 + SCAN_TILE - 1) / SCAN_TILE + 1;
    L.ydummy = take(s);   // zero labels for the squared loss (which ignores them)
    L.w = take(sizeof(double) * n);
    L.z = take(sizeof(double) * s);
    L.coef = take(sizeof(double2) * s);
    L.cnt = take(sizeof(int32_t) * s);
    L.bits = take(sizeof(uint32_t) * nw);
    L.dxg = take(sizeof(double) * s);
    L.tlist = take(sizeof(int32_t) * nw * 32);
    // [z, tlist end) is the per-sample state the HBM-state kernels touch at random: one contiguous
    // window, kept L2-resident with a persisting access policy (launch_steps)
    L.rec = take(sizeof(Rec) * nnz);
    for (int b = 0; b < 2; b++) {
        Lists &S = L.ls[b];
        S.order = take(sizeof(int32_t) * n * (b == 0 ? 2 : 1));   // set 0: two partitions (dense solve)
        S.hdesc = take(sizeof(int4) * n);
        S.flag = take(sizeof(int32_t) * n);
        S.fflag = take(sizeof(int32_t) * n);
        S.fpos = take(sizeof(int64_t) * (n + 1));
        S.flist = take(sizeof(int32_t) * n);
        S.tiles3 = take(sizeof(int64_t) * ntile);
        S.colinfo = take(sizeof(int4) * n * (b == 0 ? 2 : 1));
        S.hpos = take(sizeof(int64_t) * (n + 1));
        S.hlist = take(sizeof(int32_t) * n);
        S.hlen = take(sizeof(int64_t) * n);
        S.hstart = take(sizeof(int64_t) * (n + 1));
        S.tiles1 = take(sizeof(int64_t) * ntile);
        S.tiles2 = take(sizeof(int64_t) * ntile);
        S.nheavy = take(sizeof(int64_t));
        S.lb = take(sizeof(LbTile) * (size_t)((n + PL_TILE - 1) / PL_TILE + 1));
        S.ticket = take(sizeof(unsigned) * 2);
        S.cpos = take(sizeof(int64_t) * (n + 1));
        S.cdesc = take(sizeof(int4) * chunk_capacity(n, nnz));
        S.ccount = take(sizeof(int32_t) * n);
    }
    L.seen = take(sizeof(uint32_t) * ((n + 31) / 32));
    L.dk = take(sizeof(double) * n);
    L.deltak = take(sizeof(double) * n);
    L.gk = take(sizeof(double) * 8);
    L.hk = take(sizeof(double) * 8);
    L.part = take(sizeof(double) * 2 * GMAX * NPART);
    L.hpart = take(sizeof(HPart) * GMAX * 2);
    // the readback scalars: one block laid out as HostMirror, copied to the host in one piece
    L.mirror = take(sizeof(HostMirror));
    L.F = L.mirror + offsetof(HostMirror, F);
    L.Fcopy = L.mirror + offsetof(HostMirror, Fcopy);
    L.status = L.mirror + offsetof(HostMirror, status);
    L.err_what = L.mirror + offsetof(HostMirror, err_what);
    L.err_idx = L.mirror + offsetof(HostMirror, err_idx);
    L.stop = L.mirror + offsetof(HostMirror, stop);
    L.ticket = L.mirror + offsetof(HostMirror, ticket);
    L.counters = L.mirror + offsetof(HostMirror, counters);
    L.info = L.mirror + offsetof(HostMirror, info);
    L.bar = take(sizeof(unsigned long long));
    L.objp = take(sizeof(double) * 3 * OBJ_NB);
    L.prof = take(sizeof(long long) * 16);
    L.tl = take(sizeof(long long) * TL_STEPS * NW * TL_PTS);
    L.dbg_dx = take(sizeof(double) * s);
    L.dbg_mark = take(s);
    L.rec2 = take(sizeof(Rec) * nnz);
    L.rslot = take(sizeof(uint32_t) * nnz);
    L.ovf_cnt = take(sizeof(int) * 16);
    // dense kernel (only when every column is full): partial (g, h) per CTA per bundle column
    L.part_gh = take(nnz == s * n ? sizeof(double) * 2 * (size_t)n * DENSE_GMAX : 0);
    // sparse kernel (pcdn_sparse.cuh): CSR offset of each CSC nonzero, the written-slot bitmap over
    // those offsets (its records live in `rec`, 8 B at each offset), heavy-column arrival counters,
    // stamped directions and chunk partials
    L.cslot = take(sizeof(uint32_t) * nnz);
    L.sbits = take(sizeof(uint32_t) * (nnz / 32 + 2));
    L.ccnt = take(sizeof(int) * n);
    L.dflag = take(sizeof(DFlag) * n);
    L.cpart = take(sizeof(double2) * chunk_capacity(n, nnz));
    L.total = off + ALIGN;  // slack for base alignment
    return L;
}

}  // namespace

struct pcdn_ctx {
    int64_t s = 0, n = 0, nnz = 0;
    const int64_t *col_ptr = nullptr;
    const int32_t *row_idx = nullptr;
    const float *val = nullptr;
    const int64_t *row_ptr = nullptr;
    const int32_t *col_idx = nullptr;
    const float *csr_val = nullptr;
    const int8_t *y = nullptr;
    const double *t = nullptr;   // squared-loss targets (pcdn_set_targets; borrowed device fp64[s])
    double c = 1.0;
    int loss = 0;
    double sigma = 0.01, beta = 0.5, gamma = 0.0, nu = 1e-12;
    double mu = 0.0;   // elastic-net weight (pcdn_set_elastic; reading Z25)
    int scdn = 0;      // pcdn_set_scdn (Alg.2, reading Z27)
    int qmax = 50;
    double fstar = 0.0;
    bool has_fstar = false;
    int debug = 0;
    int profile = 0;
    int G = 0;          // CTAs of the grid-mode step kernel (cooperative launch)
    int Gc = 0;         // CTAs of the cluster-mode step kernel (one cluster)
    int G_req = 0;
    int mode_req = 0;   // 0 auto, 1 cluster, 2 grid, 3 cluster-resident, 4 dense
    int Gd = 0;         // CTAs of the dense step kernel (0 = unavailable)
    int dense_tcap = 0; // floats per tile buffer of the dense step kernel
    size_t dsmem = 0;
    int res_G = 0;      // CTAs of the cluster-resident kernel (power of two; 0 = unavailable)
    int res_lg = 0, res_Bs = 0, res_cap = 0, res_cap_req = 0;
    size_t res_smem = 0;
    int last_mode = 0;
    int heavy_len = 0;     // user override (pcdn_set_launch); 0 = per launch mode (heavy_for_mode)
    int heavy_eff = 128;   // the value in force for the current solve / step (lists and kernels)
    int l2_want = 0;       // pcdn_set_l2_persist (off by default: a device-wide carve-out)
    size_t l2_persist = 0; // bytes of L2 set aside for the per-sample state window (0 = off)
    size_t l2_window = 0;  // max access-policy window size of the device
    int num_sms = 0;
    size_t smem = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;      // builds the next outer iteration's lists during a step launch
    cudaEvent_t ev_prep = nullptr;
    unsigned char *base = nullptr;
    Layout L{};
    HostMirror *hm = nullptr;   // [3]: hm[0] for single calls, hm[1..2] the solve's readback ring
    HostMirror *hm_dev = nullptr;   // device address of the mapped pinned hm
    bool solving = false;       // inside pcdn_solve: step launches honour the device stop flag
    bool bar_clean = false;     // the grid barrier was re-armed on the device (k_obj): no memset
    unsigned prep_epoch = 0;    // k_prep_lists launches (tile-state epoch)
    bool split_prep = false;    // test knob: build the lists with k_perm + scans + compactions
    bool dense_per_outer = false;   // test knob: the dense solve as one launch per outer iteration
    int dense_outers = 0;       // > 0: the dense launch runs up to this many outer iterations
    uint64_t cur_seed = 0;
    double cur_eps = 0.0;
    int32_t *q_trace = nullptr;
    double *F_trace = nullptr;
    int64_t trace_cap = 0;
    cudaEvent_t ev[10] = {};   // 0-3 single calls / solve span, 4-7 step spans (ring of 2), 8-9 readbacks
    int64_t launches = 0;
    unsigned long long stamp = 1;   // sparse kernel: step stamps handed out so far (never reused)
    char err[512] = {0};

    template <typename T>
    T *at(size_t off) const { return reinterpret_cast<T *>(base + off); }
};

namespace {

int set_err(pcdn_ctx *ctx, int code, const char *fmt, ...)
{
    if (ctx) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

#define CU(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return set_err(ctx, PCDN_ERR_CUDA, "%s failed: %s (%s:%d)", #call,                    \
                           cudaGetErrorString(e_), __FILE__, __LINE__);                           \
    } while (0)

inline int grid1d(int64_t work, int nt = 256)
{
    int64_t g = (work + nt - 1) / nt;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (int)g;
}

// device-wide exclusive scan of in[0..n) (n bounded by *n_dev if non-null) into out[0..n]
template <typename Tin>
int scan(pcdn_ctx *ctx, const Tin *in, int64_t n_host, const int64_t *n_dev, int64_t *out, int64_t *tiles,
         int64_t *total, cudaStream_t st)
{
    const int64_t ntile = (n_host + SCAN_TILE - 1) / SCAN_TILE > 0 ? (n_host + SCAN_TILE - 1) / SCAN_TILE : 1;
    k_scan_reduce<Tin, int64_t><<<(unsigned)ntile, SCAN_NT, 0, st>>>(in, n_host, n_dev, tiles);
    k_scan_tiles<int64_t><<<1, SCAN_NT, 0, st>>>(tiles, ntile);
    k_scan_apply<Tin, int64_t><<<(unsigned)ntile, SCAN_NT, 0, st>>>(in, n_host, n_dev, tiles, out, total);
    ctx->launches += 3;
    CU(cudaGetLastError());
    return PCDN_OK;
}

// heavy-column and full-column lists for the positions held in list set `buf` (order[0..ntot))
int build_heavy(pcdn_ctx *ctx, int64_t ntot, int buf, cudaStream_t st)
{
    const Lists &S = ctx->L.ls[buf];
    int rc = scan<int32_t>(ctx, ctx->at<int32_t>(S.flag), ntot, nullptr, ctx->at<int64_t>(S.hpos),
                           ctx->at<int64_t>(S.tiles1), ctx->at<int64_t>(S.nheavy), st);
    if (rc) return rc;
    k_heavy_compact<<<grid1d(ntot), 256, 0, st>>>(ctx->at<int64_t>(S.hpos), ntot, ctx->at<int32_t>(S.order),
                                                  ctx->col_ptr, ctx->at<int32_t>(S.hlist), ctx->at<int64_t>(S.hlen),
                                                  ctx->at<int4>(S.hdesc));
    ctx->launches++;
    CU(cudaGetLastError());
    rc = scan<int64_t>(ctx, ctx->at<int64_t>(S.hlen), ntot, ctx->at<int64_t>(S.nheavy), ctx->at<int64_t>(S.hstart),
                       ctx->at<int64_t>(S.tiles2), nullptr, st);
    if (rc) return rc;
    // full columns (a nonzero in every row): their d'x contribution is folded straight from CSC
    rc = scan<int32_t>(ctx, ctx->at<int32_t>(S.fflag), ntot, nullptr, ctx->at<int64_t>(S.fpos),
                       ctx->at<int64_t>(S.tiles3), nullptr, st);
    if (rc) return rc;
    k_full_compact<<<grid1d(ntot), 256, 0, st>>>(ctx->at<int64_t>(S.fpos), ntot, ctx->at<int32_t>(S.flist));
    ctx->launches++;
    CU(cudaGetLastError());
    // the sparse kernel's chunks: counts per position, their scan, the descriptors
    k_chunk_count<<<grid1d(ntot), 256, 0, st>>>(ctx->at<int4>(S.colinfo), ntot, ctx->heavy_eff,
                                                ctx->at<int32_t>(S.ccount));
    ctx->launches++;
    CU(cudaGetLastError());
    rc = scan<int32_t>(ctx, ctx->at<int32_t>(S.ccount), ntot, nullptr, ctx->at<int64_t>(S.cpos),
                       ctx->at<int64_t>(S.tiles3), nullptr, st);
    if (rc) return rc;
    k_chunk_compact<<<grid1d(ntot), 256, 0, st>>>(ctx->at<int64_t>(S.cpos), ctx->at<int64_t>(S.hpos),
                                                  ctx->at<int4>(S.colinfo), ntot, ctx->s, ctx->at<int4>(S.cdesc));
    ctx->launches++;
    CU(cudaGetLastError());
    return PCDN_OK;
}

// a0 for outer iteration k into list set `buf`: the partition pi_k and its lists, one launch
// (lists = false: the permutation and column descriptors only -- all the dense kernel reads)
int prep_outer(pcdn_ctx *ctx, uint64_t seed, int64_t k, int buf, cudaStream_t st, bool lists = true)
{
    const Lists &S = ctx->L.ls[buf];
    if (lists && !ctx->split_prep) {
        PrepLists o{};
        o.order = ctx->at<int32_t>(S.order);
        o.colinfo = ctx->at<int4>(S.colinfo);
        o.hpos = ctx->at<int64_t>(S.hpos);
        o.hstart = ctx->at<int64_t>(S.hstart);
        o.fpos = ctx->at<int64_t>(S.fpos);
        o.nheavy = ctx->at<int64_t>(S.nheavy);
        o.hlist = ctx->at<int32_t>(S.hlist);
        o.flist = ctx->at<int32_t>(S.flist);
        o.hdesc = ctx->at<int4>(S.hdesc);
        o.cpos = ctx->at<int64_t>(S.cpos);
        o.cdesc = ctx->at<int4>(S.cdesc);
        o.lb = ctx->at<LbTile>(S.lb);
        o.ticket = ctx->at<unsigned>(S.ticket);
        const int64_t ntiles = (ctx->n + PL_TILE - 1) / PL_TILE;
        ctx->prep_epoch = (ctx->prep_epoch + 1) & 0x3fffffffu;
        if (ctx->prep_epoch == 0) ctx->prep_epoch = 1;   // 0 is the zeroed workspace's state
        k_prep_lists<<<(unsigned)ntiles, PL_NT, 0, st>>>(seed, k, ctx->n, ctx->s, ctx->col_ptr, ctx->heavy_eff,
                                                         ctx->prep_epoch, o);
        ctx->launches++;
        CU(cudaGetLastError());
        return PCDN_OK;
    }
    k_perm<<<grid1d(ctx->n), 256, 0, st>>>(seed, k, ctx->n, ctx->s, ctx->col_ptr, ctx->heavy_eff,
                                           ctx->at<int32_t>(S.order), ctx->at<int32_t>(S.flag),
                                           ctx->at<int32_t>(S.fflag), ctx->at<int4>(S.colinfo));
    ctx->launches++;
    CU(cudaGetLastError());
    return lists ? build_heavy(ctx, ctx->n, buf, st) : PCDN_OK;
}

#define SCDN_HEAVY_MSG "SCDN: a bundle column is longer than the warp split length; raise it with pcdn_set_launch(ctx, 3, 0, L)"

// the squared loss has no state before its targets are given (pcdn_set_targets)
#define PCDN_NEED_TARGETS(ctx)                                                                             \
    do {                                                                                                   \
        if ((ctx)->loss == PCDN_LOSS_SQUARED && !(ctx)->t)                                                 \
            return set_err((ctx), PCDN_ERR_INVALID, "squared loss: call pcdn_set_targets first");        \
    } while (0)

// F from scratch into F and Fcopy (one k_obj launch; no stop test, no read-back copy)
int objective_kernels(pcdn_ctx *ctx)
{
    PCDN_NEED_TARGETS(ctx);
    const Layout &L = ctx->L;
    ObjBoundary o{};
    o.c = ctx->c;
    o.mu = ctx->mu;
    o.F = ctx->at<double>(L.F);
    o.F_copy = ctx->at<double>(L.Fcopy);
    o.status = ctx->at<int>(L.status);
    o.ticket = ctx->at<unsigned>(L.ticket);
    o.bar = ctx->at<unsigned long long>(L.bar);
    k_obj<<<OBJ_NB, OBJ_NB, 0, ctx->stream>>>(ctx->s, ctx->n, ctx->at<double>(L.z), ctx->y, ctx->at<double>(L.w),
                                              ctx->loss, ctx->at<double>(L.objp), ctx->t, o);
    ctx->launches++;
    CU(cudaGetLastError());
    return PCDN_OK;
}

int refresh_z(pcdn_ctx *ctx, int zero)
{
    PCDN_NEED_TARGETS(ctx);
    const Layout &L = ctx->L;
    k_set_z<<<grid1d(ctx->s), 256, 0, ctx->stream>>>(ctx->s, ctx->row_ptr, ctx->col_idx, ctx->csr_val, ctx->y,
                                                     ctx->at<double>(L.w), ctx->loss, ctx->at<double>(L.z),
                                                     ctx->at<double2>(L.coef), zero, ctx->t);
    ctx->launches++;
    CU(cudaGetLastError());
    return PCDN_OK;
}

int readback(pcdn_ctx *ctx)
{
    CU(cudaMemcpyAsync(ctx->hm, ctx->at<HostMirror>(ctx->L.mirror), sizeof(HostMirror), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return PCDN_OK;
}

int reset_status(pcdn_ctx *ctx)
{
    const Layout &L = ctx->L;
    // status, err_what, stop (contiguous in the mirror block) and err_idx
    CU(cudaMemsetAsync(ctx->at<int>(L.status), 0, 4 * sizeof(int), ctx->stream));
    CU(cudaMemsetAsync(ctx->at<long long>(L.err_idx), 0x7f, sizeof(long long), ctx->stream));
    return PCDN_OK;
}

// Launch the persistent step kernel over `nsteps` bundles of the positions in ctx->order.
int choose_mode(const pcdn_ctx *ctx, int64_t P);
int heavy_for_mode(const pcdn_ctx *ctx, int mode, int64_t P);

// the sparse HBM-state kernel (pcdn_sparse.cuh): one cluster (mode 1) or the cooperative grid (mode 2)
const void *sparse_kernel(bool cluster, int loss)
{
    if (cluster)
        return loss == LOSS_LOGISTIC ? (const void *)k_step_sparse<ClusterSync, LOSS_LOGISTIC>
               : loss == LOSS_L2SVM  ? (const void *)k_step_sparse<ClusterSync, LOSS_L2SVM>
                                     : (const void *)k_step_sparse<ClusterSync, LOSS_SQ>;
    return loss == LOSS_LOGISTIC ? (const void *)k_step_sparse<GridSync, LOSS_LOGISTIC>
           : loss == LOSS_L2SVM  ? (const void *)k_step_sparse<GridSync, LOSS_L2SVM>
                                 : (const void *)k_step_sparse<GridSync, LOSS_SQ>;
}

const void *dense_kernel(int loss)
{
    return loss == LOSS_LOGISTIC ? (const void *)k_step_dense<LOSS_LOGISTIC>
           : loss == LOSS_L2SVM  ? (const void *)k_step_dense<LOSS_L2SVM>
                                 : (const void *)k_step_dense<LOSS_SQ>;
}

int launch_steps(pcdn_ctx *ctx, int buf, int64_t ntot, int64_t P, int64_t nsteps, int64_t trace_off, double *g_out,
                 double *h_out, double *d_out)
{
    PCDN_NEED_TARGETS(ctx);
    const Layout &L = ctx->L;
    const Lists &S = L.ls[buf];
    StepArgs a{};
    a.s = ctx->s;
    a.n = ctx->n;
    a.col_ptr = ctx->col_ptr;
    a.row_idx = ctx->row_idx;
    a.val = ctx->val;
    a.row_ptr = ctx->row_ptr;
    a.y = ctx->y;
    a.t = ctx->t;
    a.scdn = ctx->scdn;
    a.c = ctx->c;
    a.sigma = ctx->sigma;
    a.beta = ctx->beta;
    a.gamma = ctx->gamma;
    a.nu = ctx->nu;
    a.mu = ctx->mu;
    a.loss = ctx->loss;
    a.qmax = ctx->qmax;
    a.heavy_len = ctx->heavy_eff;
    a.w = ctx->at<double>(L.w);
    a.z = ctx->at<double>(L.z);
    a.coef = ctx->at<double2>(L.coef);
    a.F = ctx->at<double>(L.F);
    a.cnt = ctx->at<int32_t>(L.cnt);
    a.bits = ctx->at<uint32_t>(L.bits);
    a.rec = ctx->at<Rec>(L.rec);
    a.dxg = ctx->at<double>(L.dxg);
    a.tlist = ctx->at<int32_t>(L.tlist);
    a.order = ctx->at<int32_t>(S.order);
    a.colinfo = ctx->at<int4>(S.colinfo);
    a.hpos = ctx->at<int64_t>(S.hpos);
    a.hlist = ctx->at<int32_t>(S.hlist);
    a.hdesc = ctx->at<int4>(S.hdesc);
    a.hstart = ctx->at<int64_t>(S.hstart);
    a.fpos = ctx->at<int64_t>(S.fpos);
    a.flist = ctx->at<int32_t>(S.flist);
    a.stop = ctx->solving ? ctx->at<int>(L.stop) : nullptr;
    a.ntot = ntot;
    a.P = P;
    a.nsteps = nsteps;
    a.dk = ctx->at<double>(L.dk);
    a.deltak = ctx->at<double>(L.deltak);
    a.part = ctx->at<double>(L.part);
    a.hpart = ctx->at<HPart>(L.hpart);
    a.g_out = g_out;
    a.h_out = h_out;
    a.d_out = d_out;
    a.q_trace = ctx->q_trace;
    a.F_trace = ctx->F_trace;
    a.trace_off = trace_off;
    a.trace_cap = ctx->trace_cap;
    a.counters = ctx->at<int64_t>(L.counters);
    a.info = ctx->at<double>(L.info);
    a.debug = ctx->debug;
    a.prof = ctx->profile == 1 ? ctx->at<long long>(L.prof) : nullptr;   // (the timeline mode runs unmarked)
    a.tl = ctx->profile == 2 ? ctx->at<long long>(L.tl) : nullptr;
    a.dbg_dx = ctx->at<double>(L.dbg_dx);
    a.dbg_mark = ctx->at<uint8_t>(L.dbg_mark);
    a.bar = ctx->at<unsigned long long>(L.bar);
    a.status = ctx->at<int>(L.status);
    a.res_lg = ctx->res_lg;
    a.res_Bs = ctx->res_Bs;
    a.res_cap = ctx->res_cap;
    {
        const ResLayout RL = res_layout(ctx->res_Bs > 0 ? ctx->res_Bs : 1, ctx->res_cap);
        a.res_off[0] = (int)RL.zd;
        a.res_off[1] = (int)RL.coef;
        a.res_off[2] = (int)RL.head;
        a.res_off[3] = (int)RL.lq;
        a.res_off[4] = (int)RL.y;
        a.res_off[5] = (int)RL.recin;
        a.res_off[6] = (int)RL.tl;
        a.res_off[7] = (int)RL.total;
    }
    a.rec2 = ctx->at<Rec>(L.rec2);
    a.rslot = ctx->at<uint32_t>(L.rslot);
    a.ovf_cnt = ctx->at<int>(L.ovf_cnt);
    a.part_gh = ctx->at<double>(L.part_gh);
    a.dense_tcap = ctx->dense_tcap;
    a.n_outer = ctx->dense_outers;
    a.outer0 = 0;
    a.seed = ctx->cur_seed;
    a.eps_stop = ctx->cur_eps;
    a.fstar = ctx->fstar;
    a.objp = ctx->at<double>(L.objp);
    a.pflag = ctx->at<int32_t>(L.ls[1].flag);
    a.pfflag = ctx->at<int32_t>(L.ls[1].fflag);
    a.outers_done = ctx->at<int64_t>(L.counters) + 5;
    a.cslot = ctx->at<uint32_t>(L.cslot);
    a.sbits = ctx->at<uint32_t>(L.sbits);
    a.rv = ctx->at<double>(L.rec);
    a.cdesc = ctx->at<int4>(S.cdesc);
    a.cpos = ctx->at<int64_t>(S.cpos);
    a.cpart = ctx->at<double2>(L.cpart);
    a.ccnt = ctx->at<int>(L.ccnt);
    a.dflag = ctx->at<DFlag>(L.dflag);
    a.stamp0 = ctx->stamp;
    ctx->stamp += (unsigned long long)nsteps + 1ull;
    if (!ctx->bar_clean) CU(cudaMemsetAsync(a.bar, 0, sizeof(unsigned long long), ctx->stream));
    ctx->bar_clean = false;
    // cluster mode for steps small enough that 16 SMs keep up (hardware barrier, ~0.2 us);
    // grid mode (all SMs, software barrier) for large steps
    const int mode = choose_mode(ctx, P);
    ctx->last_mode = mode;
    if (ctx->scdn && mode != 3)
        return set_err(ctx, PCDN_ERR_INVALID, "SCDN runs on the cluster-resident kernel (mode 3; samples must fit)");
    if (mode == 4) {
        if (ctx->Gd < 1) return set_err(ctx, PCDN_ERR_INVALID, "dense step kernel unavailable for this problem");
        void *args[] = {&a};
        const void *kd = dense_kernel(ctx->loss);
        CU(cudaLaunchCooperativeKernel(kd, dim3(ctx->Gd), dim3(NT), args, ctx->dsmem,
                                       ctx->stream));
    } else if (mode == 3) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(ctx->res_G);
        cfg.blockDim = dim3(NT);
        cfg.dynamicSmemBytes = ctx->res_smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = ctx->res_G;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        void *kargs[] = {&a};
        CU(cudaLaunchKernelExC(&cfg, res_kernel(ctx->loss, ctx->scdn != 0), kargs));
    } else {
        // HBM-state kernels: the per-sample state (z, coef, cnt, bits, dxg, tlist) is gathered and
        // scattered at random every step while CSC and records stream through L2; a persisting
        // access-policy window keeps the state resident
        cudaLaunchConfig_t cfg{};
        const bool sparse = mode != 5;
        cfg.gridDim = dim3(mode == 1 ? ctx->Gc : ctx->G);
        cfg.blockDim = dim3(sparse ? SNT : NT);
        cfg.dynamicSmemBytes = sparse ? sizeof(SpSmem) : ctx->smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (mode == 1) {
            at[na].id = cudaLaunchAttributeClusterDimension;
            at[na].val.clusterDim.x = ctx->Gc;
            at[na].val.clusterDim.y = 1;
            at[na].val.clusterDim.z = 1;
            na++;
        } else {
            at[na].id = cudaLaunchAttributeCooperative;
            at[na].val.cooperative = 1;
            na++;
        }
        // only for small steps: a large step streams records and CSC through L2, and the carve-out
        // then costs more than it saves (cfg5: -4% step time at P = 4096, +26% at P = 10^6)
        const bool small_step = (double)ctx->nnz * (double)P / (double)ctx->n <= 65536.0;
        if (ctx->l2_want && small_step && ctx->l2_persist == 0) {
            // first HBM-state launch: set aside L2 for the window (device limit, once)
            int dev = 0, maxp = 0, maxw = 0;
            CU(cudaGetDevice(&dev));
            CU(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
            CU(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev));
            const size_t want = std::min((size_t)maxp, L.rec - L.z);
            if (want > 0 && maxw > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
                ctx->l2_persist = want;
                ctx->l2_window = (size_t)maxw;
            } else {
                cudaGetLastError();
                ctx->l2_want = 0;
            }
        }
        if (ctx->l2_want && small_step && ctx->l2_persist > 0) {
            const size_t wbytes = std::min(L.rec - L.z, ctx->l2_window);
            at[na].id = cudaLaunchAttributeAccessPolicyWindow;
            at[na].val.accessPolicyWindow.base_ptr = (void *)(ctx->base + L.z);
            at[na].val.accessPolicyWindow.num_bytes = wbytes;
            at[na].val.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)ctx->l2_persist / (double)wbytes);
            at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            na++;
        }
        cfg.attrs = at;
        cfg.numAttrs = na;
        if (mode == 5) CU(cudaLaunchKernelEx(&cfg, k_step<GridSync>, a));
        else {
            void *kargs[] = {&a};
            CU(cudaLaunchKernelExC(&cfg, sparse_kernel(mode == 1, ctx->loss), kargs));
        }
    }
    ctx->launches++;
    return PCDN_OK;
}

// launch mode of the step kernel for bundles of size P (see pcdn_set_launch)
// Columns longer than this are "heavy": the sparse kernel (modes 1, 2) reduces them in chunks of
// about this many nonzeros over several warps; the legacy grid kernel (mode 5) splits them
// nnz-balanced over every warp of the launch and reduces shorter ones of up to CTA_LEN inside one
// CTA; the cluster-resident kernel splits everything above a warp's 128.
int heavy_for_mode(const pcdn_ctx *ctx, int mode, int64_t P)
{
    if (ctx->heavy_len > 0) return ctx->heavy_len;
    if (mode == 2) {
        // Sparse grid kernel: when a step gives a CTA only a few columns, most of its 12 warps have
        // none of their own, and a column of 65-256 nonzeros is reduced sooner as CTA chunks (all
        // warps on one) than by one warp; with more work per CTA the chunks' CTA barriers cost more
        // than they save.  B200 (profiles/r2d/heavy_len/, profiles/r2e/knobs/), us per step at
        // heavy_len 64 / 128 / 256: config 5 P = 4096 (111 bundle nonzeros per CTA) 19.43 / 19.68 /
        // 20.38, P = 8192 (221) 22.65 / - / 23.82, P = 16,384 (443) - / 27.45 / 28.48, P = 29,500 (797)
        // 39.1 / 35.3 / 34.9, P = 1e5 94.4 / 83.6 / 80.9; config 3 P = 8192 (498) 33.9 / 31.05 / 32.4;
        // one cluster (mode 1), config 5 P = 1024: 17.75 / - / 17.34.
        const double per_cta = (double)ctx->nnz * (double)P / (double)ctx->n / (double)(ctx->G > 0 ? ctx->G : 1);
        return per_cta <= 256.0 ? 64 : per_cta <= 640.0 ? 128 : SP_CH;
    }
    if (mode == 1) return SP_CH;
    // cluster-resident kernel: config 3 (P = 1024) 18.98 / 18.88 / 19.34 / 20.75 us per step at 64 / 96 /
    // 128 / 192; config 2 has no column that long (6.75 us at any setting)
    return mode == 5 ? CTA_LEN : mode == 3 ? 96 : MED_LEN;
}

int choose_mode(const pcdn_ctx *ctx, int64_t P)
{
    int mode = ctx->mode_req;
    if (mode == 0 && ctx->Gd > 0) mode = 4;   // fully dense problem: row-block kernel
    if (mode == 0) {
        // cluster-resident when the samples fit the cluster's shared memory and the bundles are
        // small; else the HBM-state kernel as one cluster only while each of its warps has few
        // columns per step (they are processed one after another), otherwise over the whole grid
        const double est_nb = (double)ctx->nnz * (double)P / (double)ctx->n;
        if (ctx->res_G >= 2 && est_nb <= 65536.0) mode = 3;
        else mode = (ctx->Gc >= 2 && est_nb <= 16384.0 && P <= 2 * NW * ctx->Gc) ? 1 : 2;
    }
    // the sparse kernel addresses CSR offsets in 32 bits
    if ((mode == 1 || mode == 2) && ctx->nnz >= (int64_t)UINT32_MAX) mode = 5;
    return mode;
}

// The side stream that builds the next outer iteration's lists beside the cluster-resident kernel.
// Streams come from a per-device pool of SIDE_POOL, handed out round-robin to contexts (creating a
// stream per context cost ~0.2-0.8 ms in the one-call host API); a context orders its own work on
// its side stream with events, so contexts on different pool streams overlap independently (up to
// SIDE_POOL concurrently active contexts per device; beyond that two contexts share a stream and
// their list builds queue behind each other -- results are unchanged).
// set by pcdn_train_host around its pcdn_create call when it built the CSR from the CSC itself
static thread_local bool g_csr_trusted = false;

static cudaStream_t shared_side_stream()
{
    constexpr int SIDE_POOL = 8;
    static std::mutex mu;
    static cudaStream_t streams[64][SIDE_POOL] = {};
    static bool tried[64][SIDE_POOL] = {};
    static unsigned next[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return nullptr;
    }
    std::lock_guard<std::mutex> lock(mu);
    const unsigned k = next[dev]++ % SIDE_POOL;
    if (!tried[dev][k]) {
        tried[dev][k] = true;
        if (cudaStreamCreateWithFlags(&streams[dev][k], cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            streams[dev][k] = nullptr;
        }
    }
    return streams[dev][k];
}

// Load every kernel of the library once per process.  Under CUDA's default lazy module loading
// each kernel is loaded at its first use, and the one-call host API (which creates a context per
// call) was measured to pay ~8 ms per call more than with eager loading (scripts/_create_time.py).
static void preload_kernels()
{
    static bool done = false;
    if (done) return;
    done = true;
    const void *fns[] = {
        (const void *)k_perm, (const void *)k_full_compact, (const void *)k_bundle_prep, (const void *)k_bundle_unseen,
        (const void *)k_scan_reduce<int32_t, int64_t>, (const void *)k_scan_reduce<int64_t, int64_t>,
        (const void *)k_scan_apply<int32_t, int64_t>, (const void *)k_scan_apply<int64_t, int64_t>,
        (const void *)k_scan_tiles<int64_t>, (const void *)k_heavy_compact, (const void *)k_step<GridSync>,
        sparse_kernel(true, LOSS_LOGISTIC), sparse_kernel(true, LOSS_L2SVM), sparse_kernel(true, LOSS_SQ),
        sparse_kernel(false, LOSS_LOGISTIC), sparse_kernel(false, LOSS_L2SVM), sparse_kernel(false, LOSS_SQ),
        (const void *)k_chunk_count, (const void *)k_chunk_compact, res_kernel(LOSS_LOGISTIC, false), res_kernel(LOSS_L2SVM, false),
        res_kernel(LOSS_SQ, false), res_kernel(LOSS_LOGISTIC, true), res_kernel(LOSS_L2SVM, true),
        res_kernel(LOSS_SQ, true), dense_kernel(LOSS_LOGISTIC), dense_kernel(LOSS_L2SVM), dense_kernel(LOSS_SQ),
        (const void *)k_set_z, (const void *)k_obj_partial, (const void *)k_obj_final, (const void *)k_obj, (const void *)k_prep_lists, (const void *)k_solve_init, (const void *)k_validate,
        (const void *)k_validate_transpose, (const void *)k_check_finite, (const void *)k_sh_gh, (const void *)k_sh_dir,
        (const void *)k_sh_ls, (const void *)k_sh_ls_long, (const void *)k_sh_ls_final, (const void *)k_sh_commit,
        (const void *)k_sh_decide, (const void *)k_sh_add_loss};
    for (const void *f : fns) {
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) cudaGetLastError();
    }
}

int configure_launch(pcdn_ctx *ctx)
{
    preload_kernels();
    int dev = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev));
    int coop = 0;
    CU(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    if (!coop) return set_err(ctx, PCDN_ERR_CUDA, "device does not support cooperative launch");
    ctx->smem = sizeof(StepSmem);
    const void *kg = (const void *)k_step<GridSync>;
    const void *kc = sparse_kernel(true, ctx->loss);
    const void *ks = sparse_kernel(false, ctx->loss);
    CU(cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->smem));
    CU(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SpSmem)));
    CU(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SpSmem)));
    CU(cudaFuncSetAttribute(kc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int occ = 0, occs = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kg, NT, ctx->smem));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs, ks, SNT, sizeof(SpSmem)));
    if (occs < occ) occ = occs;   // one grid size serves both grid kernels
    if (occ < 1) return set_err(ctx, PCDN_ERR_CUDA, "step kernel cannot be resident (smem %zu)", ctx->smem);
    int maxg = ctx->num_sms * occ;
    if (maxg > GMAX) maxg = GMAX;
    // largest cluster the device can co-schedule with this footprint (<= 16, non-portable)
    int maxc = 0;
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(SNT);
        cfg.dynamicSmemBytes = sizeof(SpSmem);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxPotentialClusterSize(&maxc, kc, &cfg) != cudaSuccess) {
            cudaGetLastError();
            maxc = 0;
        }
        if (maxc > 16) maxc = 16;
    }
    // cluster-resident kernel: the largest power-of-two cluster whose CTAs hold ceil(s/G)
    // samples plus a record buffer of >= 256 records in shared memory
    {
        int optin = 0;
        CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        const void *kr = res_kernel(ctx->loss, false);
        const void *krs = res_kernel(ctx->loss, true);   // the SCDN instantiation: same layout
        CU(cudaFuncSetAttribute(kr, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CU(cudaFuncSetAttribute(krs, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        ctx->res_G = 0;
        const int greq = ctx->mode_req == 3 ? ctx->G_req : 0;
        for (int lg = 4; lg >= 0; lg--) {
            const int G = 1 << lg;
            if (greq > 0 && G != greq) continue;
            const int64_t Bs = (ctx->s + G - 1) / G;
            if (Bs > 32 * NT) continue;   // <= 32 owned samples per thread
            const ResLayout L0 = res_layout((int)Bs, 0);
            if ((int64_t)L0.total + 64 > optin) continue;
            int cap = (int)(((int64_t)optin - (int64_t)L0.total - 64) / (int64_t)R_BYTES_PER_RECORD);
            if (ctx->res_cap_req > 0 && ctx->res_cap_req < cap) cap = ctx->res_cap_req;
            while (cap > 0 && res_layout((int)Bs, cap).total > (size_t)optin) cap--;
            if (cap < (ctx->res_cap_req > 0 ? 1 : 256)) continue;
            const size_t sm = res_layout((int)Bs, cap).total;
            CU(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            CU(cudaFuncSetAttribute(krs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(NT);
            cfg.dynamicSmemBytes = sm;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = G;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclu = 0;
            if (cudaOccupancyMaxActiveClusters(&nclu, kr, &cfg) != cudaSuccess) {
                cudaGetLastError();
                nclu = 0;
            }
            if (nclu < 1) continue;
            ctx->res_G = G;
            ctx->res_lg = lg;
            ctx->res_Bs = (int)Bs;
            ctx->res_cap = cap;
            ctx->res_smem = sm;
            break;
        }
        if (ctx->mode_req == 3 && ctx->res_G < 1)
            return set_err(ctx, PCDN_ERR_INVALID, "cluster-resident mode unavailable for s=%lld", (long long)ctx->s);
    }
    // dense row-block kernel: every column full, rows per CTA and bundle sizes within its smem
    {
        ctx->Gd = 0;
        if (ctx->nnz == ctx->s * ctx->n) {
            int optin = 0;
            CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            // the fixed part plus two tile buffers (the step's X_B rows, copied a step ahead)
            ctx->dsmem = (size_t)optin;
            ctx->dense_tcap = (int)((((size_t)optin - dense_fixed_bytes()) / (2 * sizeof(float))) & ~(size_t)31);
            const void *kd = dense_kernel(ctx->loss);
            CU(cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->dsmem));
            int occd = 0;
            CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occd, kd, NT, ctx->dsmem));
            int gd = ctx->num_sms * occd;
            if (ctx->mode_req == 4 && ctx->G_req > 0 && ctx->G_req < gd) gd = ctx->G_req;
            if (gd > DENSE_GMAX) gd = DENSE_GMAX;
            if (gd > GMAX) gd = GMAX;
            if (gd >= 1 && (ctx->s + gd - 1) / gd + 3 <= D_RMAX) ctx->Gd = gd;   // + 3: 4-row aligned blocks
        }
        if (ctx->mode_req == 4 && ctx->Gd < 1)
            return set_err(ctx, PCDN_ERR_INVALID, "dense mode needs every column full and <= %d rows per CTA", D_RMAX);
    }
    const bool want_cluster = ctx->mode_req == 1;
    ctx->G = (!want_cluster && ctx->G_req > 0 && ctx->G_req < maxg) ? ctx->G_req : maxg;
    ctx->Gc = (want_cluster && ctx->G_req > 0 && ctx->G_req < maxc) ? ctx->G_req : maxc;
    if (ctx->mode_req == 1 && ctx->Gc < 1)
        return set_err(ctx, PCDN_ERR_INVALID, "cluster mode unavailable (max cluster size %d)", maxc);
    return PCDN_OK;
}

}  // namespace

extern "C" {

const char *pcdn_version(void) { return "pcdn-b200 0.1 (sm_100a)"; }

size_t pcdn_workspace_bytes(int64_t s, int64_t n, int64_t nnz)
{
    if (s < 1 || n < 1 || nnz < 0) return 0;
    return make_layout(s, n, nnz).total;
}

int pcdn_create(int64_t s, int64_t n, int64_t nnz, const int64_t *csc_col_ptr, const int32_t *csc_row_idx,
                const float *csc_val, const int64_t *csr_row_ptr, const int32_t *csr_col_idx, const float *csr_val,
                const int8_t *y, double c, int loss, void *workspace, size_t workspace_bytes, void *cuda_stream,
                pcdn_ctx **out)
{
    if (!out) return PCDN_ERR_INVALID;
    *out = nullptr;
    pcdn_ctx *ctx = new (std::nothrow) pcdn_ctx();
    if (!ctx) return PCDN_ERR_NOMEM;
    auto fail = [&](int code) {
        // keep ctx alive so the caller can read the error; caller must destroy it
        *out = ctx;
        return code;
    };
    if (s < 1 || n < 1 || nnz < 0 || s > INT32_MAX || n > INT32_MAX)
        return fail(set_err(ctx, PCDN_ERR_INVALID, "invalid sizes s=%lld n=%lld nnz=%lld", (long long)s,
                            (long long)n, (long long)nnz));
    if (!(c > 0) || !std::isfinite(c)) return fail(set_err(ctx, PCDN_ERR_INVALID, "c must be finite and > 0"));
    if (loss != PCDN_LOSS_LOGISTIC && loss != PCDN_LOSS_L2SVM && loss != PCDN_LOSS_SQUARED)
        return fail(set_err(ctx, PCDN_ERR_INVALID, "unknown loss %d", loss));
    if (!csc_col_ptr || !csr_row_ptr || (!y && loss != PCDN_LOSS_SQUARED) ||
        (nnz > 0 && (!csc_row_idx || !csc_val || !csr_col_idx || !csr_val)))
        return fail(set_err(ctx, PCDN_ERR_INVALID, "null input pointer"));
    ctx->L = make_layout(s, n, nnz);
    if (!workspace || workspace_bytes < ctx->L.total)
        return fail(set_err(ctx, PCDN_ERR_NOMEM, "workspace too small: need %zu bytes, got %zu", ctx->L.total,
                            workspace_bytes));
    ctx->s = s;
    ctx->n = n;
    ctx->nnz = nnz;
    ctx->col_ptr = csc_col_ptr;
    ctx->row_idx = csc_row_idx;
    ctx->val = csc_val;
    ctx->row_ptr = csr_row_ptr;
    ctx->col_idx = csr_col_idx;
    ctx->csr_val = csr_val;
    // the squared loss ignores labels: a zeroed workspace array stands in when none is given
    ctx->y = (loss == PCDN_LOSS_SQUARED && !y) ? ctx->at<int8_t>(ctx->L.ydummy) : y;
    ctx->c = c;
    ctx->loss = loss;
    ctx->stream = (cudaStream_t)cuda_stream;
    ctx->base = reinterpret_cast<unsigned char *>(align_up(reinterpret_cast<uintptr_t>(workspace)));
    {
        cudaError_t e = cudaHostAlloc(&ctx->hm, 3 * sizeof(HostMirror), cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess) return fail(set_err(ctx, PCDN_ERR_CUDA, "cudaHostAlloc: %s", cudaGetErrorString(e)));
        e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&ctx->hm_dev), ctx->hm, 0);
        if (e != cudaSuccess)
            return fail(set_err(ctx, PCDN_ERR_CUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e)));
        for (int i = 0; i < 10; i++) {
            e = cudaEventCreate(&ctx->ev[i]);
            if (e != cudaSuccess) return fail(set_err(ctx, PCDN_ERR_CUDA, "cudaEventCreate: %s", cudaGetErrorString(e)));
        }
        ctx->side = shared_side_stream();
        if (!ctx->side || cudaEventCreateWithFlags(&ctx->ev_prep, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();   // no overlap: lists are built on the context stream
            ctx->side = nullptr;
            ctx->ev_prep = nullptr;
        }
    }
    int rc = configure_launch(ctx);
    if (rc) return fail(rc);
    // zero the whole workspace once (counters, bitmaps, record counts must start at 0)
    {
        cudaError_t e = cudaMemsetAsync(ctx->base, 0, ctx->L.total - ALIGN, ctx->stream);
        if (e != cudaSuccess) return fail(set_err(ctx, PCDN_ERR_CUDA, "memset: %s", cudaGetErrorString(e)));
    }
    if ((rc = reset_status(ctx))) return fail(rc);
    const Layout &L = ctx->L;
    k_validate<<<grid1d(std::max(nnz, s > n ? s : n)), 256, 0, ctx->stream>>>(s, n, nnz, csc_col_ptr, csc_row_idx, csc_val,
                                                               csr_row_ptr, csr_col_idx, csr_val,
                                                               loss == PCDN_LOSS_SQUARED ? nullptr : y,
                                                               ctx->at<int>(L.status), ctx->at<long long>(L.err_idx),
                                                               ctx->at<int>(L.err_what));
    // the CSR/CSC consistency check and the sparse kernel's CSC -> CSR offset map (values not
    // compared for a CSR the library built itself from this CSC: pcdn_train_host with csr_* = NULL)
    k_validate_transpose<<<grid1d(s * 32), 256, 0, ctx->stream>>>(s, csc_col_ptr, csc_row_idx, csc_val, csr_row_ptr,
                                                                   csr_col_idx, csr_val, g_csr_trusted ? 0 : 1,
                                                                   ctx->at<uint32_t>(L.cslot), ctx->at<int>(L.status),
                                                                   ctx->at<long long>(L.err_idx), ctx->at<int>(L.err_what));
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(set_err(ctx, PCDN_ERR_CUDA, "validate launch: %s", cudaGetErrorString(e)));
    }
    if ((rc = readback(ctx))) return fail(rc);
    if (ctx->hm->status) {
        static const char *what[] = {"?", "col_ptr[0] != 0", "col_ptr[n] != nnz", "col_ptr not monotone",
                                     "row index out of range", "row indices not strictly increasing in a column",
                                     "non-finite CSC value", "row_ptr[0] != 0", "row_ptr[s] != nnz",
                                     "row_ptr not monotone", "CSR column index out of range",
                                     "CSR column indices not strictly increasing in a row", "non-finite CSR value",
                                     "label not in {-1,+1}", "CSR and CSC hold different nonzeros"};
        const int wv = ctx->hm->err_what >= 0 && ctx->hm->err_what <= 14 ? ctx->hm->err_what : 0;
        return fail(set_err(ctx, PCDN_ERR_INVALID, "invalid input: %s at index %lld", what[wv],
                            (long long)ctx->hm->err_idx));
    }
    // the squared loss gets its state (z, coef, F) once its targets arrive (pcdn_set_targets)
    if (loss != PCDN_LOSS_SQUARED && (rc = pcdn_reset(ctx))) return fail(rc);
    *out = ctx;
    return PCDN_OK;
}

int pcdn_set_armijo(pcdn_ctx *ctx, double sigma, double beta, double gamma, int q_max)
{
    if (!ctx) return PCDN_ERR_INVALID;
    if (!(sigma > 0 && sigma < 1) || !(beta > 0 && beta < 1) || !(gamma >= 0 && gamma < 1) || q_max < 0 || q_max > 200)
        return set_err(ctx, PCDN_ERR_INVALID, "invalid Armijo constants");
    ctx->sigma = sigma;
    ctx->beta = beta;
    ctx->gamma = gamma;
    ctx->qmax = q_max;
    return PCDN_OK;
}

int pcdn_set_targets(pcdn_ctx *ctx, const double *t)
{
    if (!ctx) return PCDN_ERR_INVALID;
    if (ctx->loss != PCDN_LOSS_SQUARED) return set_err(ctx, PCDN_ERR_INVALID, "targets belong to the squared loss");
    if (!t) return set_err(ctx, PCDN_ERR_INVALID, "null targets");
    int rc;
    if ((rc = reset_status(ctx))) return rc;
    k_check_finite<<<grid1d(ctx->s), 256, 0, ctx->stream>>>(t, ctx->s, ctx->at<int>(ctx->L.status),
                                                            ctx->at<long long>(ctx->L.err_idx));
    ctx->launches++;
    CU(cudaGetLastError());
    if ((rc = readback(ctx))) return rc;
    if (ctx->hm->status)
        return set_err(ctx, PCDN_ERR_INVALID, "non-finite target at index %lld", (long long)ctx->hm->err_idx);
    ctx->t = t;
    return pcdn_reset(ctx);   // w = 0, z, coef = (2(z - t), 2), F
}

int pcdn_set_scdn(pcdn_ctx *ctx, int on)
{
    if (!ctx) return PCDN_ERR_INVALID;
    ctx->scdn = on ? 1 : 0;
    return PCDN_OK;
}

int pcdn_set_elastic(pcdn_ctx *ctx, double mu)
{
    if (!ctx) return PCDN_ERR_INVALID;
    if (!(mu >= 0) || !std::isfinite(mu)) return set_err(ctx, PCDN_ERR_INVALID, "elastic-net weight must be finite and >= 0");
    ctx->mu = mu;
    return objective_kernels(ctx);   // the maintained F now includes (mu/2)||w||^2
}

int pcdn_set_reference(pcdn_ctx *ctx, double f_star)
{
    if (!ctx) return PCDN_ERR_INVALID;
    if (!(f_star > 0) || !std::isfinite(f_star)) return set_err(ctx, PCDN_ERR_INVALID, "F* must be finite and > 0");
    ctx->fstar = f_star;
    ctx->has_fstar = true;
    return PCDN_OK;
}

int pcdn_set_trace(pcdn_ctx *ctx, int32_t *q_trace, double *F_trace, int64_t capacity)
{
    if (!ctx) return PCDN_ERR_INVALID;
    ctx->q_trace = q_trace;
    ctx->F_trace = F_trace;
    ctx->trace_cap = capacity > 0 ? capacity : 0;
    return PCDN_OK;
}

int pcdn_set_debug(pcdn_ctx *ctx, int on)
{
    if (!ctx) return PCDN_ERR_INVALID;
    ctx->debug = (on & 1) ? 1 : 0;
    ctx->split_prep = (on & 2) != 0;
    ctx->dense_per_outer = (on & 4) != 0;
    return PCDN_OK;
}

int pcdn_set_launch(pcdn_ctx *ctx, int mode, int ctas, int heavy_len)
{
    if (!ctx) return PCDN_ERR_INVALID;
    if (mode < 0 || mode > 5 || ctas < 0 || heavy_len < 0 || (mode == 1 && ctas > 16) ||
        (mode == 3 && (ctas > 16 || (ctas & (ctas - 1)) != 0)))
        return set_err(ctx, PCDN_ERR_INVALID, "invalid launch knobs");
    ctx->mode_req = mode;
    ctx->G_req = ctas;
    if (heavy_len > 0) ctx->heavy_len = heavy_len;
    return configure_launch(ctx);
}

int pcdn_set_l2_persist(pcdn_ctx *ctx, int on)
{
    if (!ctx) return PCDN_ERR_INVALID;
    ctx->l2_want = on ? 1 : 0;
    if (on && ctx->l2_persist == 0) ctx->l2_want = 1;
    return PCDN_OK;
}

int pcdn_set_resident_cap(pcdn_ctx *ctx, int cap)
{
    if (!ctx) return PCDN_ERR_INVALID;
    if (cap < 0) return set_err(ctx, PCDN_ERR_INVALID, "negative record capacity");
    ctx->res_cap_req = cap;
    return configure_launch(ctx);
}

int pcdn_set_profile(pcdn_ctx *ctx, int on)
{
    if (!ctx) return PCDN_ERR_INVALID;
    ctx->profile = on == 2 ? 2 : (on ? 1 : 0);
    CU(cudaMemsetAsync(ctx->at<long long>(ctx->L.prof), 0, sizeof(long long) * 16, ctx->stream));
    CU(cudaMemsetAsync(ctx->at<long long>(ctx->L.tl), 0, sizeof(long long) * TL_STEPS * NW * TL_PTS, ctx->stream));
    return PCDN_OK;
}

int pcdn_warp_timeline(pcdn_ctx *ctx, int64_t *out)
{
    if (!ctx || !out) return PCDN_ERR_INVALID;
    CU(cudaMemcpyAsync(out, ctx->at<long long>(ctx->L.tl), sizeof(long long) * TL_STEPS * NW * TL_PTS,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return PCDN_OK;
}

int pcdn_phase_cycles(pcdn_ctx *ctx, int64_t *out, int32_t *mode)
{
    if (!ctx || !out) return PCDN_ERR_INVALID;
    CU(cudaMemcpyAsync(out, ctx->at<long long>(ctx->L.prof), sizeof(long long) * 16, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (mode) *mode = ctx->last_mode;
    return PCDN_OK;
}

const char *pcdn_last_error(const pcdn_ctx *ctx) { return ctx ? ctx->err : "null context"; }

void pcdn_destroy(pcdn_ctx *ctx)
{
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    // the side stream is shared by the process's contexts: wait for this context's work on it only
    if (ctx->ev_prep) {
        cudaEventSynchronize(ctx->ev_prep);
        cudaEventDestroy(ctx->ev_prep);
    }
    if (ctx->hm) cudaFreeHost(ctx->hm);
    delete ctx;
}

int pcdn_reset(pcdn_ctx *ctx)
{
    if (!ctx || !ctx->base) return PCDN_ERR_INVALID;
    const Layout &L = ctx->L;
    CU(cudaMemsetAsync(ctx->at<double>(L.w), 0, sizeof(double) * ctx->n, ctx->stream));
    int rc = refresh_z(ctx, 1);
    if (rc) return rc;
    return objective_kernels(ctx);
}

int pcdn_set_w(pcdn_ctx *ctx, const double *w)
{
    if (!ctx || !w) return PCDN_ERR_INVALID;
    const Layout &L = ctx->L;
    CU(cudaMemcpyAsync(ctx->at<double>(L.w), w, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, ctx->stream));
    int rc = refresh_z(ctx, 0);
    if (rc) return rc;
    return objective_kernels(ctx);
}

int pcdn_get_w(pcdn_ctx *ctx, double *w_out)
{
    if (!ctx || !w_out) return PCDN_ERR_INVALID;
    CU(cudaMemcpyAsync(w_out, ctx->at<double>(ctx->L.w), sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    return PCDN_OK;
}

int pcdn_get_z(pcdn_ctx *ctx, double *z_out)
{
    if (!ctx || !z_out) return PCDN_ERR_INVALID;
    CU(cudaMemcpyAsync(z_out, ctx->at<double>(ctx->L.z), sizeof(double) * ctx->s, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    return PCDN_OK;
}

int pcdn_objective(pcdn_ctx *ctx, int recompute_from_w, double *F_out)
{
    if (!ctx || !F_out) return PCDN_ERR_INVALID;
    int rc;
    if (recompute_from_w) {
        // evaluate from scratch without disturbing the maintained F: z is recomputed (exact
        // same z for an unchanged w), F_full goes to the copy slot
        if ((rc = refresh_z(ctx, 0))) return rc;
    }
    const Layout &L = ctx->L;
    PCDN_NEED_TARGETS(ctx);
    k_obj_partial<<<OBJ_NB, 256, 0, ctx->stream>>>(ctx->s, ctx->n, ctx->at<double>(L.z), ctx->y, ctx->at<double>(L.w),
                                                   ctx->loss, ctx->at<double>(L.objp), ctx->t);
    k_obj_final<<<1, OBJ_NB, 0, ctx->stream>>>(ctx->at<double>(L.objp), ctx->c, ctx->mu, ctx->at<double>(L.Fcopy), nullptr, -1.0, 0.0,
                                               nullptr, nullptr);
    ctx->launches += 2;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&ctx->hm->Fcopy, ctx->at<double>(L.Fcopy), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *F_out = ctx->hm->Fcopy;
    return PCDN_OK;
}

int pcdn_permutation(pcdn_ctx *ctx, uint64_t seed, int64_t k, int32_t *out)
{
    if (!ctx || !out || k < 0) return PCDN_ERR_INVALID;
    k_perm<<<grid1d(ctx->n), 256, 0, ctx->stream>>>(seed, k, ctx->n, ctx->s, ctx->col_ptr, ctx->heavy_eff, out,
                                                     nullptr, nullptr, nullptr);
    ctx->launches++;
    CU(cudaGetLastError());
    return PCDN_OK;
}

int pcdn_bundle_step(pcdn_ctx *ctx, const int32_t *bundle, int64_t P, pcdn_step_info *info, double *g_out,
                     double *h_out, double *d_out)
{
    if (!ctx) return PCDN_ERR_INVALID;
    if (!bundle || P < 1 || P > ctx->n) return set_err(ctx, PCDN_ERR_INVALID, "bundle size %lld out of [1, n]", (long long)P);
    const Layout &L = ctx->L;
    int rc;
    if ((rc = reset_status(ctx))) return rc;
    CU(cudaMemsetAsync(ctx->at<int64_t>(L.counters), 0, sizeof(int64_t) * 8, ctx->stream));
    const Lists &S = L.ls[0];
    ctx->heavy_eff = heavy_for_mode(ctx, choose_mode(ctx, P), P);
    k_bundle_prep<<<grid1d(P), 256, 0, ctx->stream>>>(bundle, P, ctx->n, ctx->s, ctx->col_ptr, ctx->heavy_eff,
                                                      ctx->at<int32_t>(S.order), ctx->at<int32_t>(S.flag),
                                                      ctx->at<int32_t>(S.fflag),
                                                      ctx->at<uint32_t>(L.seen), ctx->at<int>(L.status),
                                                      ctx->at<long long>(L.err_idx),
                                                      (unsigned long long *)(ctx->at<int64_t>(L.counters) + 2),
                                                      ctx->at<int4>(S.colinfo));
    k_bundle_unseen<<<grid1d(P), 256, 0, ctx->stream>>>(bundle, P, ctx->n, ctx->at<uint32_t>(L.seen));
    ctx->launches += 2;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&ctx->hm->status, ctx->at<int>(L.status), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(&ctx->hm->err_idx, ctx->at<long long>(L.err_idx), sizeof(long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->hm->status)
        return set_err(ctx, PCDN_ERR_INVALID, "bundle entry %lld is out of range or repeated", (long long)ctx->hm->err_idx);
    if ((rc = build_heavy(ctx, P, 0, ctx->stream))) return rc;
    if (ctx->debug) CU(cudaMemsetAsync(ctx->at<uint8_t>(L.dbg_mark), 0, ctx->s, ctx->stream));
    if ((rc = launch_steps(ctx, 0, P, P, 1, 0, g_out, h_out, d_out))) return rc;
    if (info) {
        if ((rc = readback(ctx))) return rc;
        const double *v = ctx->hm->info;
        info->q = (int32_t)v[0];
        info->reserved = 0;
        info->alpha = v[1];
        info->Delta = v[2];
        info->lhs = v[3];
        info->rhs = v[4];
        info->F = v[5];
        info->bundle_nnz = ctx->hm->counters[2];
        info->n_touched = (int64_t)v[7];
        if (ctx->hm->status == 3) return set_err(ctx, PCDN_ERR_NUMERIC, "non-finite line-search quantities");
        if (ctx->hm->status == 7) return set_err(ctx, PCDN_ERR_INVALID, SCDN_HEAVY_MSG);
        if (ctx->hm->status) return set_err(ctx, PCDN_ERR_CUDA, "internal consistency check failed (%d)", ctx->hm->status);
    }
    return PCDN_OK;
}

int pcdn_last_touched(pcdn_ctx *ctx, int32_t *T_out, double *dx_out, int64_t capacity, int64_t *nT)
{
    if (!ctx || !nT) return PCDN_ERR_INVALID;
    if (!ctx->debug) return set_err(ctx, PCDN_ERR_INVALID, "pcdn_last_touched needs pcdn_set_debug(ctx, 1)");
    std::vector<uint8_t> mark(ctx->s);
    std::vector<double> dx(ctx->s);
    CU(cudaMemcpyAsync(mark.data(), ctx->at<uint8_t>(ctx->L.dbg_mark), ctx->s, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(dx.data(), ctx->at<double>(ctx->L.dbg_dx), sizeof(double) * ctx->s, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    int64_t m = 0;
    for (int64_t i = 0; i < ctx->s; i++) {
        if (!mark[i]) continue;
        if (m < capacity) {
            if (T_out) T_out[m] = (int32_t)i;
            if (dx_out) dx_out[m] = dx[i];
        }
        m++;
    }
    *nT = m;
    return PCDN_OK;
}

int pcdn_solve(pcdn_ctx *ctx, int64_t P, double eps, uint64_t seed, int32_t max_outer, pcdn_solve_info *info)
{
    if (!ctx) return PCDN_ERR_INVALID;
    const auto t_start = std::chrono::steady_clock::now();
    if (P < 1 || P > ctx->n) return set_err(ctx, PCDN_ERR_INVALID, "P=%lld out of [1, n=%lld]", (long long)P, (long long)ctx->n);
    if (max_outer < 0) return set_err(ctx, PCDN_ERR_INVALID, "max_outer < 0");
    if (eps > 0 && !ctx->has_fstar) return set_err(ctx, PCDN_ERR_INVALID, "eps > 0 needs pcdn_set_reference");
    const Layout &L = ctx->L;
    const int64_t launches0 = ctx->launches;
    int rc;
    // status / error / stop / ticket / counters and the grid barrier, in one launch
    k_solve_init<<<1, 32, 0, ctx->stream>>>(ctx->at<int>(L.status), ctx->at<long long>(L.err_idx),
                                            ctx->at<int64_t>(L.counters), ctx->at<unsigned long long>(L.bar));
    ctx->launches++;
    CU(cudaGetLastError());
    const int64_t b = (ctx->n + P - 1) / P;
    int status = PCDN_BUDGET;
    int32_t k = 0;
    double F = NAN, gap = NAN, t_step_ms = 0.0;
    CU(cudaEventRecord(ctx->ev[2], ctx->stream));
    // the cluster-resident step kernel occupies one cluster of SMs: the next outer iteration's
    // partition and lists are then built concurrently on the side stream (double-buffered sets)
    const int smode = choose_mode(ctx, P);
    ctx->heavy_eff = heavy_for_mode(ctx, smode, P);
    // the dense kernel needs only the permutation: k_obj computes it (no launch of its own)
    const bool overlap = ctx->side != nullptr && smode == 3;
    const bool lists = smode != 4;
    // Outer iteration kk, queued without waiting: partition pi_kk's lists were built during the
    // previous one; the step launch; the next partition into the other list set (on the side
    // stream beside the one-cluster kernel, after the step that last read that set; else behind
    // the step launch); F from scratch with the device-side stop test; the readback into ring slot
    // kk & 1.  The host queues iteration k+1 before it waits for iteration k's readback, so the
    // GPU never idles on the host's stop decision; when iteration k ends the solve, iteration
    // k+1's step launch finds the stop flag and exits without touching the state.
    HostMirror *const ring = ctx->hm + 1;
    auto enqueue_outer = [&](int32_t kk) -> int {
        const int buf = kk & 1, r = kk & 1;
        if (kk > 0 && overlap) CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_prep, 0));
        CU(cudaEventRecord(ctx->ev[4 + 2 * r], ctx->stream));
        ctx->bar_clean = true;   // re-armed by k_solve_init / the previous outer iteration's k_obj
        int rc2 = launch_steps(ctx, buf, ctx->n, P, b, (int64_t)kk * b, nullptr, nullptr, nullptr);
        if (rc2) return rc2;
        CU(cudaEventRecord(ctx->ev[5 + 2 * r], ctx->stream));
        if (kk + 1 < max_outer && lists) {
            if (overlap && kk > 0) CU(cudaStreamWaitEvent(ctx->side, ctx->ev[5 + 2 * (r ^ 1)], 0));
            if ((rc2 = prep_outer(ctx, seed, kk + 1, buf ^ 1, overlap ? ctx->side : ctx->stream, lists))) return rc2;
            if (overlap) CU(cudaEventRecord(ctx->ev_prep, ctx->side));
        }
        // a6: F from scratch (reading Z23) and the Eq.14 test in one launch, which also writes the
        // read-back block into ring slot r (mapped pinned memory)
        {
            const Layout &L = ctx->L;
            ObjBoundary o{};
            o.c = ctx->c;
            o.mu = ctx->mu;
            o.eps = eps > 0 ? eps : 0.0;
            o.fstar = ctx->fstar;
            o.F = ctx->at<double>(L.F);
            o.status = ctx->at<int>(L.status);
            o.stop = ctx->at<int>(L.stop);
            o.ticket = ctx->at<unsigned>(L.ticket);
            o.bar = ctx->at<unsigned long long>(L.bar);
            o.mirror = ctx->at<unsigned long long>(L.mirror);
            o.mirror_host = reinterpret_cast<unsigned long long *>(ctx->hm_dev + 1 + r);
            o.mirror_words = (int)(sizeof(HostMirror) / 8);
            if (!lists && kk + 1 < max_outer) {
                const Lists &S = L.ls[buf ^ 1];
                o.perm = 1;
                o.seed = seed;
                o.k_next = kk + 1;
                o.n = ctx->n;
                o.s = ctx->s;
                o.col_ptr = ctx->col_ptr;
                o.heavy_len = ctx->heavy_eff;
                o.order = ctx->at<int32_t>(S.order);
                o.flag = ctx->at<int32_t>(S.flag);
                o.fflag = ctx->at<int32_t>(S.fflag);
                o.colinfo = ctx->at<int4>(S.colinfo);
            }
            k_obj<<<OBJ_NB, OBJ_NB, 0, ctx->stream>>>(ctx->s, ctx->n, ctx->at<double>(L.z), ctx->y,
                                                      ctx->at<double>(L.w), ctx->loss, ctx->at<double>(L.objp), ctx->t, o);
            ctx->launches++;
            CU(cudaGetLastError());
        }
        CU(cudaEventRecord(ctx->ev[8 + r], ctx->stream));
        return PCDN_OK;
    };
    struct SolvingScope {
        pcdn_ctx *c;
        ~SolvingScope() { c->solving = false; }
    } scope{ctx};
    ctx->solving = true;
    // the dense kernel runs the whole solve in one launch: its outer boundaries (a6: F from
    // scratch, the Eq.14 test, the next partition) happen inside it, with no host round trip
    const bool fused = smode == 4 && !ctx->dense_per_outer && max_outer > 0;
    if (fused) {
        struct DenseScope {
            pcdn_ctx *c;
            ~DenseScope() { c->dense_outers = 0; }
        } dscope{ctx};
        if ((rc = prep_outer(ctx, seed, 0, 0, ctx->stream, false))) return rc;
        ctx->dense_outers = max_outer;
        ctx->cur_seed = seed;
        ctx->cur_eps = eps > 0 ? eps : 0.0;
        ctx->bar_clean = true;   // k_solve_init
        CU(cudaEventRecord(ctx->ev[4], ctx->stream));
        if ((rc = launch_steps(ctx, 0, ctx->n, P, b, 0, nullptr, nullptr, nullptr))) return rc;
        CU(cudaEventRecord(ctx->ev[5], ctx->stream));
        if ((rc = readback(ctx))) return rc;
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev[4], ctx->ev[5]));
        t_step_ms = ms;
        F = ctx->hm->F;
        k = (int32_t)ctx->hm->counters[5];
        if (ctx->hm->status == 3 || !std::isfinite(F)) {
            status = PCDN_ERR_NUMERIC;
            set_err(ctx, PCDN_ERR_NUMERIC, "non-finite objective in outer iteration %d", k - 1);
        } else if (ctx->hm->status) {
            status = PCDN_ERR_CUDA;
            set_err(ctx, PCDN_ERR_CUDA, "internal consistency check failed (%d)", ctx->hm->status);
        } else if (eps > 0 && (F - ctx->fstar) / ctx->fstar <= eps) {
            status = PCDN_OK;
        }
    } else if (max_outer > 0) {
        if ((rc = prep_outer(ctx, seed, 0, 0, ctx->stream, lists))) return rc;
        if ((rc = enqueue_outer(0))) return rc;
    }
    for (k = fused ? k : 0; !fused && k < max_outer; k++) {
        if (k + 1 < max_outer) {
            if ((rc = enqueue_outer(k + 1))) return rc;
        }
        const int r = k & 1;
        CU(cudaEventSynchronize(ctx->ev[8 + r]));
        const HostMirror &m = ring[r];
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev[4 + 2 * r], ctx->ev[5 + 2 * r]));
        t_step_ms += ms;
        F = m.F;
        if (m.status == 3 || !std::isfinite(F)) {
            status = PCDN_ERR_NUMERIC;
            set_err(ctx, PCDN_ERR_NUMERIC, "non-finite objective in outer iteration %d", k);
            k++;
            break;
        }
        if (m.status == 7) {
            status = PCDN_ERR_INVALID;
            set_err(ctx, PCDN_ERR_INVALID, SCDN_HEAVY_MSG);
            k++;
            break;
        }
        if (m.status) {
            status = PCDN_ERR_CUDA;
            set_err(ctx, PCDN_ERR_CUDA, "internal consistency check failed (%d)", m.status);
            k++;
            break;
        }
        if (eps > 0) {
            gap = (F - ctx->fstar) / ctx->fstar;  // Eq.14 (the same test as k_obj_final's)
            if (gap <= eps) {
                status = PCDN_OK;
                k++;
                break;
            }
        }
    }
    // a list build for an outer iteration that was not run must finish before anything else uses
    // the list sets on the context stream
    if (overlap) CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_prep, 0));
    CU(cudaEventRecord(ctx->ev[3], ctx->stream));
    CU(cudaEventSynchronize(ctx->ev[3]));
    if (max_outer == 0) {
        if ((rc = readback(ctx))) return rc;
        F = ctx->hm->F;
    } else if (!fused) {
        ctx->hm[0] = ring[(k - 1) & 1];   // the last outer iteration taken (a queued one after it was a no-op)
    }
    if (info) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
        const int64_t *cn = ctx->hm->counters;
        info->status = status;
        info->outer_iters = k;
        info->steps = cn[0];
        info->null_steps = cn[1];
        info->nnz_processed = ctx->nnz * (int64_t)k;   // every column once per outer iteration
        info->touched_total = cn[3];
        info->positions = cn[4];
        info->kernel_launches = ctx->launches - launches0;
        info->F = F;
        info->gap = eps > 0 ? (F - ctx->fstar) / ctx->fstar : (ctx->has_fstar ? (F - ctx->fstar) / ctx->fstar : NAN);
        info->t_wall_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        info->t_step_kernel_ms = t_step_ms;
        info->t_gpu_ms = ms;
        // 16 B per bundle nonzero (index+value, gathered fp64 pair counted as
        // one fp64 word of the retained per-sample state), 16 B per touched sample, 28 B per position
        info->alg_bytes = 16.0 * (double)info->nnz_processed + 16.0 * (double)cn[3] + 28.0 * (double)cn[4];
    }
    (void)gap;
    return status;
}

// ---------------------------------------------------------------------------------------
// Sample-sharded step (pcdn_shard.cuh): host-driven phases
// ---------------------------------------------------------------------------------------
static StepArgs shard_args(pcdn_ctx *ctx, int64_t P)
{
    const Layout &L = ctx->L;
    StepArgs a{};
    a.s = ctx->s;
    a.n = ctx->n;
    a.col_ptr = ctx->col_ptr;
    a.row_idx = ctx->row_idx;
    a.val = ctx->val;
    a.row_ptr = ctx->row_ptr;
    a.y = ctx->y;
    a.t = ctx->t;
    a.c = ctx->c;
    a.sigma = ctx->sigma;
    a.beta = ctx->beta;
    a.gamma = ctx->gamma;
    a.nu = ctx->nu;
    a.mu = ctx->mu;
    a.loss = ctx->loss;
    a.qmax = ctx->qmax;
    a.w = ctx->at<double>(L.w);
    a.z = ctx->at<double>(L.z);
    a.coef = ctx->at<double2>(L.coef);
    a.cnt = ctx->at<int32_t>(L.cnt);
    a.bits = ctx->at<uint32_t>(L.bits);
    a.rec = ctx->at<Rec>(L.rec);
    a.dxg = ctx->at<double>(L.dxg);
    a.dk = ctx->at<double>(L.dk);
    a.deltak = ctx->at<double>(L.deltak);
    a.part = ctx->at<double>(L.part);
    a.F = ctx->at<double>(L.F);
    a.P = P;
    a.status = ctx->at<int>(L.status);
    return a;
}

static int shard_blocks(int64_t work, int per)
{
    int64_t b = (work + per - 1) / per;
    if (b < 1) b = 1;
    if (b > 2 * GMAX * NPART / SH_W) b = 2 * GMAX * NPART / SH_W;   // partial rows fit the part buffer
    return (int)b;
}

int pcdn_shard_gh(pcdn_ctx *ctx, const int32_t *bundle, int64_t P, double *gh_out)
{
    if (!ctx || !bundle || !gh_out || P < 1 || P > ctx->n) return PCDN_ERR_INVALID;
    PCDN_NEED_TARGETS(ctx);
    int rc;
    if ((rc = reset_status(ctx))) return rc;
    k_sh_gh<<<shard_blocks(P * 32, SH_NT), SH_NT, 0, ctx->stream>>>(shard_args(ctx, P), bundle, P, gh_out);
    ctx->launches++;
    CU(cudaGetLastError());
    return PCDN_OK;
}

int pcdn_shard_direction(pcdn_ctx *ctx, const int32_t *bundle, int64_t P, const double *gh)
{
    if (!ctx || !bundle || !gh || P < 1 || P > ctx->n) return PCDN_ERR_INVALID;
    PCDN_NEED_TARGETS(ctx);
    k_sh_dir<<<shard_blocks(P * 32, SH_NT), SH_NT, 0, ctx->stream>>>(shard_args(ctx, P), bundle, P, gh);
    ctx->launches++;
    CU(cudaGetLastError());
    return PCDN_OK;
}

int pcdn_shard_line_search(pcdn_ctx *ctx, const int32_t *bundle, int64_t P, int q0, int first, int with_l1,
                           double *out)
{
    if (!ctx || !bundle || !out || P < 1 || P > ctx->n || q0 < 0) return PCDN_ERR_INVALID;
    PCDN_NEED_TARGETS(ctx);
    const StepArgs a = shard_args(ctx, P);
    // short lists by threads, long ones by warps; their partial rows side by side, summed in order
    const int nbl = std::min(shard_blocks(ctx->s * 32, SH_LNT), 4 * ctx->num_sms);
    const int nb = std::min(shard_blocks(ctx->s, SH_NT), 2 * GMAX * NPART / SH_W - nbl);
    k_sh_ls<<<nb, SH_NT, 0, ctx->stream>>>(a, q0, first, a.part);
    k_sh_ls_long<<<nbl, SH_LNT, 0, ctx->stream>>>(a, q0, first, a.part + (size_t)nb * SH_W);
    k_sh_ls_final<<<1, SH_NT, 0, ctx->stream>>>(a, bundle, P, q0, nb + nbl, a.part, with_l1, out);
    ctx->launches += 3;
    CU(cudaGetLastError());
    return PCDN_OK;
}

int pcdn_shard_decide(pcdn_ctx *ctx, const double *tot, int q0, pcdn_shard_decision *out)
{
    if (!ctx || !tot || q0 < 0) return PCDN_ERR_INVALID;
    PCDN_NEED_TARGETS(ctx);
    int rc;
    if ((rc = reset_status(ctx))) return rc;
    k_sh_decide<<<1, 32, 0, ctx->stream>>>(shard_args(ctx, 1), tot, q0, ctx->at<double>(ctx->L.info));
    ctx->launches++;
    CU(cudaGetLastError());
    if ((rc = readback(ctx))) return rc;
    const double *v = ctx->hm->info;
    if (out) {
        out->q = (int32_t)v[0];
        out->next = (int32_t)v[1];
        out->alpha = v[2];
        out->lhs = v[3];
        out->rhs = v[4];
        out->Delta = v[5];
        out->F = v[6];
    }
    if (ctx->hm->status == 3) return set_err(ctx, PCDN_ERR_NUMERIC, "non-finite line-search quantities");
    return PCDN_OK;
}

int pcdn_shard_commit(pcdn_ctx *ctx, const int32_t *bundle, int64_t P)
{
    if (!ctx || !bundle || P < 1 || P > ctx->n) return PCDN_ERR_INVALID;
    PCDN_NEED_TARGETS(ctx);
    k_sh_commit<<<shard_blocks(ctx->s, SH_NT), SH_NT, 0, ctx->stream>>>(shard_args(ctx, P), bundle, P,
                                                                       ctx->at<double>(ctx->L.info));
    ctx->launches++;
    CU(cudaGetLastError());
    int rc;
    if ((rc = readback(ctx))) return rc;
    if (ctx->hm->status) return set_err(ctx, PCDN_ERR_CUDA, "internal consistency check failed (%d)", ctx->hm->status);
    return PCDN_OK;
}

int pcdn_shard_loss(pcdn_ctx *ctx, double *loss_out)
{
    if (!ctx || !loss_out) return PCDN_ERR_INVALID;
    PCDN_NEED_TARGETS(ctx);
    // c * sum_i phi_i of the local samples (Eq.1 without the separable terms) into loss_out (device)
    const Layout &L = ctx->L;
    k_obj_partial<<<OBJ_NB, 256, 0, ctx->stream>>>(ctx->s, 0, ctx->at<double>(L.z), ctx->y, ctx->at<double>(L.w),
                                                   ctx->loss, ctx->at<double>(L.objp), ctx->t);
    k_obj_final<<<1, OBJ_NB, 0, ctx->stream>>>(ctx->at<double>(L.objp), ctx->c, 0.0, loss_out, nullptr, -1.0, 0.0,
                                               nullptr, nullptr);
    ctx->launches += 2;
    CU(cudaGetLastError());
    return PCDN_OK;
}

int pcdn_shard_objective(pcdn_ctx *ctx, const double *loss_sum, double *F_out)
{
    if (!ctx || !loss_sum || !F_out) return PCDN_ERR_INVALID;
    PCDN_NEED_TARGETS(ctx);
    // ||w||_1 + mu/2 ||w||^2 over the replicated w, then + the rank-summed loss: the maintained F
    const Layout &L = ctx->L;
    k_obj_partial<<<OBJ_NB, 256, 0, ctx->stream>>>(0, ctx->n, ctx->at<double>(L.z), ctx->y, ctx->at<double>(L.w),
                                                   ctx->loss, ctx->at<double>(L.objp), ctx->t);
    k_obj_final<<<1, OBJ_NB, 0, ctx->stream>>>(ctx->at<double>(L.objp), ctx->c, ctx->mu, ctx->at<double>(L.F), nullptr,
                                               -1.0, 0.0, nullptr, nullptr);
    k_sh_add_loss<<<1, 32, 0, ctx->stream>>>(ctx->at<double>(L.F), loss_sum, ctx->at<double>(L.Fcopy));
    ctx->launches += 3;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&ctx->hm->Fcopy, ctx->at<double>(L.Fcopy), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *F_out = ctx->hm->Fcopy;
    return PCDN_OK;
}

}  // extern "C"

namespace {
// CSR from CSC on the device (pcdn_train_host with csr_* = NULL): the nonzeros in CSC order
// (columns ascending) are stably sorted by row, so every row lists its columns ascending -- the
// CSR a host would build.  Pairs: key = row, value = column << 32 | value bits.
__global__ void k_csc_pairs(int64_t n, int64_t nnz, const int64_t *__restrict__ col_ptr, const float *__restrict__ val,
                            unsigned long long *pairs)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = gw; j < n; j += nw)   // (the CSC was validated first; the bounds only guard)
        for (int64_t p = max(col_ptr[j], (int64_t)0) + lane; p < min(col_ptr[j + 1], nnz); p += 32)
            pairs[p] = ((unsigned long long)(uint32_t)j << 32) | (unsigned long long)__float_as_uint(val[p]);
}

__global__ void k_csr_from_sorted(int64_t s, int64_t nnz, const int32_t *__restrict__ rows,
                                  const unsigned long long *__restrict__ pairs, int64_t *row_ptr, int32_t *col_idx,
                                  float *csr_val)
{
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = tid; p < nnz; p += nth) {
        const unsigned long long v = pairs[p];
        col_idx[p] = (int32_t)(v >> 32);
        csr_val[p] = __uint_as_float((uint32_t)(v & 0xffffffffull));
    }
    for (int64_t i = tid; i <= s; i += nth) {   // row_ptr[i] = first sorted position with row >= i
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (rows[mid] < i) lo = mid + 1; else hi = mid;
        }
        row_ptr[i] = lo;
    }
}

int device_csr(int64_t s, int64_t n, int64_t nnz, const int64_t *col_ptr, const int32_t *row_idx, const float *val,
               int64_t *row_ptr, int32_t *col_idx, float *csr_val, cudaStream_t st)
{
    int32_t *rows = nullptr;
    unsigned long long *pa = nullptr, *pb = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int bits = 1;
    while ((1ll << bits) < s) bits++;
    int rc = PCDN_OK;
    // the CSC first (col_ptr monotone within [0, nnz], row indices in range, finite values): the
    // pair build below indexes by col_ptr, so a broken one must be refused before it runs
    {
        struct Chk {
            int status, what;
            long long idx;
        } *chk = nullptr, h{};
        if (cudaMallocAsync(&chk, sizeof(Chk), st) != cudaSuccess) return PCDN_ERR_NOMEM;
        if (cudaMemsetAsync(chk, 0, sizeof(Chk), st) != cudaSuccess ||
            cudaMemsetAsync(&chk->idx, 0x7f, sizeof(long long), st) != cudaSuccess)
            rc = PCDN_ERR_CUDA;
        if (rc == PCDN_OK) {
            k_validate<<<grid1d(std::max(nnz, n)), 256, 0, st>>>(s, n, nnz, col_ptr, row_idx, val, nullptr, nullptr, nullptr, nullptr,
                                                  &chk->status, &chk->idx, &chk->what);
            if (cudaGetLastError() != cudaSuccess ||
                cudaMemcpyAsync(&h, chk, sizeof(Chk), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess)
                rc = PCDN_ERR_CUDA;
            else if (h.status)
                rc = PCDN_ERR_INVALID;
        }
        cudaFreeAsync(chk, st);
        if (rc != PCDN_OK) return rc;
    }
    const int64_t m = nnz > 0 ? nnz : 1;
    if (cudaMallocAsync(&rows, sizeof(int32_t) * m, st) != cudaSuccess ||
        cudaMallocAsync(&pa, sizeof(unsigned long long) * m, st) != cudaSuccess ||
        cudaMallocAsync(&pb, sizeof(unsigned long long) * m, st) != cudaSuccess)
        rc = PCDN_ERR_NOMEM;
    if (rc == PCDN_OK && nnz > 0) {
        k_csc_pairs<<<grid1d(n * 32), 256, 0, st>>>(n, nnz, col_ptr, val, pa);
        if (cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, row_idx, rows, pa, pb, (int)nnz, 0, bits, st) !=
                cudaSuccess ||
            cudaMallocAsync(&tmp, tmp_bytes ? tmp_bytes : 1, st) != cudaSuccess ||
            cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, row_idx, rows, pa, pb, (int)nnz, 0, bits, st) !=
                cudaSuccess)
            rc = PCDN_ERR_CUDA;
    }
    if (rc == PCDN_OK) {
        k_csr_from_sorted<<<grid1d(std::max(nnz, s + 1)), 256, 0, st>>>(s, nnz, rows, pb, row_ptr, col_idx, csr_val);
        if (cudaGetLastError() != cudaSuccess) rc = PCDN_ERR_CUDA;
    }
    if (tmp) cudaFreeAsync(tmp, st);
    if (rows) cudaFreeAsync(rows, st);
    if (pa) cudaFreeAsync(pa, st);
    if (pb) cudaFreeAsync(pb, st);
    return rc;
}
}  // namespace

extern "C" {

int pcdn_train_host(int64_t s, int64_t n, int64_t nnz, const int64_t *csc_col_ptr, const int32_t *csc_row_idx,
                    const float *csc_val, const int64_t *csr_row_ptr, const int32_t *csr_col_idx,
                    const float *csr_val, const int8_t *y, double c, int loss, int64_t P, double eps, double f_star,
                    uint64_t seed, int32_t max_outer, void *cuda_stream, double *w_out, pcdn_solve_info *info)
{
    if (loss == PCDN_LOSS_SQUARED) return PCDN_ERR_INVALID;   // needs targets: use pcdn_create + pcdn_set_targets
    pcdn_ctx *ctx = nullptr;  // for CU() error text only
    if (s < 1 || n < 1 || nnz < 0 || !csc_col_ptr || !y || !w_out) return PCDN_ERR_INVALID;
    if (nnz > 0 && (!csc_row_idx || !csc_val)) return PCDN_ERR_INVALID;
    if (nnz > INT32_MAX) return PCDN_ERR_INVALID;   // 32-bit indices (row_idx, col_idx)
    // csr_* all NULL: the CSR is built on the device from the CSC (not copied, not re-checked)
    const bool csr_dev = !csr_row_ptr && !csr_col_idx && !csr_val;
    if (!csr_dev && (!csr_row_ptr || (nnz > 0 && (!csr_col_idx || !csr_val)))) return PCDN_ERR_INVALID;
    if (eps > 0 && !(f_star > 0)) return PCDN_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    {
        // keep the stream-ordered allocations of repeated calls in the device's pool instead of
        // returning them to the driver at every synchronisation (once per process)
        static bool pool_set = false;
        int dev = 0;
        cudaMemPool_t pool;
        if (!pool_set && cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) != cudaSuccess) cudaGetLastError();
            pool_set = true;
        }
    }
    const size_t ws = pcdn_workspace_bytes(s, n, nnz);
    const size_t sz[] = {sizeof(int64_t) * (n + 1), sizeof(int32_t) * nnz, sizeof(float) * nnz,
                         sizeof(int64_t) * (s + 1), sizeof(int32_t) * nnz, sizeof(float) * nnz, (size_t)s, ws,
                         sizeof(double) * n};
    const void *src[] = {csc_col_ptr, csc_row_idx, csc_val, csr_row_ptr, csr_col_idx, csr_val, y, nullptr, nullptr};
    void *d[9] = {nullptr};
    int rc = PCDN_OK;
    for (int i = 0; i < 9; i++) {
        if (cudaMallocAsync(&d[i], sz[i] ? sz[i] : 1, st) != cudaSuccess) {
            rc = PCDN_ERR_NOMEM;
            break;
        }
        if (src[i] && sz[i] && cudaMemcpyAsync(d[i], src[i], sz[i], cudaMemcpyHostToDevice, st) != cudaSuccess) {
            rc = PCDN_ERR_CUDA;
            break;
        }
    }
    if (rc == PCDN_OK && csr_dev)
        rc = device_csr(s, n, nnz, (const int64_t *)d[0], (const int32_t *)d[1], (const float *)d[2], (int64_t *)d[3],
                        (int32_t *)d[4], (float *)d[5], st);
    if (rc == PCDN_OK) {
        g_csr_trusted = csr_dev;
        rc = pcdn_create(s, n, nnz, (const int64_t *)d[0], (const int32_t *)d[1], (const float *)d[2],
                         (const int64_t *)d[3], (const int32_t *)d[4], (const float *)d[5], (const int8_t *)d[6], c,
                         loss, d[7], ws, st, &ctx);
        g_csr_trusted = false;
        if (rc == PCDN_OK && eps > 0) rc = pcdn_set_reference(ctx, f_star);
        if (rc == PCDN_OK) {
            rc = pcdn_solve(ctx, P, eps, seed, max_outer, info);
            if (rc == PCDN_OK || rc == PCDN_BUDGET) {
                int rc2 = pcdn_get_w(ctx, (double *)d[8]);
                if (rc2 == PCDN_OK &&
                    cudaMemcpyAsync(w_out, d[8], sizeof(double) * n, cudaMemcpyDeviceToHost, st) != cudaSuccess)
                    rc2 = PCDN_ERR_CUDA;
                if (rc2 == PCDN_OK && cudaStreamSynchronize(st) != cudaSuccess) rc2 = PCDN_ERR_CUDA;
                if (rc2 != PCDN_OK) rc = rc2;
            }
        }
        if (ctx) pcdn_destroy(ctx);
    }
    for (int i = 0; i < 9; i++)
        if (d[i]) cudaFreeAsync(d[i], st);
    cudaStreamSynchronize(st);
    return rc;
}

}  // extern "C"
