"""paper_1306_4080_b200 -- B200-native PCDN hot path (arXiv:1306.4080) behind a C-ABI.

Python surface = the C-ABI of include/pcdn.h with the same names (argument marshalling only),
plus `Solver`, a convenience owner of the device tensors.  torch provides device memory and
the CUDA stream; all arithmetic runs in libpcdn.so's sm_100a kernels.  There is no CPU
fallback: without libpcdn.so (or without a GPU) these calls raise.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._abi import (  # noqa: F401
    PCDN_BUDGET, PCDN_ERR_CUDA, PCDN_ERR_INVALID, PCDN_ERR_NOMEM, PCDN_ERR_NUMERIC, PCDN_LOSS_L2SVM, PCDN_LOSS_SQUARED,
    PCDN_LOSS_LOGISTIC, PCDN_OK, PCDNError, check, lib, pcdn_solve_info, pcdn_step_info,
)

__all__ = [
    "pcdn_workspace_bytes", "pcdn_create", "pcdn_set_armijo", "pcdn_set_reference", "pcdn_bundle_step",
    "pcdn_last_touched", "pcdn_solve", "pcdn_objective", "pcdn_get_w", "pcdn_set_w", "pcdn_get_z",
    "pcdn_reset", "pcdn_permutation", "pcdn_set_trace", "pcdn_set_debug", "pcdn_set_launch", "pcdn_set_resident_cap", "pcdn_set_l2_persist", "pcdn_set_elastic", "pcdn_set_targets", "pcdn_set_scdn", "pcdn_set_profile", "pcdn_phase_cycles", "pcdn_warp_timeline",
    "pcdn_last_error", "pcdn_destroy", "pcdn_train_host", "pcdn_version", "Solver", "PCDNError",
]


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(C.c_void_p)
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


# ----------------------------------------------------------------------------- C-ABI mirror
def pcdn_version() -> str:
    return lib().pcdn_version().decode()


def pcdn_workspace_bytes(s, n, nnz) -> int:
    return int(lib().pcdn_workspace_bytes(s, n, nnz))


def pcdn_create(s, n, nnz, col_ptr, row_idx, val, row_ptr, col_idx, csr_val, y, c, loss, workspace,
                stream=None):
    """Device tensors in, opaque context out (raises PCDNError on validation failure)."""
    h = C.c_void_p()
    st = lib().pcdn_create(s, n, nnz, _ptr(col_ptr), _ptr(row_idx), _ptr(val), _ptr(row_ptr), _ptr(col_idx),
                           _ptr(csr_val), _ptr(y), float(c), int(loss), _ptr(workspace),
                           workspace.numel() * workspace.element_size(), _stream(stream), C.byref(h))
    if st != PCDN_OK:
        msg = lib().pcdn_last_error(h).decode() if h.value else ""
        if h.value:
            lib().pcdn_destroy(h)
        raise PCDNError(st, msg)
    return h


def pcdn_set_armijo(ctx, sigma=0.01, beta=0.5, gamma=0.0, q_max=50):
    return check(ctx, lib().pcdn_set_armijo(ctx, sigma, beta, gamma, q_max))


def pcdn_set_reference(ctx, f_star):
    return check(ctx, lib().pcdn_set_reference(ctx, float(f_star)))


def pcdn_bundle_step(ctx, bundle, P=None, info=True, g_out=None, h_out=None, d_out=None):
    P = bundle.numel() if P is None else P
    inf = pcdn_step_info() if info else None
    check(ctx, lib().pcdn_bundle_step(ctx, _ptr(bundle), P, C.byref(inf) if inf is not None else None,
                                      _ptr(g_out), _ptr(h_out), _ptr(d_out)))
    return inf


def pcdn_last_touched(ctx, capacity):
    T = np.zeros(max(capacity, 1), dtype=np.int32)
    dx = np.zeros(max(capacity, 1), dtype=np.float64)
    nT = C.c_int64()
    check(ctx, lib().pcdn_last_touched(ctx, _ptr(T), _ptr(dx), capacity, C.byref(nT)))
    m = min(nT.value, capacity)
    return T[:m], dx[:m], nT.value


def pcdn_solve(ctx, P, eps, seed, max_outer):
    inf = pcdn_solve_info()
    st = lib().pcdn_solve(ctx, int(P), float(eps), int(seed) & 0xFFFFFFFFFFFFFFFF, int(max_outer), C.byref(inf))
    check(ctx, st, ok=(PCDN_OK, PCDN_BUDGET))
    return st, inf


def pcdn_objective(ctx, recompute_from_w=False):
    F = C.c_double()
    check(ctx, lib().pcdn_objective(ctx, 1 if recompute_from_w else 0, C.byref(F)))
    return F.value


def pcdn_get_w(ctx, w_out):
    return check(ctx, lib().pcdn_get_w(ctx, _ptr(w_out)))


def pcdn_set_w(ctx, w):
    return check(ctx, lib().pcdn_set_w(ctx, _ptr(w)))


def pcdn_get_z(ctx, z_out):
    return check(ctx, lib().pcdn_get_z(ctx, _ptr(z_out)))


def pcdn_reset(ctx):
    return check(ctx, lib().pcdn_reset(ctx))


def pcdn_permutation(ctx, seed, k, out):
    return check(ctx, lib().pcdn_permutation(ctx, int(seed) & 0xFFFFFFFFFFFFFFFF, int(k), _ptr(out)))


def pcdn_set_trace(ctx, q_trace, F_trace, capacity):
    return check(ctx, lib().pcdn_set_trace(ctx, _ptr(q_trace), _ptr(F_trace), int(capacity)))


def pcdn_set_debug(ctx, on):
    return check(ctx, lib().pcdn_set_debug(ctx, int(on)))


def pcdn_set_launch(ctx, mode=0, ctas=0, heavy_len=0):
    return check(ctx, lib().pcdn_set_launch(ctx, int(mode), int(ctas), int(heavy_len)))


def pcdn_set_scdn(ctx, on):
    return check(ctx, lib().pcdn_set_scdn(ctx, int(bool(on))))


def pcdn_set_targets(ctx, t):
    return check(ctx, lib().pcdn_set_targets(ctx, _ptr(t)))


def pcdn_set_elastic(ctx, mu):
    return check(ctx, lib().pcdn_set_elastic(ctx, float(mu)))


def pcdn_set_l2_persist(ctx, on):
    return check(ctx, lib().pcdn_set_l2_persist(ctx, int(bool(on))))


def pcdn_set_resident_cap(ctx, cap):
    return check(ctx, lib().pcdn_set_resident_cap(ctx, int(cap)))


def pcdn_set_profile(ctx, on):
    """on: 0 off, 1 per-phase cycle counters, 2 also the per-warp timeline."""
    return check(ctx, lib().pcdn_set_profile(ctx, int(on)))


def pcdn_phase_cycles(ctx):
    out = np.zeros(16, dtype=np.int64)
    mode = C.c_int32()
    check(ctx, lib().pcdn_phase_cycles(ctx, _ptr(out), C.byref(mode)))
    return out, mode.value


def pcdn_warp_timeline(ctx):
    out = np.zeros(16 * 16 * 16, dtype=np.int64)
    check(ctx, lib().pcdn_warp_timeline(ctx, _ptr(out)))
    return out.reshape(16, 16, 16)


def pcdn_last_error(ctx) -> str:
    return lib().pcdn_last_error(ctx).decode()


def pcdn_destroy(ctx):
    lib().pcdn_destroy(ctx)


def pcdn_train_host(col_ptr, row_idx, val, row_ptr, col_idx, csr_val, y, c, loss, P, eps, f_star, seed,
                    max_outer, stream=None, w_out=None):
    """Host (numpy, ideally pinned) arrays in, w out: the one-call end-to-end API.  row_ptr,
    col_idx, csr_val may all be None: the CSR is then built on the device from the CSC."""
    s, n, nnz = int(y.shape[0]), int(col_ptr.shape[0] - 1), int(col_ptr[-1])
    w = np.zeros(n, dtype=np.float64) if w_out is None else w_out

    def _want(a, dt, size, what, optional=False):
        if a is None and optional:
            return
        if not isinstance(a, np.ndarray) or a.dtype != dt or a.ndim != 1 or a.size != size or not a.flags.c_contiguous:
            raise PCDNError(PCDN_ERR_INVALID, f"pcdn_train_host: {what} must be a contiguous {np.dtype(dt).name}[{size}]")

    _want(col_ptr, np.int64, n + 1, "col_ptr")
    _want(row_idx, np.int32, nnz, "row_idx")
    _want(val, np.float32, nnz, "val")
    _want(y, np.int8, s, "y")
    _want(row_ptr, np.int64, s + 1, "row_ptr", optional=True)
    _want(col_idx, np.int32, nnz, "col_idx", optional=True)
    _want(csr_val, np.float32, nnz, "csr_val", optional=True)
    _want(w, np.float64, n, "w_out")
    inf = pcdn_solve_info()
    st = lib().pcdn_train_host(s, n, nnz, _ptr(col_ptr), _ptr(row_idx), _ptr(val), _ptr(row_ptr), _ptr(col_idx),
                               _ptr(csr_val), _ptr(y), float(c), int(loss), int(P), float(eps), float(f_star),
                               int(seed) & 0xFFFFFFFFFFFFFFFF, int(max_outer), _stream(stream), _ptr(w),
                               C.byref(inf))
    if st not in (PCDN_OK, PCDN_BUDGET):
        raise PCDNError(st, "pcdn_train_host failed")
    return st, inf, w


# ----------------------------------------------------------------------------- convenience owner
class Solver:
    """Owns device copies of one problem (CSC + CSR + y), the workspace and the context.

    `prob` is any object with fields s, n, col_ptr, row_idx, val, row_ptr, col_idx, csr_val, y,
    c, loss (e.g. synth.Problem)."""

    def __init__(self, prob, device="cuda", stream=None, sigma=0.01, beta=0.5, gamma=0.0, q_max=50):
        import torch
        self.torch = torch
        dev = torch.device(device)
        self.device = dev
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        self.s, self.n = int(prob.s), int(prob.n)
        self.nnz = int(prob.col_ptr[-1])
        T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
        self.col_ptr = T(prob.col_ptr, np.int64)
        self.row_idx = T(prob.row_idx, np.int32)
        self.val = T(prob.val, np.float32)
        self.row_ptr = T(prob.row_ptr, np.int64)
        self.col_idx = T(prob.col_idx, np.int32)
        self.csr_val = T(prob.csr_val, np.float32)
        self.y = T(prob.y, np.int8)
        self.c, self.loss = float(prob.c), int(prob.loss)
        ws = pcdn_workspace_bytes(self.s, self.n, self.nnz)
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=dev)
        self.ctx = pcdn_create(self.s, self.n, self.nnz, self.col_ptr, self.row_idx, self.val, self.row_ptr,
                               self.col_idx, self.csr_val, self.y, self.c, self.loss, self.workspace, self.stream)
        pcdn_set_armijo(self.ctx, sigma, beta, gamma, q_max)
        self.t = None
        if self.loss == PCDN_LOSS_SQUARED:   # Lasso / elastic-net regression: real targets
            self.t = T(prob.t, np.float64)
            pcdn_set_targets(self.ctx, self.t)

    # state
    def w(self):
        out = self.torch.empty(self.n, dtype=self.torch.float64, device=self.device)
        pcdn_get_w(self.ctx, out)
        return out

    def z(self):
        out = self.torch.empty(self.s, dtype=self.torch.float64, device=self.device)
        pcdn_get_z(self.ctx, out)
        return out

    def set_w(self, w):
        wt = self.torch.as_tensor(np.ascontiguousarray(w, dtype=np.float64)).to(self.device) \
            if isinstance(w, np.ndarray) else w
        pcdn_set_w(self.ctx, wt)
        self.torch.cuda.synchronize(self.device)

    def reset(self):
        pcdn_reset(self.ctx)

    def objective(self, recompute=False):
        return pcdn_objective(self.ctx, recompute)

    def permutation(self, seed, k):
        out = self.torch.empty(self.n, dtype=self.torch.int32, device=self.device)
        pcdn_permutation(self.ctx, seed, k, out)
        return out

    # hot path
    def step(self, bundle, outputs=True, debug=True):
        b = self.torch.as_tensor(np.ascontiguousarray(bundle, dtype=np.int32)).to(self.device) \
            if isinstance(bundle, (np.ndarray, list)) else bundle
        P = b.numel()
        pcdn_set_debug(self.ctx, debug)
        g = h = d = None
        if outputs:
            g, h, d = (self.torch.empty(P, dtype=self.torch.float64, device=self.device) for _ in range(3))
        inf = pcdn_bundle_step(self.ctx, b, P, True, g, h, d)
        res = dict(q=inf.q, alpha=inf.alpha, Delta=inf.Delta, lhs=inf.lhs, rhs=inf.rhs, F=inf.F,
                   bundle_nnz=inf.bundle_nnz, n_touched=inf.n_touched)
        if outputs:
            res.update(g=g.cpu().numpy(), h=h.cpu().numpy(), d=d.cpu().numpy())
        if debug:
            T, dx, nT = pcdn_last_touched(self.ctx, self.s)
            res.update(T=T, dx=dx)
        return res

    def solve(self, P, eps=0.0, seed=0, max_outer=10, fstar=None, trace=False):
        if fstar is not None:
            pcdn_set_reference(self.ctx, fstar)
        qt = Ft = None
        if trace:
            cap = max_outer * (-(-self.n // int(P)))
            qt = self.torch.zeros(max(cap, 1), dtype=self.torch.int32, device=self.device)
            Ft = self.torch.zeros(max(cap, 1), dtype=self.torch.float64, device=self.device)
            pcdn_set_trace(self.ctx, qt, Ft, cap)
        st, inf = pcdn_solve(self.ctx, P, eps, seed, max_outer)
        if trace:
            pcdn_set_trace(self.ctx, None, None, 0)
        res = inf.as_dict()
        res["rc"] = st
        if trace:
            ns = min(inf.steps, qt.numel())
            res["q_trace"] = qt[:ns].cpu().numpy()
            res["F_trace"] = Ft[:ns].cpu().numpy()
        return res

    def set_scdn(self, on=True):
        """Run SCDN (Alg.2, synchronous reading Z27) instead of PCDN (pcdn_set_scdn)."""
        pcdn_set_scdn(self.ctx, on)

    def set_elastic(self, mu):
        """Elastic-net weight: minimise c sum phi + ||w||_1 + (mu/2)||w||^2 (pcdn_set_elastic)."""
        pcdn_set_elastic(self.ctx, mu)

    def set_launch(self, mode=0, ctas=0, heavy_len=0, res_cap=None):
        if res_cap is not None:
            pcdn_set_resident_cap(self.ctx, res_cap)
        pcdn_set_launch(self.ctx, mode, ctas, heavy_len)

    def close(self):
        if getattr(self, "ctx", None) is not None:
            pcdn_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# sample-sharded step (NEXT #2): C-ABI wrappers and the rank-level driver
from .sharded import (  # noqa: E402,F401
    ShardedSolver, pcdn_shard_commit, pcdn_shard_decide, pcdn_shard_direction, pcdn_shard_gh, pcdn_shard_line_search,
    pcdn_shard_loss, pcdn_shard_objective, rank_order_sum,
)
