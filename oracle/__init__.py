"""ctypes binding of the fp64 CPU oracle (oracle/pcdn_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this package.  It shares no
code with the CUDA product path and never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pcdn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ERR_INVALID, BUDGET, ERR_NUMERIC = 0, 1, 2, 3
LOSS_LOGISTIC, LOSS_L2SVM, LOSS_SQUARED = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no OpenMP, no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Prob(C.Structure):
    _fields_ = [("s", C.c_int64), ("n", C.c_int64),
                ("col_ptr", C.c_void_p), ("row_idx", C.c_void_p), ("val", C.c_void_p),
                ("y", C.c_void_p), ("c", C.c_double), ("loss", C.c_int32), ("qmax", C.c_int32),
                ("sigma", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("nu", C.c_double), ("mu", C.c_double), ("t", C.c_void_p)]


class _State(C.Structure):
    _fields_ = [("w", C.c_void_p), ("z", C.c_void_p), ("F", C.c_double), ("dx", C.c_void_p),
                ("dxa", C.c_void_p), ("mark", C.c_void_p), ("list", C.c_void_p)]


class _StepOut(C.Structure):
    _fields_ = [("g", C.c_void_p), ("h", C.c_void_p), ("d", C.c_void_p), ("g_abs", C.c_void_p),
                ("h_abs", C.c_void_p), ("T", C.c_void_p), ("dx", C.c_void_p),
                ("dx_abs", C.c_void_p), ("nT", C.c_int64), ("q", C.c_int32), ("pad", C.c_int32),
                ("alpha", C.c_double), ("Delta", C.c_double), ("Delta_abs", C.c_double),
                ("lhs", C.c_double), ("lhs_abs", C.c_double), ("rhs", C.c_double),
                ("F_before", C.c_double), ("F_after", C.c_double),
                ("margin_accept", C.c_double), ("margin_prev", C.c_double),
                ("margin_d", C.c_double), ("bundle_nnz", C.c_int64)]


class _SolveInfo(C.Structure):
    _fields_ = [("outer_iters", C.c_int32), ("status", C.c_int32), ("steps", C.c_int64),
                ("nnz_processed", C.c_int64), ("touched_total", C.c_int64),
                ("null_steps", C.c_int64), ("F", C.c_double), ("gap", C.c_double), ("t_steps", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.ora_mix64.restype = C.c_uint64
        L.ora_mix64.argtypes = [C.c_uint64]
        L.ora_perm_at.restype = C.c_int64
        L.ora_perm_at.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64]
        L.ora_permutation.restype = None
        L.ora_permutation.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_void_p]
        L.ora_phi.restype = C.c_double
        L.ora_phi.argtypes = [C.c_int, C.c_double]
        L.ora_GH.restype = None
        L.ora_GH.argtypes = [C.c_int, C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ora_objective.restype = C.c_double
        L.ora_objective.argtypes = [C.POINTER(_Prob), C.c_void_p, C.c_void_p]
        L.ora_compute_z.restype = None
        L.ora_compute_z.argtypes = [C.POINTER(_Prob), C.c_void_p, C.c_void_p]
        L.ora_gh_all.restype = None
        L.ora_gh_all.argtypes = [C.POINTER(_Prob), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ora_newton_dir.restype = C.c_double
        L.ora_newton_dir.argtypes = [C.c_double, C.c_double, C.c_double]
        L.ora_bundle_step.restype = C.c_int
        L.ora_bundle_step.argtypes = [C.POINTER(_Prob), C.POINTER(_State), C.c_void_p, C.c_int64,
                                      C.c_int, C.POINTER(_StepOut)]
        L.ora_solve.restype = C.c_int
        L.ora_solve.argtypes = [C.POINTER(_Prob), C.c_void_p, C.c_void_p, C.c_int64, C.c_double,
                                C.c_double, C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_int64, C.POINTER(_SolveInfo), C.c_void_p, C.c_int64]
        L.ora_cdn.restype = C.c_int
        L.ora_cdn.argtypes = [C.POINTER(_Prob), C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32,
                              C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
        L.ora_scdn.restype = C.c_int
        L.ora_scdn.argtypes = [C.POINTER(_Prob), C.c_void_p, C.c_void_p, C.c_int64, C.c_uint64, C.c_int32,
                               C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.ora_min_norm_subgrad.restype = C.c_double
        L.ora_min_norm_subgrad.argtypes = [C.POINTER(_Prob), C.c_void_p, C.c_void_p, C.c_void_p]
        L.ora_loss_change.restype = C.c_double
        L.ora_loss_change.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double]
        for nm, st in (("ora_state_size", _State), ("ora_step_out_size", _StepOut),
                       ("ora_prob_size", _Prob), ("ora_solve_info_size", _SolveInfo)):
            f = getattr(L, nm)
            f.restype = C.c_int
            assert f() == C.sizeof(st), f"{nm}: struct layout mismatch"
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def mix64(x: int) -> int:
    return int(lib().ora_mix64(x & 0xFFFFFFFFFFFFFFFF))


def permutation(seed: int, k: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    lib().ora_permutation(seed, k, n, _p(out))
    return out


def phi(loss: int, m: float) -> float:
    return lib().ora_phi(loss, m)


def GH(loss: int, z: float, y: int):
    G, H = C.c_double(), C.c_double()
    lib().ora_GH(loss, z, y, C.byref(G), C.byref(H))
    return G.value, H.value


def newton_dir(g: float, h: float, wj: float) -> float:
    return lib().ora_newton_dir(g, h, wj)


def loss_change(loss: int, z: float, y: int, dx: float, alpha: float) -> float:
    return lib().ora_loss_change(loss, z, y, dx, alpha)


class Oracle:
    """Oracle bound to one problem (any object with the synth.Problem fields)."""

    def __init__(self, prob, sigma=0.01, beta=0.5, gamma=0.0, nu=1e-12, qmax=50, mu=0.0):
        """mu: elastic-net weight of (mu/2)||w||^2 (reading Z25; 0 = the paper's problem)."""
        self.p = prob
        self.col_ptr = np.ascontiguousarray(prob.col_ptr, dtype=np.int64)
        self.row_idx = np.ascontiguousarray(prob.row_idx, dtype=np.int32)
        self.val = np.ascontiguousarray(prob.val, dtype=np.float32)
        self.y = np.ascontiguousarray(prob.y, dtype=np.int8)
        self.s, self.n = int(prob.s), int(prob.n)
        tt = getattr(prob, "t", None)
        if int(prob.loss) == LOSS_SQUARED and tt is None:
            raise ValueError("the squared loss needs real targets prob.t")
        self.t = None if tt is None else np.ascontiguousarray(tt, dtype=np.float64)
        self.pb = _Prob(self.s, self.n, _p(self.col_ptr), _p(self.row_idx), _p(self.val), _p(self.y),
                        float(prob.c), int(prob.loss), int(qmax), sigma, beta, gamma, nu, float(mu),
                        _p(self.t))

    # --- plain evaluations ---
    def compute_z(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        z = np.empty(self.s, dtype=np.float64)
        lib().ora_compute_z(C.byref(self.pb), _p(w), _p(z))
        return z

    def objective(self, w, z=None):
        w = np.ascontiguousarray(w, dtype=np.float64)
        if z is None:
            z = self.compute_z(w)
        return lib().ora_objective(C.byref(self.pb), _p(z), _p(w))

    def gh(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        z = self.compute_z(w)
        g = np.empty(self.n)
        h = np.empty(self.n)
        lib().ora_gh_all(C.byref(self.pb), _p(z), _p(w), _p(g), _p(h))
        return g, h

    def min_norm_subgrad(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        z = self.compute_z(w)
        out = np.empty(self.n)
        tot = lib().ora_min_norm_subgrad(C.byref(self.pb), _p(w), _p(z), _p(out))
        return tot, out

    # --- one bundle step from state w (z recomputed from w, F from scratch) ---
    def step(self, w, bundle, mode: int = 0, F=None):
        w = np.array(w, dtype=np.float64, copy=True)
        z = self.compute_z(w)
        bundle = np.ascontiguousarray(bundle, dtype=np.int32)
        P = bundle.size
        st = _State()
        dx = np.zeros(self.s)
        dxa = np.zeros(self.s)
        mark = np.zeros(self.s, dtype=np.uint8)
        lst = np.zeros(max(self.s, 1), dtype=np.int32)
        st.w, st.z = _p(w), _p(z)
        st.F = self.objective(w, z) if F is None else float(F)
        st.dx, st.dxa, st.mark, st.list = _p(dx), _p(dxa), _p(mark), _p(lst)
        o = _StepOut()
        arrs = dict(g=np.zeros(P), h=np.zeros(P), d=np.zeros(P), g_abs=np.zeros(P), h_abs=np.zeros(P),
                    T=np.zeros(max(self.s, 1), dtype=np.int32), dx=np.zeros(max(self.s, 1)),
                    dx_abs=np.zeros(max(self.s, 1)))
        for k, a in arrs.items():
            setattr(o, k, _p(a))
        rc = lib().ora_bundle_step(C.byref(self.pb), C.byref(st), _p(bundle), P, mode, C.byref(o))
        nT = int(o.nT)
        res = dict(rc=rc, g=arrs["g"], h=arrs["h"], d=arrs["d"], g_abs=arrs["g_abs"], h_abs=arrs["h_abs"],
                   T=arrs["T"][:nT].copy(), dx=arrs["dx"][:nT].copy(), dx_abs=arrs["dx_abs"][:nT].copy(),
                   q=int(o.q), alpha=o.alpha, Delta=o.Delta, Delta_abs=o.Delta_abs, lhs=o.lhs,
                   lhs_abs=o.lhs_abs, rhs=o.rhs, F_before=o.F_before, F_after=st.F,
                   margin_accept=o.margin_accept, margin_prev=o.margin_prev, margin_d=o.margin_d,
                   bundle_nnz=int(o.bundle_nnz), w=w, z=z)
        return res

    # --- Alg.3 driver ---
    def solve(self, P, eps=0.0, fstar=1.0, seed=0, max_outer=10, w0=None, trace_cap=None, max_steps=0):
        """Alg.3 from w0 (default 0).  max_steps > 0 stops after that many bundle steps (a bounded
        CPU timing sample; rc = BUDGET)."""
        w = np.zeros(self.n) if w0 is None else np.array(w0, dtype=np.float64, copy=True)
        z = np.zeros(self.s)
        b = -(-self.n // int(P))
        cap = max_outer * b if trace_cap is None else trace_cap
        qt = np.zeros(max(cap, 1), dtype=np.int32)
        Ft = np.zeros(max(cap, 1))
        oF = np.zeros(max(max_outer, 1))
        mt = np.zeros(max(cap, 1))
        info = _SolveInfo()
        rc = lib().ora_solve(C.byref(self.pb), _p(w), _p(z), int(P), float(eps), float(fstar),
                             seed & 0xFFFFFFFFFFFFFFFF, int(max_outer), _p(qt), _p(Ft), _p(oF), cap,
                             C.byref(info), _p(mt), int(max_steps))
        ns = min(int(info.steps), cap)
        return dict(rc=rc, w=w, z=z, F=info.F, gap=info.gap, outer=int(info.outer_iters),
                    steps=int(info.steps), nnz=int(info.nnz_processed), touched=int(info.touched_total), null_steps=int(info.null_steps),
                    q_trace=qt[:ns].copy(), F_trace=Ft[:ns].copy(), outer_F=oF[:int(info.outer_iters)].copy(),
                    margin_trace=mt[:ns].copy(), t_steps=float(info.t_steps))

    def scdn(self, Pbar, seed=0, max_outer=10, w0=None):
        """Alg.2 (Shotgun CDN), synchronous reading Z27: the F trace has one entry per iteration."""
        w = np.zeros(self.n) if w0 is None else np.array(w0, dtype=np.float64, copy=True)
        z = np.zeros(self.s)
        cap = max_outer * (-(-self.n // int(Pbar)))
        Ft = np.zeros(max(cap, 1))
        steps = C.c_int64()
        F = C.c_double()
        rc = lib().ora_scdn(C.byref(self.pb), _p(w), _p(z), int(Pbar), seed & 0xFFFFFFFFFFFFFFFF, int(max_outer),
                            _p(Ft), cap, C.byref(steps), C.byref(F))
        return dict(rc=rc, w=w, z=z, F=F.value, steps=int(steps.value), F_trace=Ft[:int(steps.value)].copy())

    def cdn(self, seed=0, max_outer=10, w0=None, trace=False):
        w = np.zeros(self.n) if w0 is None else np.array(w0, dtype=np.float64, copy=True)
        z = np.zeros(self.s)
        cap = max_outer * self.n if trace else 0
        Ft = np.zeros(max(cap, 1))
        F = C.c_double()
        rc = lib().ora_cdn(C.byref(self.pb), _p(w), _p(z), seed & 0xFFFFFFFFFFFFFFFF, int(max_outer),
                           _p(Ft) if trace else None, cap, C.byref(F))
        return dict(rc=rc, w=w, z=z, F=F.value, F_trace=Ft[:cap].copy())


# ---------------------------------------------------------------------------------------------
# Lemma 1(a) (proof, Eq. "ebtdef"): for a uniformly random
# bundle B of P distinct features, lambda_bar(B) = max_{j in B} (X'X)_jj and, with lambda_k the
# k-th smallest (X'X)_jj,
#     f(P) = E[lambda_bar(B)] = (1 / C(n,P)) * sum_{k=P}^{n} lambda_k C(k-1, P-1)
# (the maximum of a P-subset is lambda_k exactly when the other P-1 members are among the k-1
# smaller ones).  Written out term by term in log-space (lgamma) so large n does not overflow.
# ---------------------------------------------------------------------------------------------
def column_sq_norms(prob) -> np.ndarray:
    """lambda_j = (X'X)_jj = sum_i x_ij^2, fp64, from the CSC columns."""
    out = np.zeros(int(prob.n))
    for j in range(int(prob.n)):
        a, b = int(prob.col_ptr[j]), int(prob.col_ptr[j + 1])
        v = np.asarray(prob.val[a:b], dtype=np.float64)
        out[j] = float(np.dot(v, v))
    return out


def expected_lambda_max(lam, P: int) -> float:
    """f(P) of Lemma 1(a)."""
    import math
    lam = np.sort(np.asarray(lam, dtype=np.float64))   # lambda_1 <= ... <= lambda_n
    n = lam.size
    if not 1 <= P <= n:
        raise ValueError("1 <= P <= n")
    log_cnp = math.lgamma(n + 1) - math.lgamma(P + 1) - math.lgamma(n - P + 1)
    tot = 0.0
    for k in range(P, n + 1):   # 1-based k
        log_c = math.lgamma(k) - math.lgamma(P) - math.lgamma(k - P + 1)
        tot += lam[k - 1] * math.exp(log_c - log_cnp)
    return tot
