"""Seeded synthetic PCDN workloads.

Letters follow the paper (Table 1): s = #samples, n = #features.
BASELINE.json's configs say "n samples x d features"; config "n" is our s and
config "d" is our n.

Every array is produced from numpy's `default_rng(seed)` in a fixed draw order,
so the same seed gives byte-identical data on every machine with the same numpy.
Nothing here evaluates the PCDN objective, gradients or directions.
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field

import numpy as np

LOSS_LOGISTIC = 0  # Eq. 2
LOSS_L2SVM = 1     # Eq. 3
LOSS_SQUARED = 2   # Lasso / elastic-net regression (reading Z26)

GEN_VERSION = 1


@dataclass
class Problem:
    """One training set {(x_i, y_i)} in both CSC and CSR form."""

    name: str
    s: int
    n: int
    col_ptr: np.ndarray   # int64[n+1]
    row_idx: np.ndarray   # int32[nnz], strictly increasing inside each column
    val: np.ndarray       # float32[nnz]
    row_ptr: np.ndarray   # int64[s+1]
    col_idx: np.ndarray   # int32[nnz], strictly increasing inside each row
    csr_val: np.ndarray   # float32[nnz]
    y: np.ndarray         # int8[s], values in {-1,+1}
    c: float
    loss: int
    P: int
    seed: int
    meta: dict = field(default_factory=dict)
    t: np.ndarray | None = None   # float64[s] real targets of the squared loss (else None)

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    def dense(self) -> np.ndarray:
        """fp64 dense copy of X (tiny problems only)."""
        X = np.zeros((self.s, self.n), dtype=np.float64)
        for j in range(self.n):
            a, b = self.col_ptr[j], self.col_ptr[j + 1]
            X[self.row_idx[a:b], j] = self.val[a:b]
        return X

    def digest(self) -> str:
        h = hashlib.sha256()
        for a in (self.col_ptr, self.row_idx, self.val, self.y):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()[:16]

    def with_loss(self, loss: int) -> "Problem":
        p = Problem(**{k: getattr(self, k) for k in self.__dataclass_fields__})
        p.loss = loss
        p.name = self.name + {LOSS_LOGISTIC: "-lr", LOSS_L2SVM: "-svm"}.get(loss, "-sq")
        return p


def shard_rows(prob: "Problem", rank: int, world: int) -> "Problem":
    """Rows [floor(rank s / world), floor((rank+1) s / world)) of `prob` as a Problem of their own
    (CSR slice, CSC rebuilt from it, labels / targets sliced); n and every parameter unchanged.
    Data layout only: the sample-sharded step gives each rank one of these."""
    r0, r1 = rank * prob.s // world, (rank + 1) * prob.s // world
    a, b = int(prob.row_ptr[r0]), int(prob.row_ptr[r1])
    row_ptr = (prob.row_ptr[r0:r1 + 1] - a).astype(np.int64)
    col_idx = prob.col_idx[a:b].copy()
    csr_val = prob.csr_val[a:b].copy()
    col_ptr, row_idx, val = csr_to_csc(r1 - r0, prob.n, row_ptr, col_idx, csr_val)
    p = Problem(name=f"{prob.name}-shard{rank}of{world}", s=r1 - r0, n=prob.n, col_ptr=col_ptr, row_idx=row_idx,
                val=val, row_ptr=row_ptr, col_idx=col_idx, csr_val=csr_val, y=prob.y[r0:r1].copy(), c=prob.c,
                loss=prob.loss, P=prob.P, seed=prob.seed, meta=dict(prob.meta, rows=(r0, r1)))
    if prob.t is not None:
        p.t = prob.t[r0:r1].copy()
    return p


def regression(prob: "Problem", noise: float = 0.1, support: int = 500, seed: int | None = None) -> "Problem":
    """The same design matrix with real targets t = X w* + N(0, noise^2) for a planted w* with
    `support` N(0,1) nonzeros (uniform without replacement), loss = LOSS_SQUARED.  Data
    generation only (a matrix-vector product), no PCDN arithmetic."""
    rng = np.random.default_rng((prob.seed if seed is None else seed) + 7919)
    k = min(int(support), prob.n)
    wstar = np.zeros(prob.n)
    wstar[rng.choice(prob.n, size=k, replace=False)] = rng.normal(size=k)
    rows = np.repeat(np.arange(prob.s), np.diff(prob.row_ptr))
    t = np.bincount(rows, weights=prob.csr_val.astype(np.float64) * wstar[prob.col_idx], minlength=prob.s)
    if noise > 0:
        t = t + rng.normal(0.0, noise, size=prob.s)
    p = prob.with_loss(LOSS_SQUARED)
    p.t = t
    return p


# ----------------------------------------------------------------------------------
# structure helpers
# ----------------------------------------------------------------------------------

def csr_to_csc(s, n, row_ptr, col_idx, csr_val):
    """Transpose CSR -> CSC with row indices ascending inside each column."""
    nnz = int(row_ptr[-1])
    rows = np.repeat(np.arange(s, dtype=np.int32), np.diff(row_ptr).astype(np.int64))
    order = np.argsort(col_idx, kind="stable")  # stable: rows stay ascending
    row_idx = rows[order].astype(np.int32)
    val = csr_val[order].astype(np.float32)
    counts = np.bincount(col_idx, minlength=n).astype(np.int64)
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    assert col_ptr[-1] == nnz
    return col_ptr, row_idx, val


def _first_k_distinct(cand: np.ndarray, k: int):
    """Per row of `cand` (b, m): the first k distinct values in draw order.

    Returns (cols (b,k) sorted ascending per row, ok mask (b,)).  This is the
    'distinct columns by rejection of repeats' rule of SURVEY.md §8(d)."""
    b, m = cand.shape
    order = np.argsort(cand, axis=1, kind="stable")
    srt = np.take_along_axis(cand, order, axis=1)
    dup_sorted = np.zeros_like(srt, dtype=bool)
    dup_sorted[:, 1:] = srt[:, 1:] == srt[:, :-1]
    dup = np.zeros_like(dup_sorted)
    np.put_along_axis(dup, order, dup_sorted, axis=1)
    keep = ~dup
    rank = np.cumsum(keep, axis=1)
    sel = keep & (rank <= k)
    ok = rank[:, -1] >= k
    out = np.zeros((b, k), dtype=cand.dtype)
    rows_ok = np.nonzero(ok)[0]
    if rows_ok.size:
        vals = cand[rows_ok][sel[rows_ok]].reshape(rows_ok.size, k)
        out[rows_ok] = np.sort(vals, axis=1)
    return out, ok


def _distinct_rows(s, k, n, draw, rng, batch=65536):
    """(s,k) int32 matrix of distinct column ids per row, each row sorted."""
    out = np.empty((s, k), dtype=np.int32)
    m = max(2 * k, k + 16)
    for a in range(0, s, batch):
        b = min(s, a + batch)
        todo = np.arange(a, b)
        mm = m
        while todo.size:
            cand = draw(rng, (todo.size, mm))
            cols, ok = _first_k_distinct(cand, k)
            out[todo[ok]] = cols[ok]
            todo = todo[~ok]
            mm *= 2
    return out


def _uniform_draw(n):
    def draw(rng, shape):
        return rng.integers(0, n, size=shape, dtype=np.int64)
    return draw


def _zipf_draw(n, a):
    """Finite Zipf(a) popularity: rank r (1-based) has weight r^-a; rank r -> column r-1."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-a)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]

    def draw(rng, shape):
        u = rng.random(size=shape)
        idx = np.searchsorted(cdf, u, side="right")
        return np.minimum(idx, n - 1).astype(np.int64)
    return draw


def _labels(s, row_ptr, col_idx, csr_val, wstar, noise_sd, flip_p, rng):
    """y_i = sign(x_i . w* [+ N(0, sd^2)]) with sign(0)=+1, then k% independent flips."""
    rows = np.repeat(np.arange(s), np.diff(row_ptr))
    margin = np.bincount(rows, weights=csr_val.astype(np.float64) * wstar[col_idx], minlength=s)
    if noise_sd > 0:
        margin = margin + rng.normal(0.0, noise_sd, size=s)
    y = np.where(margin >= 0.0, 1, -1).astype(np.int8)
    if flip_p > 0:
        flip = rng.random(size=s) < flip_p
        y[flip] = -y[flip]
    return y


def _planted_w(n, k, rng):
    w = np.zeros(n, dtype=np.float64)
    supp = rng.choice(n, size=k, replace=False)
    w[supp] = rng.normal(size=k)
    return w


def _normalize_rows(row_ptr, vals64):
    s = row_ptr.size - 1
    rows = np.repeat(np.arange(s), np.diff(row_ptr))
    nrm = np.sqrt(np.bincount(rows, weights=vals64 * vals64, minlength=s))
    nrm[nrm == 0] = 1.0
    return (vals64 / nrm[rows]).astype(np.float32)


def _assemble(name, s, n, cols_mat_or_csr, vals32, y, c, loss, P, seed, meta):
    if isinstance(cols_mat_or_csr, tuple):
        row_ptr, col_idx = cols_mat_or_csr
    else:
        k = cols_mat_or_csr.shape[1]
        row_ptr = np.arange(s + 1, dtype=np.int64) * k
        col_idx = cols_mat_or_csr.reshape(-1).astype(np.int32)
    col_ptr, row_idx, val = csr_to_csc(s, n, row_ptr, col_idx, vals32)
    meta = dict(meta)
    meta.update(nnz=int(row_ptr[-1]), pos_frac=float((y > 0).mean()),
                empty_cols=int(np.sum(np.diff(col_ptr) == 0)),
                max_col=int(np.max(np.diff(col_ptr))) if n else 0)
    return Problem(name=name, s=s, n=n, col_ptr=col_ptr, row_idx=row_idx, val=val,
                   row_ptr=row_ptr.astype(np.int64), col_idx=col_idx.astype(np.int32),
                   csr_val=vals32.astype(np.float32), y=y, c=float(c), loss=loss, P=int(P),
                   seed=int(seed), meta=meta)


# ----------------------------------------------------------------------------------
# the five BASELINE.json configs
# ----------------------------------------------------------------------------------

def _cfg1(scale=1.0):
    seed = 0
    rng = np.random.default_rng(seed)
    s, n, k = 1000, 2000, 20
    cols = _distinct_rows(s, k, n, _uniform_draw(n), rng)
    v = np.abs(rng.normal(size=s * k))
    row_ptr = np.arange(s + 1, dtype=np.int64) * k
    vals = _normalize_rows(row_ptr, v)
    wstar = _planted_w(n, 50, rng)
    y = _labels(s, row_ptr, cols.reshape(-1), vals, wstar, 0.1, 0.0, rng)
    return _assemble("cfg1", s, n, cols, vals, y, 1.0, LOSS_LOGISTIC, 64, seed,
                     dict(max_outer=20, eps=1e-3))


def _cfg2(scale=1.0):
    seed = 1
    rng = np.random.default_rng(seed)
    s, n, k = 20000, 50000, 50
    cols = _distinct_rows(s, k, n, _uniform_draw(n), rng)
    v = np.abs(rng.normal(size=s * k))
    row_ptr = np.arange(s + 1, dtype=np.int64) * k
    vals = _normalize_rows(row_ptr, v)
    wstar = _planted_w(n, 500, rng)
    y = _labels(s, row_ptr, cols.reshape(-1), vals, wstar, 0.0, 0.05, rng)
    return _assemble("cfg2", s, n, cols, vals, y, 1.0, LOSS_L2SVM, 256, seed,
                     dict(max_outer=1000, eps=1e-3))


def _zero_truncated_poisson(lam, size, rng):
    k = rng.poisson(lam, size=size)
    bad = np.nonzero(k == 0)[0]
    while bad.size:
        k[bad] = rng.poisson(lam, size=bad.size)
        bad = bad[k[bad] == 0]
    return k


def _cfg3(scale=1.0):
    seed = 2
    rng = np.random.default_rng(seed)
    s, n, k = 20000, 1_000_000, 450
    cols = _distinct_rows(s, k, n, _zipf_draw(n, 1.1), rng, batch=4096)
    row_ptr = np.arange(s + 1, dtype=np.int64) * k
    col_idx = cols.reshape(-1)
    tf = np.log1p(_zero_truncated_poisson(2.0, s * k, rng).astype(np.float64))
    df = np.bincount(col_idx, minlength=n).astype(np.float64)
    idf = 1.0 + np.log((1.0 + s) / (1.0 + df))
    vals = _normalize_rows(row_ptr, tf * idf[col_idx])
    wstar = _planted_w(n, 2000, rng)
    y = _labels(s, row_ptr, col_idx, vals, wstar, 0.0, 0.03, rng)
    return _assemble("cfg3", s, n, cols, vals, y, 4.0, LOSS_LOGISTIC, 1024, seed,
                     dict(P_sweep=[1, 64, 1024, 8192], eps=1e-3))


def _cfg4(scale=1.0):
    seed = 3
    rng = np.random.default_rng(seed)
    s, n = 6000, 5000
    X = rng.normal(size=(s, n)).astype(np.float32)  # no normalization
    wstar = _planted_w(n, 100, rng)
    margin = X.astype(np.float64) @ wstar + rng.normal(0.0, 0.5, size=s)
    y = np.where(margin >= 0.0, 1, -1).astype(np.int8)
    row_ptr = np.arange(s + 1, dtype=np.int64) * n
    col_idx = np.tile(np.arange(n, dtype=np.int32), s)
    csr_val = X.reshape(-1)
    col_ptr = np.arange(n + 1, dtype=np.int64) * s
    row_idx = np.tile(np.arange(s, dtype=np.int32), n)
    val = np.ascontiguousarray(X.T).reshape(-1)
    return Problem(name="cfg4", s=s, n=n, col_ptr=col_ptr, row_idx=row_idx, val=val,
                   row_ptr=row_ptr, col_idx=col_idx, csr_val=csr_val, y=y, c=0.5,
                   loss=LOSS_LOGISTIC, P=500, seed=seed,
                   meta=dict(nnz=s * n, pos_frac=float((y > 0).mean()), eps=1e-3))


def _cfg5(scale=1.0):
    seed = 4
    rng = np.random.default_rng(seed)
    s, n, k = int(2_000_000 * scale), int(20_000_000 * scale), 40
    cols = _distinct_rows(s, k, n, _zipf_draw(n, 1.05), rng, batch=1 << 18)
    row_ptr = np.arange(s + 1, dtype=np.int64) * k
    vals = np.full(s * k, 1.0 / np.sqrt(k), dtype=np.float32)
    wstar = _planted_w(n, max(1, int(20000 * scale)), rng)
    y = _labels(s, row_ptr, cols.reshape(-1), vals, wstar, 0.0, 0.05, rng)
    return _assemble("cfg5", s, n, cols, vals, y, 1.0, LOSS_LOGISTIC, 4096, seed,
                     dict(eps=1e-3, scale=scale))


CONFIGS = {1: _cfg1, 2: _cfg2, 3: _cfg3, 4: _cfg4, 5: _cfg5}


def _cache_dir():
    d = os.environ.get("PCDN_SYNTH_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "pcdn_synth"))
    return d


def config(i: int, loss: int | None = None, scale: float = 1.0, cache: bool = True) -> Problem:
    """BASELINE.json configs[i-1] (1-based).

    A cache under ~/.cache/pcdn_synth (or $PCDN_SYNTH_CACHE) only saves time:
    the data is fully determined by (i, scale, GEN_VERSION)."""
    key = f"cfg{i}_s{scale}_v{GEN_VERSION}"
    path = os.path.join(_cache_dir(), key + ".npz")
    p = None
    if cache and i >= 3 and os.path.exists(path):
        try:
            z = np.load(path, allow_pickle=True)
            p = Problem(name=str(z["name"]), s=int(z["s"]), n=int(z["n"]),
                        col_ptr=z["col_ptr"], row_idx=z["row_idx"], val=z["val"],
                        row_ptr=z["row_ptr"], col_idx=z["col_idx"], csr_val=z["csr_val"],
                        y=z["y"], c=float(z["c"]), loss=int(z["loss"]), P=int(z["P"]),
                        seed=int(z["seed"]), meta=z["meta"].item())
        except Exception:
            p = None
    if p is None:
        p = CONFIGS[i](scale) if i == 5 else CONFIGS[i]()
        if cache and i >= 3:
            try:
                os.makedirs(_cache_dir(), exist_ok=True)
                tmp = path + f".tmp{os.getpid()}.npz"
                np.savez(tmp, name=p.name, s=p.s, n=p.n, col_ptr=p.col_ptr, row_idx=p.row_idx,
                         val=p.val, row_ptr=p.row_ptr, col_idx=p.col_idx, csr_val=p.csr_val,
                         y=p.y, c=p.c, loss=p.loss, P=p.P, seed=p.seed,
                         meta=np.array(p.meta, dtype=object))
                os.replace(tmp, path)
            except OSError:
                pass
    if loss is not None and loss != p.loss:
        p = p.with_loss(loss)
    return p


# ----------------------------------------------------------------------------------
# small fixtures for pins and parity
# ----------------------------------------------------------------------------------

def from_dense(X, y, c=1.0, loss=LOSS_LOGISTIC, P=1, name="dense", seed=0, keep_zeros=False) -> Problem:
    """Build a Problem from a dense matrix (float values are cast to fp32 first)."""
    X = np.asarray(X, dtype=np.float32)
    s, n = X.shape
    mask = np.ones_like(X, dtype=bool) if keep_zeros else (X != 0)
    rr, cc = np.nonzero(mask)
    row_ptr = np.zeros(s + 1, dtype=np.int64)
    np.cumsum(np.bincount(rr, minlength=s), out=row_ptr[1:])
    col_idx = cc.astype(np.int32)
    csr_val = X[rr, cc].astype(np.float32)
    col_ptr, row_idx, val = csr_to_csc(s, n, row_ptr, col_idx, csr_val)
    y = np.asarray(y, dtype=np.int8)
    return Problem(name=name, s=s, n=n, col_ptr=col_ptr, row_idx=row_idx, val=val,
                   row_ptr=row_ptr, col_idx=col_idx, csr_val=csr_val, y=y, c=float(c),
                   loss=int(loss), P=int(P), seed=int(seed), meta={})


def tiny(seed: int, s: int, n: int, density: float = 0.2, loss: int = LOSS_LOGISTIC,
         c: float = 1.0, P: int = 4, positive: bool = False, empty_cols: int = 0,
         dup_cols: int = 0, dense_rows: int = 0, planted: bool = True,
         flip: float = 0.1, scale: float = 1.0, full_cols: int = 0) -> Problem:
    """Random small problem with optional nasty structure (empty columns,
    duplicated columns, fully dense rows, full columns = a nonzero in every row)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((s, n)) < density
    vals = rng.normal(size=(s, n)) * scale
    if positive:
        vals = np.abs(vals)
    if dense_rows:
        mask[rng.choice(s, size=min(dense_rows, s), replace=False)] = True
    X = np.where(mask, vals, 0.0)
    if dup_cols and n >= 2:
        for _ in range(dup_cols):
            a, b = rng.choice(n, size=2, replace=False)
            X[:, b] = X[:, a]
    if empty_cols:
        X[:, rng.choice(n, size=min(empty_cols, n), replace=False)] = 0.0
    if full_cols:
        fc = rng.choice(n, size=min(full_cols, n), replace=False)
        v = rng.normal(size=(s, fc.size)) * scale
        X[:, fc] = np.where(v == 0.0, 1.0, v)
    X = X.astype(np.float32)
    if planted:
        wstar = rng.normal(size=n) * (rng.random(n) < 0.3)
        m = X.astype(np.float64) @ wstar
        y = np.where(m >= 0, 1, -1).astype(np.int8)
        fl = rng.random(s) < flip
        y[fl] = -y[fl]
    else:
        y = np.where(rng.random(s) < 0.5, 1, -1).astype(np.int8)
    return from_dense(X, y, c=c, loss=loss, P=P, name=f"tiny{seed}", seed=seed)
