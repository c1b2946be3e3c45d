"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these compares the oracle with itself: every expected value is a closed
form, a brute-force/numeric computation written independently here in numpy or
scipy, a value from tests/golden/ (with citation), or an invariant the paper
proves.  Each test names the passage it pins.  CPU only (-m "not gpu").
"""
import json
import math
import os

import numpy as np
import pytest

import synth
from synth import LOSS_L2SVM, LOSS_LOGISTIC

GOLD = os.path.join(os.path.dirname(__file__), "golden")

LOSSES = [LOSS_LOGISTIC, LOSS_L2SVM]


# ------------------------------------------------------------------ numpy references
def np_loss(prob, w, X=None):
    """L(w) = c sum_i phi(y_i x_i'w), Eq.1-3, evaluated densely in numpy."""
    X = prob.dense() if X is None else X
    m = prob.y.astype(np.float64) * (X @ w)
    if prob.loss == LOSS_LOGISTIC:
        return prob.c * np.sum(np.logaddexp(0.0, -m))
    return prob.c * np.sum(np.maximum(0.0, 1.0 - m) ** 2)


def np_F(prob, w, X=None):
    return np_loss(prob, w, X) + np.sum(np.abs(w))


def np_grad(prob, w, X):
    yv = prob.y.astype(np.float64)
    m = yv * (X @ w)
    if prob.loss == LOSS_LOGISTIC:
        coef = -yv / (1.0 + np.exp(m))           # d/dz log(1+e^{-yz}) = -y/(1+e^{yz})
    else:
        coef = -2.0 * yv * np.maximum(0.0, 1.0 - m)
    return prob.c * (X.T @ coef)


# ------------------------------------------------------------------ F (a6, Eq.1-3)
@pytest.mark.parametrize("loss", LOSSES)
def test_objective_at_zero_closed_form(oracle_mod, loss):
    """F(0) = c s ln2 (LR) and c s (SVM) (Eq.2/3 at w=0)."""
    for p in (synth.config(1, loss=loss), synth.tiny(3, 37, 11, c=2.5, loss=loss)):
        o = oracle_mod.Oracle(p)
        F0 = o.objective(np.zeros(p.n))
        want = p.c * p.s * (math.log(2.0) if loss == LOSS_LOGISTIC else 1.0)
        assert abs(F0 - want) <= 1e-12 * want


@pytest.mark.parametrize("loss", LOSSES)
def test_objective_matches_dense_numpy(oracle_mod, loss):
    """Eq.1 from scratch vs an independent dense numpy evaluation, incl. large margins (Z19)."""
    rng = np.random.default_rng(7)
    for seed in range(5):
        p = synth.tiny(seed, 30, 12, density=0.4, loss=loss, c=0.7 + seed, scale=10.0 if seed == 4 else 1.0)
        o = oracle_mod.Oracle(p)
        X = p.dense()
        for _ in range(4):
            w = rng.normal(size=p.n) * (5.0 if seed >= 3 else 0.5)
            assert math.isclose(o.objective(w), np_F(p, w, X), rel_tol=1e-12, abs_tol=1e-12)


# ------------------------------------------------------------------ g, h (a1, Eq.13, App. A.2)
@pytest.mark.parametrize("loss", LOSSES)
def test_gh_at_zero_closed_form(oracle_mod, loss):
    """At w=0: g = -(c/2) X'y, h = (c/4) lambda (LR); g = -2c X'y, h = 2c lambda (SVM)."""
    p = synth.tiny(11, 40, 17, density=0.3, loss=loss, c=1.7, empty_cols=2)
    X = p.dense()
    g, h = oracle_mod.Oracle(p).gh(np.zeros(p.n))
    Xty = X.T @ p.y.astype(np.float64)
    lam = np.sum(X * X, axis=0)
    if loss == LOSS_LOGISTIC:
        g_want, h_want = -(p.c / 2) * Xty, (p.c / 4) * lam
    else:
        g_want, h_want = -2 * p.c * Xty, 2 * p.c * lam
    h_want = np.maximum(h_want, 1e-12)          # reading Z4 (empty columns)
    np.testing.assert_allclose(g, g_want, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(h, h_want, rtol=1e-12, atol=1e-13)


def test_gh_spec_examples(oracle_mod):
    """LR x=[1],y=1,w=0,c=1 -> g=-0.5,h=0.25; SVM -> g=-2,h=2;
    SVM with y w'x = 2 -> g=0, h=nu."""
    for loss, g0, h0 in ((LOSS_LOGISTIC, -0.5, 0.25), (LOSS_L2SVM, -2.0, 2.0)):
        p = synth.from_dense([[1.0]], [1], c=1.0, loss=loss)
        g, h = oracle_mod.Oracle(p).gh(np.zeros(1))
        assert g[0] == g0 and h[0] == h0
    p = synth.from_dense([[1.0]], [1], c=1.0, loss=LOSS_L2SVM)
    g, h = oracle_mod.Oracle(p).gh(np.array([2.0]))
    assert g[0] == 0.0 and h[0] == 1e-12


@pytest.mark.parametrize("loss", LOSSES)
def test_gradient_finite_differences(oracle_mod, loss):
    """g_j = dL/dw_j by central differences of an independent numpy L."""
    rng = np.random.default_rng(5)
    p = synth.tiny(21, 25, 9, density=0.5, loss=loss, c=1.3)
    X = p.dense()
    o = oracle_mod.Oracle(p)
    for _ in range(5):
        w = rng.normal(size=p.n) * 0.4
        g, _ = o.gh(w)
        m = p.y * (X @ w)
        if loss == LOSS_L2SVM and np.min(np.abs(1 - m)) < 1e-3:
            continue
        eps = 1e-6
        fd = np.array([(np_loss(p, w + eps * e, X) - np_loss(p, w - eps * e, X)) / (2 * eps)
                       for e in np.eye(p.n)])
        np.testing.assert_allclose(g, fd, rtol=1e-6, atol=1e-7)


def test_hessian_finite_differences_lr(oracle_mod):
    """h_j = d^2L/dw_j^2 (Eq.13) by central differences of the numpy gradient."""
    rng = np.random.default_rng(6)
    p = synth.tiny(22, 25, 9, density=0.5, loss=LOSS_LOGISTIC, c=0.9)
    X = p.dense()
    o = oracle_mod.Oracle(p)
    for _ in range(5):
        w = rng.normal(size=p.n) * 0.5
        _, h = o.gh(w)
        eps = 1e-5
        fd = np.array([(np_grad(p, w + eps * e, X)[j] - np_grad(p, w - eps * e, X)[j]) / (2 * eps)
                       for j, e in enumerate(np.eye(p.n))])
        np.testing.assert_allclose(h, np.maximum(fd, 1e-12), rtol=1e-6, atol=1e-9)


def test_svm_generalized_hessian_active_set(oracle_mod):
    """App. A.2: h_j = 2c sum_{i: y_i w'x_i < 1} x_ij^2 (strict)."""
    rng = np.random.default_rng(8)
    p = synth.tiny(23, 30, 8, density=0.6, loss=LOSS_L2SVM, c=0.6)
    X = p.dense()
    o = oracle_mod.Oracle(p)
    for _ in range(5):
        w = rng.normal(size=p.n)
        _, h = o.gh(w)
        act = (p.y * (X @ w)) < 1.0
        want = np.maximum(2 * p.c * np.sum((X * X)[act], axis=0), 1e-12)
        np.testing.assert_allclose(h, want, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("loss", LOSSES)
def test_lemma1b_hessian_bounds(oracle_mod, loss):
    """Lemma 1(b): 0 < h_j <= theta c lambda_j (+nu floor)."""
    theta = 0.25 if loss == LOSS_LOGISTIC else 2.0
    rng = np.random.default_rng(9)
    p = synth.tiny(24, 50, 20, density=0.3, loss=loss, c=3.0, empty_cols=3)
    lam = np.sum(p.dense() ** 2, axis=0)
    o = oracle_mod.Oracle(p)
    for _ in range(10):
        _, h = o.gh(rng.normal(size=p.n) * 2)
        assert np.all(h > 0)
        assert np.all(h <= theta * p.c * lam * (1 + 1e-12) + 1e-12)


# ------------------------------------------------------------------ d (a2, Eq.4-5)
def test_newton_dir_spec_examples(oracle_mod):
    """SPEC.md:214-216 (re-derived): (g,h,w)=(-3,2,0)->1; (0.5,1,2)->-1.5; (0,1,0.5)->-0.5."""
    assert oracle_mod.newton_dir(-3.0, 2.0, 0.0) == 1.0
    assert oracle_mod.newton_dir(0.5, 1.0, 2.0) == -1.5
    assert oracle_mod.newton_dir(0.0, 1.0, 0.5) == -0.5


def test_newton_dir_is_1d_minimizer(oracle_mod):
    """Eq.5 is the argmin of Eq.4: brute force over 10^4 random (g,h,w) triples
    by vectorized ternary search of the convex q(d)=g d + h d^2/2 + |w+d|, plus the kink."""
    rng = np.random.default_rng(10)
    N = 10000
    g = rng.normal(size=N) * rng.choice([0.1, 1, 10], size=N)
    h = np.exp(rng.normal(size=N))
    w = rng.normal(size=N) * rng.choice([0, 0.1, 3], size=N)

    def q(d):
        return g * d + 0.5 * h * d * d + np.abs(w + d)

    lo = -(np.abs(g) + 1) / h - np.abs(w) - 1
    hi = -lo
    for _ in range(200):
        m1 = lo + (hi - lo) / 3
        m2 = hi - (hi - lo) / 3
        left = q(m1) <= q(m2)
        hi = np.where(left, m2, hi)
        lo = np.where(left, lo, m1)
    dbf = 0.5 * (lo + hi)
    kink = -w
    dbf = np.where(q(kink) <= q(dbf), kink, dbf)
    d = np.array([oracle_mod.newton_dir(a, b, c) for a, b, c in zip(g, h, w)])
    assert np.all(q(d) <= q(dbf) + 1e-9 * (1 + np.abs(q(dbf))))
    np.testing.assert_allclose(d, dbf, rtol=1e-6, atol=1e-6 * (1 + np.max(np.abs(dbf))))


# ------------------------------------------------------------------ worked example (golden)
def test_worked_example_golden(oracle_mod):
    """tests/golden/worked_example_lr.json (derived by hand, cited there)."""
    gold = json.load(open(os.path.join(GOLD, "worked_example_lr.json")))
    e = gold["expected"]
    pr = gold["problem"]
    p = synth.from_dense([[pr["x"]]], [pr["y"]], c=pr["c"], loss=LOSS_LOGISTIC)
    r = oracle_mod.Oracle(p).step(np.zeros(1), [0])
    for k in ("g", "h", "d", "Delta"):
        assert math.isclose(float(r[k] if np.isscalar(r[k]) else r[k][0]), e[k], rel_tol=1e-14)
    assert math.isclose(r["F_before"], e["F0"], rel_tol=1e-14)
    assert math.isclose(r["lhs"], e["lhs_q0"], rel_tol=1e-12)
    assert math.isclose(r["F_after"], e["F1"], rel_tol=1e-12)
    assert r["q"] == e["q"]


# ------------------------------------------------------------------ Delta (Lemma 1(c))
@pytest.mark.parametrize("loss", LOSSES)
def test_lemma1c_delta_bound_and_monotone(oracle_mod, loss):
    """Lemma 1(c): Delta <= (gamma-1) d'Hd, and the
    accepted step decreases F (checked against numpy F); zero direction -> Delta=0."""
    rng = np.random.default_rng(12)
    for seed in range(6):
        p = synth.tiny(30 + seed, 40, 16, density=0.3, loss=loss, c=2.0)
        X = p.dense()
        o = oracle_mod.Oracle(p)
        w = rng.normal(size=p.n) * 0.3 * (seed % 3)
        B = rng.choice(p.n, size=1 + seed * 2, replace=False)
        r = o.step(w, B)
        assert r["rc"] == 0
        dHd = np.sum(r["h"] * r["d"] ** 2)
        assert r["Delta"] <= -dHd + 1e-12 * (1 + abs(r["Delta"]))
        wn = w.copy()
        wn[B] += r["alpha"] * r["d"]
        assert np_F(p, wn, X) <= np_F(p, w, X) + 1e-12 * np_F(p, w, X)
    # zero direction: huge lambda-equivalent (tiny c) -> every |g|<1 at w=0
    p = synth.tiny(40, 20, 6, density=0.5, loss=loss, c=1e-3)
    r = oracle_mod.Oracle(p).step(np.zeros(p.n), np.arange(p.n))
    assert np.all(r["d"] == 0) and r["Delta"] == 0 and r["q"] == 0 and r["T"].size == 0
    assert r["F_after"] == r["F_before"]


# ------------------------------------------------------------------ T, dx (a3)
@pytest.mark.parametrize("loss", LOSSES)
def test_touched_set_and_dx_dense(oracle_mod, loss):
    """T = rows with a structural nonzero in a column with d_j != 0 (Z8), ascending;
    dx = X_B d_B (Alg.4 l.1) vs dense numpy."""
    rng = np.random.default_rng(13)
    for seed in range(6):
        p = synth.tiny(50 + seed, 45, 20, density=0.15, loss=loss, c=4.0, empty_cols=2, dup_cols=1)
        X = p.dense()
        w = rng.normal(size=p.n) * 0.2
        B = rng.choice(p.n, size=7, replace=False)
        r = oracle_mod.Oracle(p).step(w, B)
        nzB = B[r["d"] != 0]
        S = np.zeros((p.s, p.n), dtype=bool)
        for j in range(p.n):
            S[p.row_idx[p.col_ptr[j]:p.col_ptr[j + 1]], j] = True
        T_want = np.nonzero(S[:, nzB].any(axis=1))[0]
        np.testing.assert_array_equal(r["T"], T_want)
        dx_want = (X[:, B] @ r["d"])[T_want]
        np.testing.assert_allclose(r["dx"], dx_want, rtol=1e-12, atol=1e-14)


# ------------------------------------------------------------------ q, alpha (a4, Eq.6/12)
@pytest.mark.parametrize("loss", LOSSES)
def test_loss_change_matches_direct_phi(oracle_mod, loss):
    """Reading Z7: the per-sample change used by Eq.12 equals phi(m+u)-phi(m),
    computed directly with numpy, including |u|>1 and large margins."""
    rng = np.random.default_rng(14)
    for _ in range(3000):
        z = rng.normal() * rng.choice([0.1, 1, 5, 40])
        y = int(rng.choice([-1, 1]))
        dx = rng.normal() * rng.choice([0.01, 1, 10])
        a = 0.5 ** int(rng.integers(0, 6))
        got = oracle_mod.loss_change(loss, z, y, dx, a)
        m0, m1 = y * z, y * (z + a * dx)
        if loss == LOSS_LOGISTIC:
            want = np.logaddexp(0, -m1) - np.logaddexp(0, -m0)
        else:
            want = max(0.0, 1 - m1) ** 2 - max(0.0, 1 - m0) ** 2
        assert abs(got - want) <= 1e-12 * max(1.0, abs(np.logaddexp(0, -m0)) + abs(want)) + 1e-15


@pytest.mark.parametrize("loss", LOSSES)
def test_line_search_incremental_vs_direct(oracle_mod, loss):
    """Eq.12 (retained quantities) == Eq.6 (direct F): same q; the accepted q passes
    and q-1 fails when re-checked with an independent numpy F."""
    rng = np.random.default_rng(15)
    checked = 0
    for seed in range(25):
        if seed % 2:
            p = synth.tiny(60 + seed, 30, 14, density=0.4, loss=loss, c=float(rng.choice([0.5, 4, 30])))
        else:   # correlated columns: the P-dim step overshoots and backtracks (q > 0)
            Xc = rng.normal(size=(30, 2)) @ rng.normal(size=(2, 14)) + 0.05 * rng.normal(size=(30, 14))
            p = synth.from_dense(Xc, np.where(rng.random(30) < 0.5, 1, -1), c=30.0, loss=loss)
        X = p.dense()
        o = oracle_mod.Oracle(p)
        w = rng.normal(size=p.n) * 0.5
        B = rng.choice(p.n, size=int(rng.integers(1, p.n + 1)), replace=False)
        r0 = o.step(w, B, mode=0)
        r1 = o.step(w, B, mode=1)
        assert r0["rc"] == 0 and r1["rc"] == 0
        assert r0["q"] == r1["q"]
        assert math.isclose(r0["lhs"], r1["lhs"], rel_tol=1e-8, abs_tol=1e-10 * (1 + r0["lhs_abs"]))
        F0 = np_F(p, w, X)
        sig, beta = 0.01, 0.5

        def dec(q):
            a = beta ** q
            wn = w.copy()
            wn[B] += a * r0["d"]
            return np_F(p, wn, X) - F0, sig * a * r0["Delta"]

        lhs, rhs = dec(r0["q"])
        assert lhs <= rhs + 1e-10 * (1 + abs(lhs))
        if r0["q"] > 0:
            lhs, rhs = dec(r0["q"] - 1)
            assert lhs > rhs - 1e-10 * (1 + abs(lhs))
            checked += 1
    assert checked >= 3


@pytest.mark.parametrize("loss", LOSSES)
def test_armijo_interval_property(oracle_mod, loss):
    """F convex along d and phi'(0+) < 0 => the acceptance set is an interval [0, a_bar]:
    every q' > accepted q also passes (numpy direct F)."""
    rng = np.random.default_rng(16)
    for seed in range(10):
        p = synth.tiny(90 + seed, 25, 10, density=0.5, loss=loss, c=10.0)
        X = p.dense()
        w = rng.normal(size=p.n) * 0.2
        B = np.arange(p.n)
        r = oracle_mod.Oracle(p).step(w, B)
        F0 = np_F(p, w, X)
        for q in range(r["q"], r["q"] + 8):
            a = 0.5 ** q
            wn = w.copy()
            wn[B] += a * r["d"]
            assert np_F(p, wn, X) - F0 <= 0.01 * a * r["Delta"] + 1e-10 * F0


@pytest.mark.parametrize("loss", LOSSES)
def test_theorem1_corrected_alpha_bound(oracle_mod, loss):
    """Theorem 1 with the corrected constant of reading Z14:
    alpha >= min(1, beta * 2 h_min (1-sigma+sigma gamma) / (theta c sum_{j in B} lambda_j))."""
    theta = 0.25 if loss == LOSS_LOGISTIC else 2.0
    rng = np.random.default_rng(17)
    for seed in range(40):
        base = rng.normal(size=(30, 3))
        X = base @ rng.normal(size=(3, 10)) + 0.05 * rng.normal(size=(30, 10))   # correlated columns
        y = np.where(rng.random(30) < 0.5, 1, -1)
        c = float(rng.choice([0.1, 1, 10, 100]))
        p = synth.from_dense(X, y, c=c, loss=loss)
        lam = np.sum(p.dense() ** 2, axis=0)
        w = rng.normal(size=10) * 0.1
        B = rng.choice(10, size=int(rng.integers(2, 11)), replace=False)
        r = oracle_mod.Oracle(p).step(w, B)
        nz = r["d"] != 0
        if not nz.any():
            continue
        hmin = np.min(r["h"][nz])
        bound = min(1.0, 0.5 * 2 * hmin * (1 - 0.01) / (theta * c * np.sum(lam[B])))
        assert r["alpha"] >= bound * (1 - 1e-12)


@pytest.mark.parametrize("loss", LOSSES)
def test_separable_bundle_additivity(oracle_mod, loss):
    """Reading Z24: on disjoint column supports, LHS at the accepted alpha equals the sum of
    per-column changes at that alpha (numpy), and min_j q_j <= q <= max_j q_j."""
    rng = np.random.default_rng(18)
    for seed in range(20):
        s, P = 24, 4
        X = np.zeros((s, P))
        rows = rng.permutation(s)
        for j in range(P):
            X[rows[j * 6:(j + 1) * 6], j] = rng.normal(size=6) * 2
        y = np.where(rng.random(s) < 0.5, 1, -1)
        p = synth.from_dense(X, y, c=float(rng.choice([1, 5, 50])), loss=loss)
        Xd = p.dense()
        w = rng.normal(size=P) * 0.3
        o = oracle_mod.Oracle(p)
        r = o.step(w, np.arange(P))
        a = r["alpha"]
        F0 = np_F(p, w, Xd)
        per = 0.0
        for j in range(P):
            wn = w.copy()
            wn[j] += a * r["d"][j]
            per += np_F(p, wn, Xd) - F0
        assert math.isclose(r["lhs"], per, rel_tol=1e-9, abs_tol=1e-12 * (1 + F0))
        qs = [o.step(w, [j])["q"] for j in range(P) if r["d"][j] != 0]
        if qs:
            assert min(qs) <= r["q"] <= max(qs)


# ------------------------------------------------------------------ permutation (a0, Eq.8)
def test_permutation_is_bijection(oracle_mod):
    for n in (1, 2, 3, 4, 5, 17, 64, 65, 1000, 1023, 1025, 4097):
        for seed, k in ((0, 0), (1, 3), (12345, 7)):
            pi = oracle_mod.permutation(seed, k, n)
            assert np.array_equal(np.sort(pi), np.arange(n))


def test_permutation_bundle_sizes():
    """n=5, P=2 -> bundles of sizes 2,2,1; n=P -> one bundle."""
    n, P = 5, 2
    sizes = [min(P, n - t) for t in range(0, n, P)]
    assert sizes == [2, 2, 1]


def test_permutation_uniformity(oracle_mod):
    """'random disjoint partitions': over 20000 (seed,k) draws with n=6,
    each feature lands in the first bundle (P=2) with frequency 1/3 +- 0.02,
    and every (feature, position) cell is within 5 sigma of uniform."""
    n, P, N = 6, 2, 20000
    counts = np.zeros((n, n))
    for r in range(N):
        pi = oracle_mod.permutation(r // 50, r % 50, n)
        counts[pi, np.arange(n)] += 1
    first = counts[:, :P].sum(axis=1) / N
    assert np.all(np.abs(first - P / n) < 0.02)
    e = N / n
    sd = math.sqrt(N * (1 / n) * (1 - 1 / n))
    assert np.all(np.abs(counts - e) < 5 * sd)


def test_permutation_pairwise_independence(oracle_mod):
    """Adjacent positions are not correlated: P(pi(0)=a, pi(1)=b) ~ 1/(n(n-1))."""
    n, N = 5, 20000
    cnt = np.zeros((n, n))
    for r in range(N):
        pi = oracle_mod.permutation(99 + r, 1, n)
        cnt[pi[0], pi[1]] += 1
    off = cnt[~np.eye(n, dtype=bool)]
    e = N / (n * (n - 1))
    assert np.all(np.abs(off - e) < 5 * math.sqrt(e))
    assert np.all(np.diag(cnt) == 0)


def np_mix64(x):
    """SplitMix64's 64-bit finalizer (reading Z2), numpy uint64 (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def np_permutation(seed, k, n):
    """pi_k written out from DESIGN.md reading Z2, independently of oracle/: an 8-round balanced
    Feistel network on 2*hb bits, hb = ceil(ceil(log2 n) / 2) (>= 1), keyed by
    kk = mix64(mix64(seed ^ 0x6A09E667F3BCC909) ^ k) with round keys mix64(kk + (r+1) * golden64),
    round function (L, R) -> (R, L ^ (mix64(key_r ^ R) & mask)), then cycle walking (re-encrypt
    until the value is < n).  Vectorised over all positions t."""
    bits = 0
    while bits < 63 and (1 << bits) < n:
        bits += 1
    hb = max(1, (bits + 1) // 2)
    mask = np.uint64((1 << hb) - 1)
    kk = int(np_mix64(np_mix64(np.uint64((seed ^ 0x6A09E667F3BCC909) & (2**64 - 1))) ^ np.uint64(k)))
    keys = [np_mix64(np.uint64((kk + (r + 1) * 0x9E3779B97F4A7C15) & (2**64 - 1))) for r in range(8)]

    def enc(x):
        L, R = x >> np.uint64(hb), x & mask
        for r in range(8):
            L, R = R, L ^ (np_mix64(keys[r] ^ R) & mask)
        return (L << np.uint64(hb)) | R

    x = enc(np.arange(n, dtype=np.uint64))
    bad = np.nonzero(x >= np.uint64(n))[0]
    while bad.size:
        x[bad] = enc(x[bad])
        bad = bad[x[bad] >= np.uint64(n)]
    return x.astype(np.int64)


def test_permutation_matches_independent_feistel(oracle_mod):
    """Reading Z2 pinned against an independent numpy implementation of the documented
    construction (not a call into oracle/), including a seed >= 2^63 and n = 10^6."""
    for seed, k, n in ((0, 0, 1), (0, 0, 2), (3, 1, 5), (7, 3, 64), (12345, 7, 1000), (2**63 + 5, 11, 4097),
                       (1, 2, 65537), (2, 0, 1000000)):
        np.testing.assert_array_equal(oracle_mod.permutation(seed, k, n), np_permutation(seed, k, n),
                                      err_msg=f"seed={seed} k={k} n={n}")


def test_permutation_known_answer_vectors(oracle_mod):
    """tests/golden/perm_kat.json (scripts/make_perm_kat.py, from oracle/ when it was pinned):
    the oracle still produces the stored vectors, up to n = 2*10^7 (config 5); the numpy
    re-implementation agrees with them where it is cheap."""
    import hashlib
    kat = json.load(open(os.path.join(GOLD, "perm_kat.json")))
    for c in kat["cases"]:
        seed, k, n = int(c["seed"]), c["k"], c["n"]
        pi = oracle_mod.permutation(seed, k, n)
        assert pi[:16].tolist() == c["head"] and pi[-4:].tolist() == c["tail"], (seed, k, n)
        assert hashlib.sha256(pi.astype("<i4").tobytes()).hexdigest() == c["sha256"], (seed, k, n)
        if n <= 50000:
            assert np_permutation(seed, k, n)[:16].tolist() == c["head"]


# ------------------------------------------------------------------ non-default Armijo constants
ARMIJO = [(0.01, 0.5, 0.0), (0.3, 0.7, 0.5), (0.1, 0.9, 0.9)]


@pytest.mark.parametrize("loss", LOSSES)
@pytest.mark.parametrize("gamma", [0.3, 0.9])
def test_delta_gamma_term_at_zero(oracle_mod, loss, gamma):
    """Eq.7 with gamma > 0.  At w = 0 every coordinate of Eq.5's d lies on one
    side of the kink (d_j = -(g_j+1)/h_j >= 0, -(g_j-1)/h_j <= 0, or 0), so the proof of Lemma 1(c)
     holds with equality: Delta = (gamma - 1) sum_j h_j d_j^2.  Both sides from
    independent numpy closed forms at w = 0: g = -(c/2) X'y, h = (c/4) lambda (LR); g = -2c X'y,
    h = 2c lambda (SVM).  A dropped or sign-flipped gamma term fails this."""
    for seed in range(4):
        p = synth.tiny(300 + seed, 40, 12, density=0.4, loss=loss, c=float(1 + 2 * seed))
        X = p.dense()
        yv = p.y.astype(np.float64)
        lam = np.sum(X ** 2, axis=0)
        if loss == LOSS_LOGISTIC:
            g, h = -(p.c / 2) * (X.T @ yv), (p.c / 4) * lam
        else:
            g, h = -2 * p.c * (X.T @ yv), 2 * p.c * lam
        h = np.maximum(h, 1e-12)
        d = np.where(g + 1 <= 0, -(g + 1) / h, np.where(g - 1 >= 0, -(g - 1) / h, 0.0))
        o = oracle_mod.Oracle(p, gamma=gamma)
        B = np.arange(p.n)
        r = o.step(np.zeros(p.n), B)
        want = (gamma - 1) * np.sum(h * d * d)
        assert np.any(d != 0)
        assert math.isclose(r["Delta"], want, rel_tol=1e-12, abs_tol=1e-14), (r["Delta"], want)
        # and Lemma 1(c) as an inequality from a random state
        w = np.random.default_rng(seed).normal(size=p.n) * 0.4
        r = o.step(w, B)
        assert r["Delta"] <= (gamma - 1) * np.sum(r["h"] * r["d"] ** 2) + 1e-12 * (1 + abs(r["Delta"]))


@pytest.mark.parametrize("loss", LOSSES)
@pytest.mark.parametrize("sigma,beta,gamma", ARMIJO)
def test_line_search_nondefault_constants(oracle_mod, loss, sigma, beta, gamma):
    """Eq.6 with non-default sigma, beta, gamma: the incremental decision (Eq.12)
    equals the direct one, the accepted alpha = beta^q (repeated multiplication, Z11) passes and
    the previous candidate fails when re-checked with an independent numpy F, and Delta includes
    gamma sum h d^2."""
    rng = np.random.default_rng(int(sigma * 100) + int(beta * 10) + loss)
    checked = 0
    for seed in range(20):
        Xc = rng.normal(size=(30, 2)) @ rng.normal(size=(2, 12)) + 0.05 * rng.normal(size=(30, 12))
        p = synth.from_dense(Xc, np.where(rng.random(30) < 0.5, 1, -1), c=float(rng.choice([3, 30])), loss=loss)
        X = p.dense()
        o = oracle_mod.Oracle(p, sigma=sigma, beta=beta, gamma=gamma)
        w = rng.normal(size=p.n) * 0.5
        B = rng.choice(p.n, size=int(rng.integers(2, p.n + 1)), replace=False)
        r0, r1 = o.step(w, B, mode=0), o.step(w, B, mode=1)
        assert r0["rc"] == 0 and r0["q"] == r1["q"]
        Fw = np_F(p, w, X)
        # Delta: g d + gamma h d^2 + |w+d| - |w| over the bundle, g and h from numpy
        gn = np_grad(p, w, X)[B]
        Delta = np.sum(gn * r0["d"] + gamma * r0["h"] * r0["d"] ** 2 + np.abs(w[B] + r0["d"]) - np.abs(w[B]))
        assert math.isclose(r0["Delta"], Delta, rel_tol=1e-9, abs_tol=1e-9)

        def alpha(q):
            a = 1.0
            for _ in range(q):
                a *= beta
            return a

        def dec(q):
            wn = w.copy()
            wn[B] += alpha(q) * r0["d"]
            return np_F(p, wn, X) - Fw, sigma * alpha(q) * r0["Delta"]

        assert r0["alpha"] == alpha(r0["q"])
        lhs, rhs = dec(r0["q"])
        assert lhs <= rhs + 1e-10 * (1 + abs(lhs))
        if r0["q"] > 0:
            lhs, rhs = dec(r0["q"] - 1)
            assert lhs > rhs - 1e-10 * (1 + abs(lhs))
            checked += 1
    assert checked >= 3


@pytest.mark.parametrize("loss", LOSSES)
@pytest.mark.parametrize("sigma,beta,gamma", ARMIJO)
def test_theorem1_bound_nondefault_constants(oracle_mod, loss, sigma, beta, gamma):
    """Theorem 1 with reading Z14's corrected constant and the
    paper's (1 - sigma + sigma gamma) factor: alpha >= min(1, beta * 2 h_min (1 - sigma + sigma
    gamma) / (theta c sum_{j in B} lambda_j)) for non-default sigma, beta, gamma."""
    theta = 0.25 if loss == LOSS_LOGISTIC else 2.0
    rng = np.random.default_rng(170 + loss)
    for seed in range(40):
        X = rng.normal(size=(30, 3)) @ rng.normal(size=(3, 10)) + 0.05 * rng.normal(size=(30, 10))
        y = np.where(rng.random(30) < 0.5, 1, -1)
        c = float(rng.choice([0.1, 1, 10, 100]))
        p = synth.from_dense(X, y, c=c, loss=loss)
        lam = np.sum(p.dense() ** 2, axis=0)
        w = rng.normal(size=10) * 0.1
        B = rng.choice(10, size=int(rng.integers(2, 11)), replace=False)
        r = oracle_mod.Oracle(p, sigma=sigma, beta=beta, gamma=gamma).step(w, B)
        nz = r["d"] != 0
        if not nz.any():
            continue
        hmin = np.min(r["h"][nz])
        bound = min(1.0, beta * 2 * hmin * (1 - sigma + sigma * gamma) / (theta * c * np.sum(lam[B])))
        assert r["alpha"] >= bound * (1 - 1e-12)


# ------------------------------------------------------------------ solve (Alg.3)
def test_one_dimensional_closed_forms(oracle_mod):
    """s=1,x=1,y=+1: LR w*=ln(c-1), F*=c ln(c/(c-1)) + ln(c-1); SVM w*=1-1/(2c), F*=1-1/(4c),
    reached in one Newton step (derived from Eq.1-3 by setting the subgradient to 0)."""
    c = 4.0
    p = synth.from_dense([[1.0]], [1], c=c, loss=LOSS_LOGISTIC)
    r = oracle_mod.Oracle(p).solve(1, max_outer=80)
    assert abs(r["w"][0] - math.log(c - 1)) < 1e-10
    assert math.isclose(r["F"], c * math.log(c / (c - 1)) + math.log(c - 1), rel_tol=1e-13)
    for c in (1.0, 3.0):
        p = synth.from_dense([[1.0]], [1], c=c, loss=LOSS_L2SVM)
        r = oracle_mod.Oracle(p).solve(1, max_outer=1)
        assert math.isclose(r["w"][0], 1 - 1 / (2 * c), rel_tol=1e-15)
        assert math.isclose(r["F"], 1 - 1 / (4 * c), rel_tol=1e-15)


@pytest.mark.parametrize("loss", LOSSES)
def test_p1_equals_cdn(oracle_mod, loss):
    """PAPER.md:234 'CDN is a special case of PCDN with bundle size P=1': the PCDN oracle
    at P=1 and the separately coded Alg.1 walk the same iterates."""
    for seed in range(4):
        p = synth.tiny(100 + seed, 30, 12, density=0.3, loss=loss, c=3.0)
        o = oracle_mod.Oracle(p)
        a = o.solve(1, max_outer=6, seed=seed)
        b = o.cdn(seed=seed, max_outer=6, trace=True)
        np.testing.assert_allclose(a["w"], b["w"], rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(a["F_trace"], b["F_trace"], rtol=1e-11)


def _scipy_fstar(p):
    """Independent reference optimum: L-BFGS-B on w = u - v, u, v >= 0 (smooth reformulation)."""
    from scipy.optimize import minimize
    X = p.dense()
    n = p.n

    def f(uv):
        w = uv[:n] - uv[n:]
        gl = np_grad(p, w, X)
        return np_loss(p, w, X) + np.sum(uv), np.concatenate([gl + 1.0, -gl + 1.0])

    r = minimize(f, np.zeros(2 * n), jac=True, method="L-BFGS-B", bounds=[(0, None)] * (2 * n),
                 options=dict(maxiter=50000, maxfun=100000, ftol=1e-16, gtol=1e-13))
    return r.fun


@pytest.mark.parametrize("loss", LOSSES)
def test_global_convergence_all_P_and_scipy(oracle_mod, loss):
    """Global convergence for any P (App. A.5): every P in {1, n/4, n/2, n}
    reaches the same F*, which equals an independent scipy optimum within 1e-6
    (SPEC.md:286, 521); KKT residual -> 0; monotone F (Lemma 1(c))."""
    p = synth.tiny(200, 40, 16, density=0.35, loss=loss, c=2.0)
    o = oracle_mod.Oracle(p)
    ref = _scipy_fstar(p)
    F0 = o.objective(np.zeros(p.n))
    sg0, _ = o.min_norm_subgrad(np.zeros(p.n))
    for P in (1, 4, 8, 16):
        r = o.solve(P, max_outer=400, seed=3)
        assert r["rc"] == 2
        assert abs(r["F"] - ref) <= 1e-6 * abs(ref), (P, r["F"], ref)
        Ft = np.concatenate([[F0], r["F_trace"]])
        assert np.all(np.diff(Ft) <= 1e-12 * F0)
        sg, _ = o.min_norm_subgrad(r["w"])
        assert sg <= 1e-4 * max(sg0, 1.0)


@pytest.mark.parametrize("loss", LOSSES)
def test_maintained_z_matches_recomputed(oracle_mod, loss):
    """Retained w'x_i stays consistent with z = Xw."""
    p = synth.tiny(300, 60, 30, density=0.2, loss=loss, c=5.0)
    o = oracle_mod.Oracle(p)
    r = o.solve(7, max_outer=20, seed=1)
    z = o.compute_z(r["w"])
    np.testing.assert_allclose(r["z"], z, rtol=1e-8, atol=1e-10)
    assert math.isclose(r["F"], np_F(p, r["w"]), rel_tol=1e-12)


def test_stop_rule_eq14(oracle_mod):
    """Eq.14 stop test at outer boundaries: with F* known, gap <= eps stops with OK."""
    p = synth.config(1)
    o = oracle_mod.Oracle(p)
    full = o.solve(p.P, max_outer=60, seed=0)
    fstar = full["F"]
    r = o.solve(p.P, eps=1e-3, fstar=fstar, max_outer=60, seed=0)
    assert r["rc"] == 0 and r["gap"] <= 1e-3
    assert r["outer"] <= full["outer"]
    # the gap at the previous outer boundary was above eps
    if r["outer"] > 1:
        assert (r["outer_F"][-2] - fstar) / fstar > 1e-3


@pytest.mark.parametrize("loss", LOSSES)
def test_no_null_steps_before_convergence(oracle_mod, loss):
    """Reading Z10: an exhausted line search (null step) only happens at fp64 rounding level;
    Theorem 1 says it cannot happen in exact arithmetic.  Until the
    relative gap is below 1e-9 no step may be null."""
    p = synth.tiny(400, 50, 20, density=0.3, loss=loss, c=4.0)
    o = oracle_mod.Oracle(p)
    fstar = o.solve(5, max_outer=600, seed=2)["F"]
    r = o.solve(5, eps=1e-9, fstar=fstar, max_outer=600, seed=2)
    assert r["rc"] == 0 and r["null_steps"] == 0


# ------------------------------------------------------------------ elastic net (NEXT #4, Z25)
# F(w) = c sum_i phi_i + ||w||_1 + (mu/2)||w||_2^2 (PCDN "can be easily
# extended to ... elastic net").  Every expected value below comes from numpy / scipy / a closed
# form written here, never from the oracle.
MUS = [0.5, 3.0]


def np_F_en(prob, w, mu, X=None):
    return np_F(prob, w, X) + 0.5 * mu * float(np.dot(w, w))


@pytest.mark.parametrize("loss", LOSSES)
@pytest.mark.parametrize("mu", MUS)
def test_elastic_objective_and_gradient(oracle_mod, loss, mu):
    """F with the (mu/2)||w||^2 term against numpy; g_j = d(L + mu/2 ||w||^2)/dw_j by central
    differences, h_j = the LR Hessian diagonal + mu (SVM: 2c sum x^2 over I(w) + mu)."""
    rng = np.random.default_rng(71)
    p = synth.tiny(71, 25, 9, density=0.5, loss=loss, c=1.3)
    X = p.dense()
    o = oracle_mod.Oracle(p, mu=mu)
    for _ in range(4):
        w = rng.normal(size=p.n) * 0.4
        assert math.isclose(o.objective(w), np_F_en(p, w, mu, X), rel_tol=1e-12)
        m = p.y * (X @ w)
        if loss == LOSS_L2SVM and np.min(np.abs(1 - m)) < 1e-3:
            continue
        g, h = o.gh(w)
        eps = 1e-6
        sm = lambda v: np_loss(p, v, X) + 0.5 * mu * float(np.dot(v, v))
        fd = np.array([(sm(w + eps * e) - sm(w - eps * e)) / (2 * eps) for e in np.eye(p.n)])
        np.testing.assert_allclose(g, fd, rtol=1e-6, atol=1e-7)
        if loss == LOSS_LOGISTIC:
            s_ = 1.0 / (1.0 + np.exp(-m))
            hd = p.c * ((X * X).T @ (s_ * (1 - s_))) + mu
        else:
            hd = p.c * ((X * X).T @ (2.0 * (1 - m > 0))) + mu
        np.testing.assert_allclose(h, hd, rtol=1e-12)


def test_elastic_one_dimensional_closed_forms(oracle_mod):
    """s=1, x=1, y=+1.  SVM: F = c(1-w)^2 + |w| + mu w^2/2 is quadratic on (0, 1):
    w* = (2c-1)/(2c+mu), reached in one Newton step.  LR: F'(w) = -c/(1+e^w) + 1 + mu w = 0 on
    w > 0, solved here by scipy's brentq (independent of the oracle)."""
    from scipy.optimize import brentq
    for c, mu in ((1.0, 0.5), (3.0, 2.0), (10.0, 0.1)):
        p = synth.from_dense([[1.0]], [1], c=c, loss=LOSS_L2SVM)
        r = oracle_mod.Oracle(p, mu=mu).solve(1, max_outer=1)
        ws = (2 * c - 1) / (2 * c + mu)
        assert math.isclose(r["w"][0], ws, rel_tol=1e-14)
        assert math.isclose(r["F"], c * (1 - ws) ** 2 + ws + 0.5 * mu * ws * ws, rel_tol=1e-14)
    for c, mu in ((4.0, 0.5), (20.0, 3.0)):
        p = synth.from_dense([[1.0]], [1], c=c, loss=LOSS_LOGISTIC)
        r = oracle_mod.Oracle(p, mu=mu).solve(1, max_outer=200)
        ws = brentq(lambda v: -c / (1 + math.exp(v)) + 1 + mu * v, 1e-12, 50.0, xtol=1e-15)
        assert abs(r["w"][0] - ws) < 1e-10
        assert math.isclose(r["F"], c * math.log1p(math.exp(-ws)) + ws + 0.5 * mu * ws * ws, rel_tol=1e-13)


@pytest.mark.parametrize("loss", LOSSES)
@pytest.mark.parametrize("mu", MUS)
def test_elastic_line_search_incremental_vs_direct(oracle_mod, loss, mu):
    """The line search's elastic-net term (Eq.12 from retained quantities + mu a d (w + a d/2))
    against the direct F difference: same accepted q, LHS within rounding, and the accepted q
    re-checked with numpy's F."""
    rng = np.random.default_rng(91)
    for seed in range(12):
        Xc = rng.normal(size=(30, 2)) @ rng.normal(size=(2, 14)) + 0.05 * rng.normal(size=(30, 14))
        p = synth.from_dense(Xc, np.where(rng.random(30) < 0.5, 1, -1), c=30.0, loss=loss)
        X = p.dense()
        o = oracle_mod.Oracle(p, mu=mu)
        w = rng.normal(size=p.n) * 0.5
        B = rng.choice(p.n, size=int(rng.integers(1, p.n + 1)), replace=False)
        r0 = o.step(w, B, mode=0)
        r1 = o.step(w, B, mode=1)
        assert r0["q"] == r1["q"]
        assert math.isclose(r0["lhs"], r1["lhs"], rel_tol=1e-8, abs_tol=1e-10 * (1 + r0["lhs_abs"]))
        a = 0.5 ** r0["q"]
        wn = w.copy()
        wn[B] += a * r0["d"]
        assert np_F_en(p, wn, mu, X) - np_F_en(p, w, mu, X) <= 0.01 * a * r0["Delta"] + 1e-10 * (1 + abs(r0["lhs"]))


def _scipy_fstar_en(p, mu):
    """L-BFGS-B on w = u - v, u, v >= 0 with the (mu/2)||u - v||^2 term."""
    from scipy.optimize import minimize
    X = p.dense()
    n = p.n

    def f(uv):
        w = uv[:n] - uv[n:]
        gl = np_grad(p, w, X) + mu * w
        return np_loss(p, w, X) + np.sum(uv) + 0.5 * mu * float(np.dot(w, w)), np.concatenate([gl + 1.0, -gl + 1.0])

    r = minimize(f, np.zeros(2 * n), jac=True, method="L-BFGS-B", bounds=[(0, None)] * (2 * n),
                 options=dict(maxiter=50000, maxfun=100000, ftol=1e-16, gtol=1e-13))
    return r.fun


@pytest.mark.parametrize("loss", LOSSES)
def test_elastic_global_convergence_and_cdn(oracle_mod, loss):
    """With mu > 0: every P reaches the scipy optimum within 1e-6, F is monotone, the KKT
    residual (with mu w_j in the gradient) -> 0, and P = 1 walks the separately coded CDN's
    iterates (its line search uses the direct (mu/2)((w+ad)^2 - w^2))."""
    mu = 1.5
    p = synth.tiny(210, 40, 16, density=0.35, loss=loss, c=2.0)
    o = oracle_mod.Oracle(p, mu=mu)
    ref = _scipy_fstar_en(p, mu)
    F0 = o.objective(np.zeros(p.n))
    sg0, _ = o.min_norm_subgrad(np.zeros(p.n))
    for P in (1, 5, 16):
        r = o.solve(P, max_outer=300, seed=4)
        assert abs(r["F"] - ref) <= 1e-6 * abs(ref), (P, r["F"], ref)
        Ft = np.concatenate([[F0], r["F_trace"]])
        assert np.all(np.diff(Ft) <= 1e-12 * F0)
        sg, _ = o.min_norm_subgrad(r["w"])
        assert sg <= 1e-4 * max(sg0, 1.0)
    a = o.solve(1, max_outer=5, seed=2)
    b = o.cdn(seed=2, max_outer=5, trace=True)
    np.testing.assert_allclose(a["w"], b["w"], rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(a["F_trace"], b["F_trace"], rtol=1e-11)


# ------------------------------------------------------------------ Lasso (NEXT #4, Z26)
# F(w) = c sum_i (t_i - x_i'w)^2 + ||w||_1 (+ (mu/2)||w||^2): "PCDN ... can be
# easily extended to other problems such as Lasso and elastic net".  References: numpy, closed
# forms, and scikit-learn's coordinate-descent Lasso / ElasticNet (an independent solver).
from synth import LOSS_SQUARED  # noqa: E402


def _reg(seed, s, n, density, c, noise=0.1, support=4):
    p = synth.tiny(seed, s, n, density=density, c=c)
    return synth.regression(p, noise=noise, support=support)


def np_F_sq(p, w, mu=0.0, X=None):
    X = p.dense() if X is None else X
    r = p.t - X @ w
    return p.c * float(np.dot(r, r)) + np.sum(np.abs(w)) + 0.5 * mu * float(np.dot(w, w))


def test_squared_objective_gh(oracle_mod):
    """F, g_j by central differences, h_j = 2c sum_i x_ij^2 (+ mu), against numpy."""
    rng = np.random.default_rng(81)
    for mu in (0.0, 1.0):
        p = _reg(81, 25, 9, 0.5, 1.3)
        X = p.dense()
        o = oracle_mod.Oracle(p, mu=mu)
        for _ in range(4):
            w = rng.normal(size=p.n) * 0.4
            assert math.isclose(o.objective(w), np_F_sq(p, w, mu, X), rel_tol=1e-12)
            g, h = o.gh(w)
            sm = lambda v: p.c * float(np.dot(p.t - X @ v, p.t - X @ v)) + 0.5 * mu * float(np.dot(v, v))
            eps = 1e-6
            fd = np.array([(sm(w + eps * e) - sm(w - eps * e)) / (2 * eps) for e in np.eye(p.n)])
            np.testing.assert_allclose(g, fd, rtol=1e-6, atol=1e-7)
            np.testing.assert_allclose(h, 2 * p.c * np.sum(X * X, axis=0) + mu, rtol=1e-13)


def test_squared_one_dimensional_closed_form(oracle_mod):
    """s=1, x=1: F = c(t - w)^2 + |w| has w* = soft(t, 1/(2c)) = sign(t) max(|t| - 1/(2c), 0),
    reached in one Newton step (a quadratic)."""
    for t, c in ((2.0, 1.0), (-3.0, 0.5), (0.2, 1.0), (5.0, 10.0)):
        p = synth.from_dense([[1.0]], [1], c=c)
        p = synth.regression(p, noise=0.0, support=1)
        p.t = np.array([t])
        r = oracle_mod.Oracle(p).solve(1, max_outer=1)
        ws = math.copysign(max(abs(t) - 1 / (2 * c), 0.0), t)
        assert abs(r["w"][0] - ws) <= 1e-15 * max(1.0, abs(ws))
        assert math.isclose(r["F"], c * (t - ws) ** 2 + abs(ws), rel_tol=1e-14)


@pytest.mark.parametrize("mu", [0.0, 0.8])
def test_squared_matches_sklearn(oracle_mod, mu):
    """The oracle's optimum equals scikit-learn's (an independent coordinate-descent solver):
    Lasso(alpha) minimises (1/2s)||t - Xw||^2 + alpha ||w||_1, i.e. our F with c = 1/(2 s alpha);
    ElasticNet(alpha, l1_ratio=rho) gives c = 1/(2 s alpha rho), mu = (1 - rho)/rho.  Every P
    reaches it (global convergence); P = 1 walks the separately coded CDN."""
    from sklearn.linear_model import ElasticNet, Lasso
    p = _reg(91, 60, 20, 0.4, 1.0, noise=0.2, support=6)
    X = p.dense()
    s_ = p.s
    if mu == 0.0:
        alpha = 0.02
        p.c = 1.0 / (2 * s_ * alpha)
        m = Lasso(alpha=alpha, fit_intercept=False, tol=1e-14, max_iter=1000000).fit(X, p.t)
    else:
        rho = 1.0 / (1.0 + mu)
        alpha = 0.02 / rho
        p.c = 1.0 / (2 * s_ * alpha * rho)
        m = ElasticNet(alpha=alpha, l1_ratio=rho, fit_intercept=False, tol=1e-14, max_iter=1000000).fit(X, p.t)
    ref = np_F_sq(p, m.coef_, mu, X)
    o = oracle_mod.Oracle(p, mu=mu)
    for P in (1, 5, 20):
        r = o.solve(P, max_outer=600, seed=2)
        assert abs(r["F"] - ref) <= 1e-7 * abs(ref), (P, r["F"], ref)
        np.testing.assert_allclose(r["w"], m.coef_, atol=1e-5)
    a = o.solve(1, max_outer=4, seed=6)
    b = o.cdn(seed=6, max_outer=4, trace=True)
    np.testing.assert_allclose(a["w"], b["w"], rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(a["F_trace"], b["F_trace"], rtol=1e-11)


def test_squared_line_search_incremental_vs_direct(oracle_mod):
    """a dx (a dx + 2(z - t)) summed over T (the Z26 summand) against the direct F difference."""
    rng = np.random.default_rng(93)
    for seed in range(10):
        Xc = rng.normal(size=(30, 2)) @ rng.normal(size=(2, 14)) + 0.05 * rng.normal(size=(30, 14))
        p = synth.regression(synth.from_dense(Xc, np.ones(30), c=5.0), noise=0.3, support=4, seed=seed)
        o = oracle_mod.Oracle(p)
        w = rng.normal(size=p.n) * 0.5
        B = rng.choice(p.n, size=int(rng.integers(1, p.n + 1)), replace=False)
        r0 = o.step(w, B, mode=0)
        r1 = o.step(w, B, mode=1)
        assert r0["q"] == r1["q"]
        assert math.isclose(r0["lhs"], r1["lhs"], rel_tol=1e-8, abs_tol=1e-10 * (1 + r0["lhs_abs"]))


# ------------------------------------------------------------------ SCDN (NEXT #3, Z27)
@pytest.mark.parametrize("loss", LOSSES)
def test_scdn_pbar1_is_cdn(oracle_mod, loss):
    """Alg.2 with P-bar = 1 updates one coordinate at a time with its own 1-D Armijo step: it IS
    the separately coded CDN (Alg.1), iterate for iterate."""
    for seed in range(3):
        p = synth.tiny(300 + seed, 30, 12, density=0.3, loss=loss, c=3.0)
        o = oracle_mod.Oracle(p)
        a = o.scdn(1, seed=seed, max_outer=5)
        b = o.cdn(seed=seed, max_outer=5, trace=True)
        np.testing.assert_allclose(a["w"], b["w"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(a["F_trace"], b["F_trace"], rtol=1e-12)


@pytest.mark.parametrize("loss", LOSSES)
def test_scdn_can_increase_F_where_pcdn_cannot(oracle_mod, loss):
    """with correlated features SCDN's parallel updates (no joint line search) can
    increase F; PCDN on the same bundles is monotone (Lemma 1(c) + the P-dim Armijo rule).  Each
    SCDN update alone passes its own Armijo test (checked with numpy)."""
    rng = np.random.default_rng(7)
    Xc = rng.normal(size=(40, 1)) @ np.ones((1, 16)) + 0.02 * rng.normal(size=(40, 16))   # near-duplicate columns
    p = synth.from_dense(Xc, np.where(rng.random(40) < 0.5, 1, -1), c=10.0, loss=loss)
    o = oracle_mod.Oracle(p)
    F0 = o.objective(np.zeros(p.n))
    sc = o.scdn(16, seed=1, max_outer=3)
    Fs = np.concatenate([[F0], sc["F_trace"]])
    assert np.any(np.diff(Fs) > 1e-9 * F0)          # SCDN rises somewhere
    pc = o.solve(16, seed=1, max_outer=3)
    Fp = np.concatenate([[F0], pc["F_trace"]])
    assert np.all(np.diff(Fp) <= 1e-12 * F0)         # PCDN never does
    # and the one-dimensional steps of the first SCDN iteration each pass Armijo alone
    X = p.dense()
    w = np.zeros(p.n)
    g, h = o.gh(w)
    for j in range(p.n):
        d = oracle_mod.newton_dir(g[j], h[j], 0.0)
        delta = g[j] * d + abs(d)
        if d == 0.0:
            continue
        ok = False
        for q in range(51):
            a = 0.5 ** q
            e = np.zeros(p.n)
            e[j] = a * d
            if np_F(p, e, X) - np_F(p, w, X) <= 0.01 * a * delta + 1e-12:
                ok = True
                break
        assert ok
