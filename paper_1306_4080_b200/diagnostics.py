"""Diagnostics of the bundle-size choice (Fig. 1).

Not on the hot path: host-side quantities that explain the measured P sweep
(scripts/p_sweep.py).  Lemma 1(a): for a random bundle of P distinct
features the expected largest column norm is
    E[lambda_bar(B)] = sum_{k=P}^{n} lambda_(k) C(k-1, P-1) / C(n, P)
(lambda_(k) ascending), and Eq.15 bounds the iterations to accuracy eps by
T_eps^up proportional to E[lambda_bar(B)] / (P eps).  Here the probabilities
C(k-1, P-1)/C(n, P) are built by a product recurrence over k (an independent formulation of the
oracle's lgamma sum; tests/test_diagnostics.py checks one against the other and brute force)."""
from __future__ import annotations

import numpy as np


def column_sq_norms(col_ptr, val) -> np.ndarray:
    """lambda_j = sum_i x_ij^2 for each CSC column (fp64)."""
    col_ptr = np.asarray(col_ptr, dtype=np.int64)
    v = np.asarray(val, dtype=np.float64)
    n = col_ptr.size - 1
    cols = np.repeat(np.arange(n), np.diff(col_ptr))
    return np.bincount(cols, weights=v * v, minlength=n)


def max_weights(n: int, P: int) -> np.ndarray:
    """w[k-1] = Pr(max of a uniform P-subset of {1..n} is k) = C(k-1,P-1)/C(n,P), k = 1..n."""
    if not 1 <= P <= n:
        raise ValueError("1 <= P <= n")
    w = np.zeros(n)
    # Pr(max = n) = P/n; Pr(max = k-1) / Pr(max = k) = (k-P)/(k-1)
    p = P / n
    for k in range(n, P - 1, -1):
        w[k - 1] = p
        if k > P:
            p *= (k - P) / (k - 1)
    return w


def expected_lambda_max(lam, P: int) -> float:
    lam = np.sort(np.asarray(lam, dtype=np.float64))
    return float(np.dot(max_weights(lam.size, P), lam))
