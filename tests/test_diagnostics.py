"""Lemma 1(a): the expected largest (X'X)_jj of a random bundle.
The oracle's closed form is pinned by brute force over all P-subsets, the statements of the
lemma, and it pins the product-side formulation used by scripts/p_sweep.py."""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from paper_1306_4080_b200 import diagnostics as dg


@pytest.mark.parametrize("n", [1, 2, 5, 8])
def test_expected_lambda_max_brute_force(n):
    rng = np.random.default_rng(n)
    lam = rng.random(n) * 3.0
    lam[rng.integers(n)] = lam[0]   # a tie
    for P in range(1, n + 1):
        subsets = list(itertools.combinations(range(n), P))
        brute = sum(max(lam[list(s)]) for s in subsets) / len(subsets)
        assert math.isclose(oracle.expected_lambda_max(lam, P), brute, rel_tol=1e-12)
        assert math.isclose(dg.expected_lambda_max(lam, P), brute, rel_tol=1e-12)


def test_lemma1a_statements():
    """E[lambda_bar] increases with P, is constant for constant lambda, E/P decreases with P."""
    prob = synth.config(1)
    lam = oracle.column_sq_norms(prob)
    np.testing.assert_allclose(dg.column_sq_norms(prob.col_ptr, prob.val), lam, rtol=1e-12)
    f = [oracle.expected_lambda_max(lam, P) for P in (1, 2, 4, 16, 64, 256, 1024, 2000)]
    assert all(b >= a - 1e-12 * abs(a) for a, b in zip(f, f[1:]))
    # P = n: the largest lambda; P = 1: the mean (lgamma weights carry ~1e-12 relative rounding)
    assert math.isclose(f[-1], lam.max(), rel_tol=1e-9) and math.isclose(f[0], lam.mean(), rel_tol=1e-9)
    Ps = (1, 2, 4, 16, 64, 256, 1024, 2000)
    r = [v / P for v, P in zip(f, Ps)]
    assert all(b < a for a, b in zip(r, r[1:]))
    for P in (1, 7, 50):
        assert math.isclose(oracle.expected_lambda_max(np.full(50, 2.5), P), 2.5, rel_tol=1e-12)
    for P in (1, 64, 2000):
        assert math.isclose(dg.expected_lambda_max(lam, P), oracle.expected_lambda_max(lam, P), rel_tol=1e-10)
