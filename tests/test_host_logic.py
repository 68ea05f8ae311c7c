"""CPU tests of host-side logic that needs no device: the synthetic C5
matrix generator against the reference's from_coo construction, the row
partition's padded gather layout."""

import numpy as np
import pytest

from paper_1309_4616_b200.sparse import CsrMatrix, synthetic_symmetric


@pytest.mark.parametrize("n,r,seed", [(64, 3, 5), (5000, 6, 5), (20000, 6, 1234)])
def test_synthetic_symmetric_equals_from_coo(n, r, seed):
    a = synthetic_symmetric(n, r, seed=seed)
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n, dtype=np.int64), r)
    cols = rng.integers(0, n, size=n * r)
    vals = -rng.random(n * r)
    ar = np.arange(n)
    b = CsrMatrix.from_coo(n, n, np.concatenate([rows, cols, ar]), np.concatenate([cols, rows, ar]),
                           np.concatenate([vals, vals, np.full(n, 12.0)]), sum_duplicates=True)
    a._validate()
    assert np.array_equal(a.row_ptr, b.row_ptr)
    assert np.array_equal(a.col_idx, b.col_idx) and a.col_idx.dtype == np.int32
    assert a.vals.tobytes() == b.vals.tobytes()
    # symmetric by construction
    d = a.to_dense() if n <= 5000 else None
    if d is not None:
        assert np.array_equal(d, d.T)
