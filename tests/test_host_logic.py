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


@pytest.mark.parametrize("kind", ["f64", "f32", "c128"])
def test_field_binary_matches_reference_bytes(golden, kind, tmp_path):
    from paper_1309_4616_b200.errors import EvaluationError
    from paper_1309_4616_b200.grid import Field, Grid3D, read_field_binary, write_field_binary

    d = golden("field_binary")
    g = Grid3D(*(int(v) for v in d[f"{kind}_dims"]))
    ref = d[f"{kind}_bytes"].tobytes()
    path = tmp_path / f"{kind}.bin"
    write_field_binary(Field(g, d[f"{kind}_values"]), path)
    assert path.read_bytes() == ref
    f = read_field_binary(path)
    assert f.grid == g and f.kind == kind and f.values.tobytes() == d[f"{kind}_values"].tobytes()
    path.write_bytes(ref[:-1])
    with pytest.raises(EvaluationError):
        read_field_binary(path)
    path.write_bytes(ref[:10])
    with pytest.raises(EvaluationError):
        read_field_binary(path)


def test_grid_and_field_contracts():
    from paper_1309_4616_b200.errors import GridMismatchError
    from paper_1309_4616_b200.grid import Field, Grid3D, eval_on_grid, linear_index

    g = Grid3D(4, 3, 2)
    assert g == Grid3D(4, 3, 2) and hash(g) == hash(Grid3D(4, 3, 2)) and g != Grid3D(3, 4, 2)
    assert g.shape == (2, 3, 4) and g.n == 24 and g.spacing() == (0.2, 0.25, 1 / 3)
    with pytest.raises(ValueError):
        Grid3D(0, 1, 1)
    with pytest.raises(AttributeError):
        g.nx = 5
    assert linear_index(g, 3, 2, 1) == 23
    with pytest.raises(IndexError):
        linear_index(g, 4, 0, 0)
    with pytest.raises(GridMismatchError):
        Field(g, np.zeros(23))
    x, y, z = g.meshgrid()
    f = eval_on_grid(g, lambda a, b, c: a + 10 * b + 100 * c)
    assert np.array_equal(f.values, (x + 10 * y + 100 * z).reshape(-1))
    pointwise = eval_on_grid(g, lambda a, b, c: float(a) * 2.0)  # scalar-only callable
    assert np.array_equal(pointwise.values, (2.0 * x).reshape(-1))
