"""The propagate path on the CPU side: the oracle's complex CSR restatement
and the Matrix Market reader/writer, pinned against fixtures the reference
produced (tests/golden/make_golden.py: csr_complex_cases)."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1309_4616_b200.errors import MatrixMarketError
from paper_1309_4616_b200.mmio import read_matrix_market, write_matrix_market

MATS = ("real", "herm")


def _csr(d, name):
    n = len(d[f"{name}_row_ptr"]) - 1
    return orc.Csr(n, d[f"{name}_row_ptr"], d[f"{name}_col"].astype(np.int32), d[f"{name}_vals"])


def _series(d, name):
    for k in range(int(d[f"{name}_nseries"])):
        key = f"{name}_s{k}"
        a, b, tol, mv = d[key + "_meta"]
        yield key, float(a), float(b), float(tol), int(mv), str(d[key + "_axis"]), d[key + "_dd"], d[key + "_xi"]


@pytest.mark.parametrize("name", MATS)
def test_oracle_complex_rows_bitwise(golden, oracle, name):
    d = golden("csr_complex")
    a = _csr(d, name)
    assert oracle.csr_fused_z(a, 0.7 - 0.2j, -1.3, d["x"]).tobytes() == d[f"{name}_y"].tobytes()
    assert oracle.csr_fused_z(a, 1.0, 0.0, d["x"], use_beta=False).tobytes() == d[f"{name}_spmv"].tobytes()


@pytest.mark.parametrize("name", MATS)
def test_oracle_complex_series_bitwise(golden, oracle, name):
    d = golden("csr_complex")
    a = _csr(d, name)
    for key, lo, hi, tol, mv_ref, axis, dd, xi in _series(d, name):
        gamma, center = 0.25 * (hi - lo), 0.5 * (lo + hi)
        alpha = (-1j / gamma) if axis == "imag" else 1.0 / gamma
        p, mv = oracle.newton_csr_z(a, dd, xi, center, gamma, alpha, d["x"], tol)
        assert mv == mv_ref, key
        assert p.tobytes() == d[key + "_p"].tobytes(), key


def test_matrix_market_reader_matches_reference(golden, tmp_path):
    d = golden("csr_complex")
    for name in d["mm_good"]:
        path = tmp_path / f"{name}.mtx"
        path.write_text(str(d[f"mm_{name}_text"]))
        a = read_matrix_market(path)
        assert [a.nrows, a.ncols] == list(d[f"mm_{name}"]), name
        assert np.array_equal(a.row_ptr, d[f"mm_{name}_row_ptr"]), name
        assert np.array_equal(a.col_idx, d[f"mm_{name}_col"]), name
        assert a.vals.dtype == d[f"mm_{name}_vals"].dtype and a.vals.tobytes() == d[f"mm_{name}_vals"].tobytes()
    for name in d["mm_bad"]:
        path = tmp_path / f"bad_{name}.mtx"
        path.write_text(str(d[f"mmbad_{name}_text"]))
        with pytest.raises(MatrixMarketError) as ei:
            read_matrix_market(path)
        assert ei.value.line == int(d[f"mmbad_{name}_line"]), name
        assert str(ei.value) == str(d[f"mmbad_{name}_msg"]), name


def test_matrix_market_empty_and_roundtrip(golden, tmp_path):
    empty = tmp_path / "empty.mtx"
    empty.write_text("")
    with pytest.raises(MatrixMarketError) as ei:
        read_matrix_market(empty)
    assert ei.value.line == 1
    d = golden("csr_complex")
    from paper_1309_4616_b200.sparse import CsrMatrix

    for name in MATS:
        n = len(d[f"{name}_row_ptr"]) - 1
        a = CsrMatrix(n, n, d[f"{name}_row_ptr"], d[f"{name}_col"], d[f"{name}_vals"])
        path = tmp_path / f"{name}.mtx"
        write_matrix_market(a, path, comment="roundtrip")
        b = read_matrix_market(path)
        assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
        assert a.vals.tobytes() == b.vals.tobytes()  # 17 significant digits round-trip exactly
