"""The product's host-side interpolant set-up (paper_1309_4616_b200.matfunc,
SURVEY 8(a) row a6) against the reference's own Leja points and divided
differences (tests/golden/leja.npz, written by the unmodified reference), and
the set-up cache: identical requests return the same interpolant."""

import numpy as np

import paper_1309_4616_b200 as es


def test_product_interpolant_matches_reference_goldens(golden):
    d = golden("leja")
    assert np.array_equal(es.canonical_leja_points(151), d["canonical"])
    for i in range(int(d["ncases"])):
        a, b, s = d[f"i{i}_spec"]
        it = es.make_interpolant(es.SpectralInterval(float(a), float(b)), str(d[f"i{i}_target"]), float(s), 150)
        assert np.array_equal(it.xi, d[f"i{i}_xi"]), i
        # the reference's numpy ops in its order: bitwise on this numpy build
        assert it.dd.tobytes() == np.asarray(d[f"i{i}_dd"], dtype=it.dd.dtype).tobytes(), i


def test_interpolant_cache_returns_identical_object():
    iv = es.SpectralInterval(-3.0, 0.0)
    a = es.make_interpolant(iv, "phi1", -0.5, 40, 1e-9)
    b = es.make_interpolant(es.SpectralInterval(-3.0, 0.0), "phi1", -0.5, 40, 1e-9)
    c = es.make_interpolant(iv, "phi1", -0.5, 40, 1e-8)
    assert a is b and c is not a
    assert np.array_equal(a.dd, c.dd)  # tol does not enter the coefficients
