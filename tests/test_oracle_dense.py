"""Independent validation of the oracle's build-defined exponential
Rosenbrock-Euler step (no reference counterpart) and of
its exponential-Euler step, against dense linear algebra.

Patterns: the reference's own dense oracles (``pkg/tests/oracles.py:109-129``:
phi1 through scipy's expm of the augmented matrix) and its order-of-
convergence check (``pkg/src/expstencil/verify.py:128-151``).  CPU only.
"""

import math

import numpy as np
import pytest

from oracle import oracle as orc

scipy_linalg = pytest.importorskip("scipy.linalg")


def dense_matrix(spec: orc.StencilSpec) -> np.ndarray:
    """A assembled column by column from unit vectors (the stencil itself is
    pinned bitwise to reference goldens elsewhere)."""
    n = spec.n
    cols = [orc.stencil_fused(spec, 1.0, 0.0, np.eye(1, n, j)[0]) for j in range(n)]
    return np.stack(cols, axis=1)


def phi1_apply(m: np.ndarray, v: np.ndarray) -> np.ndarray:
    """phi1(M) v = top-right column of expm([[M, v], [0, 0]])."""
    n = m.shape[0]
    aug = np.zeros((n + 1, n + 1))
    aug[:n, :n] = m
    aug[:n, n] = v
    return scipy_linalg.expm(aug)[:n, n]


def dense_rosenbrock(a: np.ndarray, u: np.ndarray, h: float) -> np.ndarray:
    g = orc.combustion(u)
    gp = orc.combustion_jac(u)
    f = g - a @ u
    m = a - np.diag(gp)
    return u + h * phi1_apply(-h * m, f)


def dense_expeuler(a: np.ndarray, u: np.ndarray, h: float) -> np.ndarray:
    return scipy_linalg.expm(-h * a) @ u + h * phi1_apply(-h * a, orc.combustion(u))


@pytest.mark.parametrize("mode", [orc.MODE_ZERO, orc.MODE_NEUMANN])
@pytest.mark.parametrize("dims", [(6, 5, 4), (9, 7, 1)])
def test_rosenbrock_step_matches_dense_expm(dims, mode, oracle):
    spec = orc.StencilSpec(*dims, mode=mode, coeff_kind=orc.COEFF_RADIAL if dims[2] == 1 else 0)
    a = dense_matrix(spec)
    u = 1.0 + 0.1 * np.random.default_rng(17).random(spec.n)
    for h in (2e-4, 2e-3):
        got, mv = oracle.rosenbrock_step(spec, u, h, 1e-14)
        ref = dense_rosenbrock(a, u, h)
        assert mv > 2
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref)), (dims, mode, h)


def test_jacobian_is_derivative_of_combustion(oracle):
    u = np.linspace(0.6, 2.2, 401)
    eps = 1e-6
    fd = (orc.combustion(u + eps) - orc.combustion(u - eps)) / (2 * eps)
    np.testing.assert_allclose(orc.combustion_jac(u), fd, rtol=1e-7, atol=1e-7)


def test_expeuler_step_matches_dense_expm(oracle):
    spec = orc.StencilSpec(7, 6, 5)
    a = dense_matrix(spec)
    u = 1.0 + 0.1 * np.random.default_rng(19).random(spec.n)
    h = 1e-3
    got, _ = oracle.expeuler_step(spec, u, h, 1e-14)
    ref = dense_expeuler(a, u, h)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def _observed_orders(step, u0, t_end, hs, ref):
    errs = []
    for h in hs:
        u = u0.copy()
        for _ in range(int(round(t_end / h))):
            u = step(u, h)
        errs.append(float(np.max(np.abs(u - ref))))
    return [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)], errs


def test_rosenbrock_is_second_order(oracle):
    # exponential Rosenbrock-Euler is order 2 on autonomous problems; the
    # reference solution is the same scheme at a 64x finer step
    spec = orc.StencilSpec(8, 7, 6)
    u0 = 1.0 + 0.1 * np.random.default_rng(23).random(spec.n)
    t_end = 0.02

    def step(u, h):
        return oracle.rosenbrock_step(spec, u, h, 1e-14)[0]

    hs = (5e-3, 2.5e-3, 1.25e-3)
    ref = u0.copy()
    for _ in range(int(round(t_end / (hs[-1] / 16)))):
        ref = step(ref, hs[-1] / 16)
    orders, errs = _observed_orders(step, u0, t_end, hs, ref)
    assert all(1.8 <= p <= 2.5 for p in orders), (orders, errs)


def test_expeuler_is_first_order(oracle):
    spec = orc.StencilSpec(8, 7, 6)
    u0 = 1.0 + 0.1 * np.random.default_rng(29).random(spec.n)
    t_end = 0.02

    def step(u, h):
        return oracle.expeuler_step(spec, u, h, 1e-14)[0]

    hs = (5e-3, 2.5e-3, 1.25e-3)
    ref = u0.copy()
    for _ in range(int(round(t_end / (hs[-1] / 16)))):
        ref = step(ref, hs[-1] / 16)
    orders, errs = _observed_orders(step, u0, t_end, hs, ref)
    assert all(0.9 <= p <= 1.3 for p in orders), (orders, errs)
