"""Host-side logic on CPU: separable tables and the native Kronecker/Galerkin
factors reproduce the oracle's directly assembled, scipy-coarsened operators."""

import ctypes

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import problems as op
from paper_2311_13862_b200 import _native, problems as pp


def native_factors(spec, n, m0, level):
    face, node = spec.separable_tables(n)
    cells = [m0 * 2 ** i for i in range(int(np.log2(n // m0)) + 1)]
    nl = cells[level]
    out = np.zeros((spec.n_terms, 3, 3, 2, nl + 1))
    _native.call("rbws_kron_factors", n, m0, spec.n_terms, face.ctypes.data, node.ctypes.data,
                 level, out.ctypes.data, out.size)
    return out


def tri(diag, up, n):
    m = n - 1
    d = diag[1:n]
    u = up[1:n - 1]
    return sp.diags([u, d, u], [-1, 0, 1], shape=(m, m))


def operator_from_factors(fac, theta, n):
    A = None
    for q in range(fac.shape[0]):
        for d in range(3):
            X = tri(fac[q, d, 0, 0], fac[q, d, 0, 1], n)
            Y = tri(fac[q, d, 1, 0], fac[q, d, 1, 1], n)
            Z = tri(fac[q, d, 2, 0], fac[q, d, 2, 1], n)
            T = theta[q] * sp.kron(sp.kron(Z, Y), X)
            A = T if A is None else A + T
    return A.tocsr()


@pytest.mark.parametrize("pspec,ospec,n,m0", [
    (pp.thermal_block((2, 2, 1)), op.thermal_block((2, 2, 1)), 16, 4),
    (pp.thermal_block((2, 2, 2)), op.thermal_block((2, 2, 2)), 16, 2),
    (pp.smooth_affine(6), op.smooth_affine(6), 16, 4),
])
def test_factors_reproduce_all_levels(pspec, ospec, n, m0):
    oprob = op.OracleProblem(ospec, n, m0)
    mu = op.sample_mus(ospec, 1, seed=3)[0]
    theta = ospec.theta(mu)
    for lvl in range(oprob.levels):
        nl = oprob.cells[lvl]
        A = operator_from_factors(native_factors(pspec, n, m0, lvl), theta, nl)
        ref = oprob.operator(mu, level=lvl)
        err = abs(A - ref).max()
        assert err <= 1e-13 * abs(ref).max(), (lvl, err)


def test_rhs_and_thetas_match_oracle():
    for pspec, ospec in ((pp.thermal_block((2, 2, 1)), op.thermal_block((2, 2, 1))),
                         (pp.smooth_affine(6), op.smooth_affine(6))):
        mus = pp.sample_mus(pspec, 5, seed=9)
        np.testing.assert_array_equal(mus, op.sample_mus(ospec, 5, seed=9))
        np.testing.assert_array_equal(pspec.thetas(mus)[2], ospec.theta(mus[2]))


def test_bounds_rejected():
    spec = pp.thermal_block((2, 1, 1))
    with pytest.raises(ValueError):
        spec.check_mus([[0.01, 1.0]])
    with pytest.raises(ValueError):
        spec.check_mus([[1.0, 1.0, 1.0]])


def test_kron_factor_errors():
    spec = pp.thermal_block((2, 1, 1))
    face, node = spec.separable_tables(16)
    out = np.zeros(10)
    with pytest.raises(_native.NativeError):
        _native.call("rbws_kron_factors", 16, 3, 2, face.ctypes.data, node.ctypes.data, 0,
                     out.ctypes.data, out.size)
