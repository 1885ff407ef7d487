"""example-2 on the full-node path, host side (CPU): the product's free-DoF masks,
termwise Galerkin hierarchy, full-node coefficient arrays and mu-dependent right-hand
sides against the unmodified reference's goldens (tests/golden/golden_fem2.npz)."""

from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2311_13862_b200 import fem
from paper_2311_13862_b200.fem_fn import FnFemProblem, fn_coef

G = np.load(Path(__file__).parent / "golden" / "golden_fem2.npz")
CASES = (("n8m2", 3, 2), ("n16m4", 3, 4))


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def case(request):
    tag, levels, m0 = request.param
    return f"fem2_{tag}", FnFemProblem(fem.example2(), levels=levels, m0=m0, host_only=True)


def _golden_op(k, lvl):
    ip = G[f"{k}_op{lvl}_indptr"]
    return sp.csr_matrix((G[f"{k}_op{lvl}_data"], G[f"{k}_op{lvl}_indices"], ip),
                         shape=(len(ip) - 1,) * 2)


def test_free_dofs(case):
    k, p = case
    np.testing.assert_array_equal(p.free_by_level[-1], G[f"{k}_free"])


def test_operators_every_level(case):
    k, p = case
    mu = G[f"{k}_mus"][0]
    for lvl in range(p.levels):
        A, B = p.operator_host(mu, lvl), _golden_op(k, lvl)
        assert A.shape == B.shape
        assert abs(A - B).max() <= 1e-13 * abs(B).max()


def test_full_node_coefficients_round_trip(case):
    """The [27][(c+1)^3] arrays the device combines hold exactly the CSR entries."""
    k, p = case
    for lvl in range(p.levels):
        c = p.cells[lvl]
        free = p.free_by_level[lvl]
        for T in p.terms_by_level[lvl]:
            C = fn_coef(T, free, c)
            assert np.count_nonzero(C) == T.count_nonzero()
            assert np.all(C[:, ~p.masks[lvl]] == 0.0)
            # row sums through the stencil equal the CSR row sums
            np.testing.assert_allclose(C.sum(0)[free], np.asarray(T.sum(1)).ravel(),
                                       rtol=1e-12, atol=1e-15)


def test_rhs(case):
    k, p = case
    f = p.rhs_host(G[f"{k}_mus"])
    ref = G[f"{k}_rhs"]
    np.testing.assert_allclose(f, ref, rtol=1e-13, atol=1e-15 * abs(ref).max())
