"""Pin the oracle's multispace RB preconditioner (rbi-msrbcg) against golden vectors of the
real reference (tests/golden/make_golden.py --msrb)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import msrb as om
from oracle import problems as op
from oracle import solvers as so

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_msrb.npz"


@pytest.fixture(scope="module")
def gm():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="module")
def trained(gm):
    prob = op.OracleProblem(op.thermal_block((2, 2, 1)), 16, 4)

    def hf(mu, rhs=None):
        A = prob.operator(mu)
        import scipy.sparse.linalg as spla
        return spla.spsolve(A.tocsc(), prob.rhs() if rhs is None else rhs)

    N, K = (int(v) for v in gm["msrb_tb221_n16_NK"])
    hier = om.msrb_train(list(gm["msrb_tb221_n16_train"]), N, K, hf, prob.operator,
                         lambda mu: prob.rhs())
    return prob, hier


def _span_err(A, B):
    """Largest principal-angle sine between the column spans of A and B (orthonormal)."""
    return np.linalg.norm(A - B @ (B.T @ A), 2)


def test_pod_bases_match_reference(gm, trained):
    _, hier = trained
    ref = gm["msrb_tb221_n16_init"]
    assert hier.init_basis.basis.shape == ref.shape
    np.testing.assert_allclose(hier.init_basis.eigenvalues[:10], gm["msrb_tb221_n16_init_eig"][:10],
                               rtol=1e-9)
    assert _span_err(hier.init_basis.basis, ref) <= 1e-8
    for k, W in enumerate(hier.bases):
        assert _span_err(W, gm[f"msrb_tb221_n16_basis{k}"]) <= 1e-6, k


def test_rbi_msrbcg_matches_reference(gm, trained):
    prob, hier = trained
    for m, mu in enumerate(gm["msrb_tb221_n16_test"]):
        A, f = prob.operator(mu), prob.rhs()
        x, rep = om.rbi_msrbcg_solve(A, f, hier, delta=1e-10, l_max=60)
        assert abs(rep.iterations - int(gm["msrb_tb221_n16_iters"][m])) <= 1
        h = gm["msrb_tb221_n16_hist"][m]
        np.testing.assert_allclose(rep.history[:8], h[:8], rtol=1e-6)
        assert np.linalg.norm(x - gm["msrb_tb221_n16_x"][m]) <= 1e-6 * np.linalg.norm(x)


# ---- the same method on the reference's assembled problem example-1 (per-parameter right-hand
# sides): goldens from the unmodified reference, make_golden.py --msrb-fem
GOLDEN_FEM = Path(__file__).resolve().parent / "golden" / "golden_msrb_fem.npz"


@pytest.fixture(scope="module")
def trained_fem():
    from oracle import fem as of
    g = dict(np.load(GOLDEN_FEM))
    prob = of.OracleFemProblem(of.Example1(), levels=3, m0=4)

    def hf(mu, rhs=None):
        import scipy.sparse.linalg as spla
        return spla.spsolve(prob.operator(mu).tocsc(), prob.rhs(mu) if rhs is None else rhs)

    N, K = (int(v) for v in g["msrb_ex1_n16_NK"])
    hier = om.msrb_train(list(g["msrb_ex1_n16_train"]), N, K, hf, prob.operator, prob.rhs)
    return prob, hier, g


def test_example1_pod_bases_match_reference(trained_fem):
    _, hier, g = trained_fem
    np.testing.assert_allclose(hier.init_basis.eigenvalues[:6], g["msrb_ex1_n16_init_eig"][:6],
                               rtol=1e-9)
    assert _span_err(hier.init_basis.basis, g["msrb_ex1_n16_init"]) <= 1e-8
    for k, W in enumerate(hier.bases):
        assert _span_err(W, g[f"msrb_ex1_n16_basis{k}"]) <= 1e-6, k


def test_example1_rbi_msrbcg_matches_reference(trained_fem):
    prob, hier, g = trained_fem
    for m, mu in enumerate(g["msrb_ex1_n16_test"]):
        x, rep = om.rbi_msrbcg_solve(prob.operator(mu), prob.rhs(mu), hier, delta=1e-10, l_max=60)
        assert abs(rep.iterations - int(g["msrb_ex1_n16_iters"][m])) <= 1
        np.testing.assert_allclose(rep.history[:8], g["msrb_ex1_n16_hist"][m][:8], rtol=1e-6)
        assert np.linalg.norm(x - g["msrb_ex1_n16_x"][m]) <= 1e-8 * np.linalg.norm(x)
