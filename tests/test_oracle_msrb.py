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
