"""Pin the oracle's Gauss-Seidel smoother (smoother="gs") against golden vectors of the
real reference (tests/golden/make_golden.py --gs)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import problems as op
from oracle import solvers as so

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_gs.npz"


@pytest.fixture(scope="module")
def ggs():
    return dict(np.load(GOLDEN))


@pytest.mark.parametrize("nu", [1, 2])
def test_gs_vcycle_matches_reference(ggs, nu):
    prob = op.OracleProblem(op.thermal_block((2, 2, 1)), 16, m0=4)
    ctx = so.mg_context_for(prob, ggs["gs_vcycle_tb221_n16_mu"], nu=nu, smoother="gs")
    out = so.mg_vcycle(ggs["gs_vcycle_tb221_n16_in"], ctx)
    ref = ggs[f"gs_vcycle_tb221_n16_nu{nu}_out"]
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("tag,spec,n", [
    ("tb221", op.thermal_block((2, 2, 1)), 16),
    ("smooth6", op.smooth_affine(6), 16),
    ("tb222", op.thermal_block((2, 2, 2)), 32),
])
def test_gs_mgcg_matches_reference(ggs, tag, spec, n):
    prob = op.OracleProblem(spec, n, m0=4)
    key = f"gs_mgcg_{tag}_n{n}"
    delta = float(ggs[key + "_delta"])
    for m, mu in enumerate(ggs[key + "_mus"]):
        A, f = prob.operator(mu), prob.rhs()
        x, rep = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(prob, mu, smoother="gs"),
                               delta=delta, l_max=60)
        assert rep.iterations == int(ggs[key + "_iters"][m])
        ref = ggs[key + "_x"][m]
        assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)


def test_gs_is_sequential_sweep():
    """The vectorised triangular solve equals the row-by-row update of csr_gauss_seidel."""
    prob = op.OracleProblem(op.thermal_block((2, 1, 1)), 8, m0=4)
    A = prob.operator(np.array([0.5, 3.0])).tocsr()
    rng = np.random.default_rng(1)
    b, x0 = rng.standard_normal(A.shape[0]), rng.standard_normal(A.shape[0])
    for fwd in (True, False):
        want = x0.copy()
        rows = range(A.shape[0]) if fwd else range(A.shape[0] - 1, -1, -1)
        for i in rows:
            lo, hi = A.indptr[i], A.indptr[i + 1]
            s, d = 0.0, 0.0
            for jj in range(lo, hi):
                if A.indices[jj] == i:
                    d = A.data[jj]
                else:
                    s += A.data[jj] * want[A.indices[jj]]
            want[i] = (b[i] - s) / d
        got = so.gs_sweep(A, x0.copy(), b, fwd)
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-14)
