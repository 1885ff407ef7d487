"""example-2 (the reference's mixed problem: zero-flux face x = 1, anisotropic
piecewise-constant coefficient, mu-dependent source, z-plane smoothers): the oracle
restatement against the unmodified reference's goldens (tests/golden/golden_fem2.npz,
make_golden.py --fem2).  CPU only."""

from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fem as of
from oracle import solvers as so

G = np.load(Path(__file__).parent / "golden" / "golden_fem2.npz")
CASES = (("n8m2", 3, 2), ("n16m4", 3, 4))
SMOOTHERS = (("planejacobi", "auto"), ("planez", "plane-z"), ("jacobi", "jacobi"))


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def case(request):
    tag, levels, m0 = request.param
    return f"fem2_{tag}", of.OracleFemProblem(of.Example2(), levels=levels, m0=m0)


def _golden_op(k, lvl):
    ip = G[f"{k}_op{lvl}_indptr"]
    return sp.csr_matrix((G[f"{k}_op{lvl}_data"], G[f"{k}_op{lvl}_indices"], ip),
                         shape=(len(ip) - 1,) * 2)


def test_free_dofs_keep_the_zero_flux_face(case):
    """Free DoFs = interior + the whole x = n face, its edge nodes included
    (problems.py:63-75 with neumann_face_x1: the face is 'closed', edges stay free)."""
    k, prob = case
    np.testing.assert_array_equal(prob.free_by_level[-1], G[f"{k}_free"])
    n = prob.n
    assert len(prob.free_by_level[-1]) == (n - 1) ** 3 + (n + 1) ** 2


def test_operators_every_level(case):
    k, prob = case
    mu = G[f"{k}_mus"][0]
    for lvl in range(prob.levels):
        A, B = prob.operator(mu, lvl), _golden_op(k, lvl)
        assert A.shape == B.shape
        assert abs(A - B).max() <= 1e-13 * abs(B).max()


def test_mu_dependent_rhs(case):
    k, prob = case
    for mu, f in zip(G[f"{k}_mus"], G[f"{k}_rhs"]):
        np.testing.assert_allclose(prob.rhs(mu), f, rtol=1e-13, atol=1e-15 * abs(f).max())


@pytest.mark.parametrize("key,kind", SMOOTHERS, ids=[s[0] for s in SMOOTHERS])
def test_vcycle(case, key, kind):
    k, prob = case
    ctx = so.mg_context_for(prob, G[f"{k}_mus"][0], smoother=kind)
    ref = G[f"{k}_vcyc_{key}"]
    v = so.mg_vcycle(G[f"{k}_vcyc_b"], ctx)
    assert np.linalg.norm(v - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("key,kind", SMOOTHERS, ids=[s[0] for s in SMOOTHERS])
def test_mgcg(case, key, kind):
    """Zero-init MGCG to 1e-10: same iteration counts, histories and solutions."""
    k, prob = case
    for i, mu in enumerate(G[f"{k}_mus"]):
        A, f = prob.operator(mu), prob.rhs(mu)
        x, rep = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(prob, mu, smoother=kind),
                               delta=1e-10, l_max=80)
        assert rep.iterations == G[f"{k}_{key}_iters"][i]
        h = G[f"{k}_{key}_hist"][i]
        h = h[~np.isnan(h)]
        np.testing.assert_allclose(rep.history, h, rtol=1e-6)
        ref = G[f"{k}_{key}_x"][i]
        assert np.linalg.norm(x - ref) <= 1e-9 * np.linalg.norm(ref)


def test_plane_smoothers_are_grid_independent():
    """The plane smoothers' iteration counts do not grow with the grid (the reason the
    reference defaults to them for the anisotropic problem, multigrid.py:8-11, 183-188);
    point Jacobi's do."""
    a, b = "fem2_n8m2", "fem2_n16m4"
    for key in ("planejacobi", "planez"):
        assert abs(int(G[f"{b}_{key}_iters"].max()) - int(G[f"{a}_{key}_iters"].max())) <= 1
    assert G[f"{b}_jacobi_iters"].min() > G[f"{a}_jacobi_iters"].max()


def test_default_smoother_is_plane_jacobi():
    prob = of.OracleFemProblem(of.Example2(), levels=2, m0=2)
    assert so.default_smoother(prob) == "plane-jacobi"
    ctx = so.mg_context_for(prob, of.Example2.bounds[:, 0], smoother="auto")
    assert ctx.smoother == "plane-jacobi" and ctx.omega == so.PLANE_OMEGA
    prob1 = of.OracleFemProblem(of.Example1(), levels=2, m0=2)
    assert so.default_smoother(prob1) == "jacobi"
