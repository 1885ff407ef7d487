"""smoother="gs" on the GPU (hyperplane-ordered lexicographic Gauss-Seidel) against the
reference's own golden vectors (tests/golden/golden_gs.npz) and the oracle."""

from pathlib import Path

import numpy as np
import pytest

from oracle import problems as op
from oracle import solvers as so

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_gs.npz"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build
    build.build(verbose=False)


@pytest.fixture(scope="module")
def ggs():
    return dict(np.load(GOLDEN))


def _pkg():
    import paper_2311_13862_b200 as pkg
    return pkg


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("nu", [1, 2])
def test_gs_vcycle_matches_reference_golden(ggs, nu):
    pkg = _pkg()
    prob = pkg.ParametricProblem(pkg.thermal_block((2, 2, 1)), levels=3, m0=4)
    mu = ggs["gs_vcycle_tb221_n16_mu"][None]
    ctx = pkg.mg_context_for(prob, mu, nu=nu, smoother="gs")
    out = pkg.mg_vcycle(pkg.to_padded(ggs["gs_vcycle_tb221_n16_in"], 16), ctx)
    got = pkg.from_padded(out, 16, 1)[0]
    assert _rel(got, ggs[f"gs_vcycle_tb221_n16_nu{nu}_out"]) <= 1e-12


@pytest.mark.parametrize("tag,case,n", [("tb221", (2, 2, 1), 16), ("smooth6", "smooth", 16),
                                        ("tb222", (2, 2, 2), 32)])
def test_gs_mgcg_matches_reference_golden(ggs, tag, case, n):
    pkg = _pkg()
    spec = pkg.smooth_affine(6) if case == "smooth" else pkg.thermal_block(case)
    prob = pkg.ParametricProblem(spec, levels=int(np.log2(n // 4)) + 1, m0=4)
    key = f"gs_mgcg_{tag}_n{n}"
    mus, delta = ggs[key + "_mus"], float(ggs[key + "_delta"])
    ctx = pkg.mg_context_for(prob, mus, smoother="gs")
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=delta, l_max=60)
    got = pkg.from_padded(x, n, len(mus))
    for m in range(len(mus)):
        assert abs(reps[m].iterations - int(ggs[key + "_iters"][m])) <= 1
        assert _rel(got[m], ggs[key + "_x"][m]) <= 1e-8
        assert reps[m].config["smoother"] == "gs"


def test_gs_batch_matches_oracle_and_rejects_unknown():
    pkg = _pkg()
    prob = pkg.ParametricProblem(pkg.thermal_block((2, 1, 1)), levels=4, m0=4)
    oprob = op.OracleProblem(op.thermal_block((2, 1, 1)), 32, 4)
    mus = op.sample_mus(op.thermal_block((2, 1, 1)), 5, seed=71)
    ctx = pkg.mg_context_for(prob, mus, nu=2, smoother="gs")
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    got = pkg.from_padded(x, 32, 5)
    for m in range(5):
        A, f = oprob.operator(mus[m]), oprob.rhs()
        xr, rr = so.mgcg_solve(A, f, np.zeros_like(f),
                               so.mg_context_for(oprob, mus[m], nu=2, smoother="gs"),
                               delta=1e-10, l_max=60)
        assert abs(reps[m].iterations - rr.iterations) <= 1
        assert _rel(got[m], xr) <= 1e-8
    with pytest.raises(ValueError):
        pkg.mg_context_for(prob, mus, smoother="plane-jacobi")


def test_smoother_switch_rebuilds_cached_graph():
    """Switching a solved batch from Jacobi to Gauss-Seidel must not replay the cached
    Jacobi PCG graph: the solve equals a fresh Gauss-Seidel context's, bit for bit."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    prob = pkg.ParametricProblem(pkg.thermal_block((2, 2, 1)), levels=3, m0=4)
    mus = op.sample_mus(op.thermal_block((2, 2, 1)), 4, seed=21)
    ctx = pkg.mg_context_for(prob, mus)
    pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)  # caches the graph
    _native.call("rbws_batch_set_smoother", ctx.handle, 1)
    ctx.setup(mus)
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    fresh = pkg.mg_context_for(prob, mus, smoother="gs")
    xr, rr = pkg.mgcg_solve(None, prob.rhs(), None, fresh, delta=1e-10, l_max=60)
    assert [r.iterations for r in reps] == [r.iterations for r in rr]
    assert torch.equal(x, xr)
