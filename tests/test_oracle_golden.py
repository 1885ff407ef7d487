"""Pin the CPU oracle against golden vectors produced by the real reference.

tests/golden/make_golden.py runs the reference package (rbws, Cython backend)
on the same FV problems; these tests prove the oracle restatement reproduces it
before it is trusted as the checker for the CUDA path.
"""

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import problems as op
from oracle import solvers as so


def test_operators_all_levels(golden):
    spec = op.thermal_block((2, 1, 1))
    prob = op.OracleProblem(spec, 8, m0=2)
    mu = golden["ops_tb211_n8_mu"]
    for lvl in range(prob.levels):
        A = prob.operator(mu, level=lvl).toarray()
        ref = golden[f"ops_tb211_n8_l{lvl}"]
        assert A.shape == ref.shape
        assert np.max(np.abs(A - ref)) <= 1e-14 * np.max(np.abs(ref))
    np.testing.assert_array_equal(prob.rhs(mu), golden["ops_tb211_n8_rhs"])


def test_vcycle_matches_reference(golden):
    prob = op.OracleProblem(op.thermal_block((2, 2, 1)), 16, m0=4)
    ctx = so.mg_context_for(prob, golden["vcycle_tb221_n16_mu"])
    out = so.mg_vcycle(golden["vcycle_tb221_n16_in"], ctx)
    ref = golden["vcycle_tb221_n16_out"]
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("tag,spec,n", [
    ("tb211", op.thermal_block((2, 1, 1)), 16),
    ("tb221", op.thermal_block((2, 2, 1)), 32),
    ("tb222", op.thermal_block((2, 2, 2)), 16),
    ("smooth6", op.smooth_affine(6), 16),
])
def test_mgcg_matches_reference(golden, tag, spec, n):
    prob = op.OracleProblem(spec, n, m0=4)
    key = f"mgcg_{tag}_n{n}"
    delta = float(golden[key + "_delta"])
    for m, xr, hr, it in zip(golden[key + "_mus"], golden[key + "_x"],
                             golden[key + "_hist"], golden[key + "_iters"]):
        A, f = prob.operator(m), prob.rhs(m)
        x, rep = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(prob, m),
                               delta=delta, l_max=60)
        assert rep.iterations == it
        h = np.asarray(rep.history)
        np.testing.assert_allclose(h[:6], hr[:6], rtol=1e-9)
        assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)


def test_l1roc_offline_online_matches_reference(golden):
    spec = op.thermal_block((2, 2, 1))
    prob = op.OracleProblem(spec, 16, m0=4)
    train = golden["l1roc_tb221_n16_train"]

    def hf(m):
        return spla.splu(prob.operator(m).tocsc()).solve(prob.rhs(m))

    model = so.l1roc_offline(list(train), 6, hf, prob.operator, prob.operator_rows,
                             prob.rhs, seed=3)
    np.testing.assert_array_equal(model.collocation, golden["l1roc_tb221_n16_colloc"])
    np.testing.assert_array_equal(model.solution_points, golden["l1roc_tb221_n16_xs"])
    np.testing.assert_array_equal(model.residual_points, golden["l1roc_tb221_n16_xr"])
    np.testing.assert_array_equal(train[model.chosen], golden["l1roc_tb221_n16_chosen_mus"])
    W = golden["l1roc_tb221_n16_W"]
    assert np.max(np.abs(model.basis - W)) <= 1e-9 * np.max(np.abs(W))
    np.testing.assert_allclose(model.transform, golden["l1roc_tb221_n16_T"], rtol=1e-8, atol=1e-14)
    np.testing.assert_allclose(model.indicator_history, golden["l1roc_tb221_n16_hist"], rtol=1e-8)
    assert bool(model.saturated) == bool(golden["l1roc_tb221_n16_saturated"])
    for i, m in enumerate(golden["l1roc_tb221_n16_test"]):
        A, f = prob.operator(m), prob.rhs(m)
        u0, c, _ = so.l1roc_online(model, A, f)
        ref = golden["l1roc_tb221_n16_u0"][i]
        assert np.linalg.norm(u0 - ref) <= 1e-9 * np.linalg.norm(ref)
        np.testing.assert_allclose(c, golden["l1roc_tb221_n16_c"][i], rtol=1e-7, atol=1e-12)
        x, rep = so.rbi_mgcg_solve(prob, m, model, delta=1e-10, l_max=60)
        assert rep.iterations == golden["rbi_tb221_n16_iters"][i]
        xr = golden["rbi_tb221_n16_x"][i]
        assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)


def test_l1roc_saturation_matches_reference(golden):
    spec = op.thermal_block((2, 1, 1))
    prob = op.OracleProblem(spec, 16, m0=4)

    def hf(m):
        return spla.splu(prob.operator(m).tocsc()).solve(prob.rhs(m))

    model = so.l1roc_offline(list(golden["l1roc_tb211_n16_train"]), 8, hf, prob.operator,
                             prob.operator_rows, prob.rhs, seed=0)
    assert model.saturated and bool(golden["l1roc_tb211_n16_saturated"])
    np.testing.assert_array_equal(model.collocation, golden["l1roc_tb211_n16_colloc"])
    np.testing.assert_allclose(model.indicator_history, golden["l1roc_tb211_n16_hist"], rtol=1e-8)


# known-answer cases the reference's own unit tests hold (tests/test_rb.py, test_krylov.py)
def test_deim_known_answers():
    col, idx, _, _ = so.deim_extend(None, [], np.array([1.0, 3.0, 2.0]))
    assert idx == 1 and np.allclose(col, [1 / 3, 1.0, 2 / 3])
    e0 = np.array([1.0, 0.0, 0.0])
    col, idx, c, _ = so.deim_extend(e0[:, None], [0], np.array([1.0, 1.0, 0.0]))
    assert np.allclose(c, [1.0]) and idx == 1 and np.allclose(col, [0, 1, 0])
    with pytest.raises(so.DegenerateBasisError):
        so.deim_extend(e0[:, None], [0], e0)
    _, idx, _, _ = so.deim_extend(None, [], np.array([1.0, 3.0, 2.0]), exclude={1})
    assert idx == 2


def test_pcg_known_answers():
    import scipy.sparse as sp
    A = sp.diags([1.0, 2.0, 3.0]).tocsr()
    x, rep = so.pcg_solve(A, np.array([1.0, 2.0, 3.0]), np.zeros(3), delta=1e-12)
    assert rep.iterations <= 3 and np.allclose(x, 1.0, atol=1e-10)
    x, rep = so.pcg_solve(sp.eye(7).tocsr(), np.arange(1.0, 8.0), np.full(7, 3.0), delta=1e-12)
    assert rep.iterations == 1
    with pytest.raises(so.OperatorError):
        so.pcg_solve(sp.diags([1.0, -1.0]).tocsr(), np.array([0.0, 1.0]), np.zeros(2))


def test_lhs_stratification():
    pts = np.array(so.lhs_sample(2, 4, [[0, 1], [0, 1]], seed=3))
    for d in range(2):
        assert sorted((pts[:, d] * 4).astype(int)) == [0, 1, 2, 3]
