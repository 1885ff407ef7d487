"""The reference-signature layer (paper_2311_13862_b200/compat.py) against the reference's
own outputs: its experiment driver (experiment.py:108-172, goldens recorded from the
unmodified run_experiment by make_golden.py --experiment) replayed call for call, and the
per-parameter solver / RB calls on the FV problems (golden_fd.npz)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import problems as op
from oracle import solvers as so

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build
    build.build(verbose=False)


def _rb():
    from paper_2311_13862_b200 import compat
    return compat


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def run_experiment_calls(rb, pid, levels, m0, n_train, n_test, dims, deltas, seed=0, l_max=60,
                         methods=("mgcg", "rbi-mgcg"), nu=1, smoother="auto"):
    """The call sequence of the reference's run_experiment (experiment.py:108-172) on the
    compat module: LHS sets from one SeedSequence, the LU-backed greedy, and per test
    parameter mg_context_for + rbi_pcg_solve for every (method, N, delta)."""
    spec = rb.get_problem(pid)
    prob = rb.ParametricProblem(spec, levels=levels, m0=m0)
    train_seed, test_seed = np.random.SeedSequence(seed).spawn(2)
    train = rb.lhs_sample(spec.p, n_train, spec.bounds, seed=train_seed)
    test = rb.lhs_sample(spec.p, n_test, spec.bounds, seed=test_seed)
    hf = rb.HighFidelitySolver(prob, method="lu")
    model = None
    if "rbi-mgcg" in methods:
        model = rb.l1roc_offline(train, max(dims), hf, prob.operator, prob.operator_rows,
                                 prob.rhs, seed=seed)
    systems = [(prob.operator(mu), prob.rhs(mu)) for mu in test]
    solves = []
    for method in methods:
        for N in ((0,) if method == "mgcg" else dims):
            for delta in deltas:
                mcfg = rb.MethodConfig(method, delta=delta, l_max=l_max, N=N, nu=nu,
                                       smoother=smoother, K_max=8)
                for mu, (A, f) in zip(test, systems):
                    ctx = rb.mg_context_for(prob, mu, nu=nu, smoother=smoother)
                    x, rep = rb.rbi_pcg_solve(A, f, mcfg, mg_ctx=ctx, l1roc_model=model,
                                              msrb_hier=None, mu=mu)
                    solves.append((f"{method}|{N}|{delta!r}", x, rep))
    return np.array(train), np.array(test), model, solves


@pytest.mark.parametrize("tag,pid,levels,m0,n_train,n_test,dims,deltas,methods", [
    ("ex1", "example-1", 3, 4, 16, 3, (4, 6), (1e-10, 1e-12), ("mgcg", "rbi-mgcg")),
    ("ex2", "example-2", 3, 4, 12, 3, (4,), (1e-10,), ("mgcg", "rbi-mgcg")),
])
def test_experiment_loop_matches_reference(tag, pid, levels, m0, n_train, n_test, dims, deltas,
                                           methods):
    g = np.load(GOLDEN / "golden_experiment.npz")
    k = f"exp_{tag}"
    rb = _rb()
    train, test, model, solves = run_experiment_calls(rb, pid, levels, m0, n_train, n_test,
                                                      dims, deltas, methods=methods)
    np.testing.assert_array_equal(train, g[f"{k}_train"])
    np.testing.assert_array_equal(test, g[f"{k}_test"])
    if model is not None:
        np.testing.assert_allclose(model.chosen_mus, g[f"{k}_chosen"], rtol=0, atol=0)
        np.testing.assert_allclose(model.indicator_history, g[f"{k}_hist"], rtol=1e-6)
    # solves were recorded in loop order: match them one to one
    keys = list(g[f"{k}_keys"])
    ref = [(keys[i], g[f"{k}_x{i}"], int(g[f"{k}_it{i}"])) for i in range(len(keys))]
    ref = [r for r in ref if r[0].split("|")[0] in methods]
    assert [s[0] for s in solves] == [r[0] for r in ref]
    for (key, x, rep), (_, xr, itr) in zip(solves, ref):
        assert abs(rep.iterations - itr) <= 1, (key, rep.iterations, itr)
        assert _rel(x, xr) <= 1e-8, (key, _rel(x, xr))
        assert rep.converged and rep.method == key.split("|")[0]
        assert rep.config["config_hash"]


def _fd(rb, blocks, n, m0=4):
    spec = rb.get_problem(f"thermal-block-{blocks[0]}x{blocks[1]}x{blocks[2]}")
    levels = int(np.log2(n // m0)) + 1
    return rb.ParametricProblem(spec, levels=levels, m0=m0)


def test_per_parameter_mgcg_matches_reference_golden(golden):
    """mgcg_solve(A, f, x0, ctx) per parameter, numpy in / out (multigrid.py:225-232)."""
    rb = _rb()
    prob = _fd(rb, (2, 2, 1), 32)
    key = "mgcg_tb221_n32"
    delta = float(golden[key + "_delta"])
    for m, xr, it in zip(golden[key + "_mus"], golden[key + "_x"], golden[key + "_iters"]):
        A, f = prob.operator(m), prob.rhs(m)
        ctx = rb.mg_context_for(prob, m)
        x, rep = rb.mgcg_solve(A, f, np.zeros_like(f), ctx, delta=delta, l_max=60, mu=m)
        assert abs(rep.iterations - int(it)) <= 1
        assert _rel(x, xr) <= 1e-8
        assert isinstance(x, np.ndarray) and x.shape == f.shape
        np.testing.assert_array_equal(rep.mu, m)


def test_l1roc_reference_signature_matches_golden(golden):
    """l1roc_offline(mus, N, hf, operator, operator_rows, rhs, seed) (rb.py:208-216),
    l1roc_online(model, A, b) and rbi_pcg_solve per parameter."""
    rb = _rb()
    prob = _fd(rb, (2, 2, 1), 16)
    train = golden["l1roc_tb221_n16_train"]
    hf = rb.HighFidelitySolver(prob, method="mgcg", delta=1e-14, l_max=200)
    model = rb.l1roc_offline(list(train), 6, hf, prob.operator, prob.operator_rows, prob.rhs,
                             seed=3)
    np.testing.assert_array_equal(model.collocation, golden["l1roc_tb221_n16_colloc"])
    np.testing.assert_array_equal(model.chosen_mus, golden["l1roc_tb221_n16_chosen_mus"])
    W = golden["l1roc_tb221_n16_W"]
    assert np.max(np.abs(model.basis - W)) <= 1e-8 * np.max(np.abs(W))
    sub = model.prefix(4)
    assert sub.dim == 4 and len(sub.collocation) == 7
    for m, mu in enumerate(golden["l1roc_tb221_n16_test"]):
        A, f = prob.operator(mu), prob.rhs(mu)
        u0, c = rb.l1roc_online(model, A, f)
        assert _rel(u0, golden["l1roc_tb221_n16_u0"][m]) <= 1e-9
        np.testing.assert_allclose(c, golden["l1roc_tb221_n16_c"][m], rtol=1e-7, atol=1e-12)
        cfg = rb.MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=model.dim)
        x, rep = rb.rbi_pcg_solve(A, f, cfg, mg_ctx=rb.mg_context_for(prob, mu),
                                  l1roc_model=model, mu=mu)
        assert abs(rep.iterations - int(golden["rbi_tb221_n16_iters"][m])) <= 1
        assert _rel(x, golden["rbi_tb221_n16_x"][m]) <= 1e-8
        assert rb.initial_residual(A, f, u0) < 1.0


def test_operator_object_matches_oracle():
    """A @ x, A.diagonal(), A[rows, :], operator_rows on every level vs the oracle's
    assembled operators (grid.py:246-264)."""
    rb = _rb()
    prob = _fd(rb, (2, 2, 2), 16)
    oprob = op.OracleProblem(op.thermal_block((2, 2, 2)), 16, 4)
    mu = op.sample_mus(op.thermal_block((2, 2, 2)), 1, seed=4)[0]
    rng = np.random.default_rng(0)
    for lvl in range(1, prob.levels):
        A, Ar = prob.operator(mu, level=lvl), oprob.operator(mu, level=lvl)
        x = rng.standard_normal(A.shape[0])
        assert _rel(A @ x, Ar @ x) <= 1e-13
        np.testing.assert_allclose(A.diagonal(), Ar.diagonal(), rtol=1e-13)
    A, Ar = prob.operator(mu), oprob.operator(mu)
    rows = [0, 17, 1000, A.shape[0] - 1]
    np.testing.assert_allclose(A[rows, :].toarray(), Ar[rows, :].toarray(), atol=1e-15)
    np.testing.assert_allclose(prob.operator_rows(mu, rows).toarray(),
                               oprob.operator_rows(mu, rows).toarray(), atol=1e-15)
    np.testing.assert_allclose(prob.rhs(mu), oprob.rhs(mu), rtol=1e-15)


def test_pcg_with_custom_preconditioner_and_cg_match_oracle():
    """pcg_solve with an arbitrary preconditioner callable and cg_solve follow the
    reference's loop (krylov.py:42-114): same iterations and histories as the oracle."""
    rb = _rb()
    prob = _fd(rb, (2, 1, 1), 16)
    oprob = op.OracleProblem(op.thermal_block((2, 1, 1)), 16, 4)
    mu = np.array([0.7, 3.0])
    A, Ar = prob.operator(mu), oprob.operator(mu)
    f = prob.rhs(mu)
    d = Ar.diagonal()
    jac = lambda r, k: r / d  # noqa: E731
    x, rep = rb.pcg_solve(A, f, np.zeros_like(f), precond=jac, delta=1e-8, l_max=400)
    xr, rr = so.pcg_solve(Ar, f, np.zeros_like(f), jac, delta=1e-8, l_max=400)
    assert rep.iterations == rr.iterations
    np.testing.assert_allclose(rep.history, rr.history, rtol=1e-9)
    assert _rel(x, xr) <= 1e-10
    x, rep = rb.cg_solve(A, f, np.zeros_like(f), delta=1e-6, l_max=500)
    xr, rr = so.pcg_solve(Ar, f, np.zeros_like(f), None, delta=1e-6, l_max=500)
    assert rep.method == "cg" and abs(rep.iterations - rr.iterations) <= 1
    # the native MG loop and the reference loop with the V-cycle callable agree
    ctx = rb.mg_context_for(prob, mu)
    x1, r1 = rb.mgcg_solve(A, f, np.zeros_like(f), ctx, delta=1e-10, l_max=60)
    x2, r2 = rb.pcg_solve(A, f, np.zeros_like(f), precond=lambda r, k: rb.mg_vcycle(r, ctx),
                          delta=1e-10, l_max=60, method="mgcg")
    assert r1.iterations == r2.iterations and _rel(x1, x2) <= 1e-12
    # residual_log: the preconditioned residuals of every iteration (warmstart.py:108-110)
    log = []
    cfg = rb.MethodConfig("mgcg", delta=1e-10, l_max=60)
    x3, r3 = rb.rbi_pcg_solve(A, f, cfg, mg_ctx=ctx, residual_log=log)
    assert len(log) == r3.iterations and r3.iterations == r1.iterations


def test_errors_follow_reference():
    rb = _rb()
    prob = _fd(rb, (2, 1, 1), 16)
    with pytest.raises(ValueError):
        prob.operator([100.0, 1.0])
    with pytest.raises(ValueError):
        rb.MethodConfig("nope")
    A, f = prob.operator([1.0, 1.0]), prob.rhs([1.0, 1.0])
    with pytest.raises(ValueError):
        rb.rbi_pcg_solve(A, f, rb.MethodConfig("rbi-mgcg", N=2), mg_ctx=None)
    with pytest.raises(ValueError):
        rb.pcg_solve(A, f, np.zeros_like(f), delta=0.0)
    with pytest.raises(ValueError):
        rb.HighFidelitySolver(prob, method="qr")


@pytest.mark.parametrize("tag", ["tb221", "ex1"])
def test_rbi_msrbcg_reference_signature_matches_golden(tag):
    """The reference's third method through its own call sequence (make_golden.py --msrb /
    --msrb-fem: msrb_train(train, N, K, hf, p.operator, p.rhs), then per test parameter
    rbi_pcg_solve(A, f, cfg, msrb_hier=hier, mu=mu)) on the compat module: the FV thermal block
    and the reference's own assembled problem example-1."""
    rb = _rb()
    if tag == "tb221":
        g, k = dict(np.load(GOLDEN / "golden_msrb.npz")), "msrb_tb221_n16"
        prob = _fd(rb, (2, 2, 1), 16)
    else:
        g, k = dict(np.load(GOLDEN / "golden_msrb_fem.npz")), "msrb_ex1_n16"
        prob = rb.ParametricProblem(rb.get_problem("example-1"), levels=3, m0=4)
    N, K = (int(v) for v in g[f"{k}_NK"])
    hf = rb.HighFidelitySolver(prob, method="lu")
    hier = rb.msrb_train(list(g[f"{k}_train"]), N, K, hf, prob.operator, prob.rhs)
    cfg = rb.MethodConfig("rbi-msrbcg", delta=1e-10, l_max=60, N=N, K_max=K)
    for m, mu in enumerate(g[f"{k}_test"]):
        A, f = prob.operator(mu), prob.rhs(mu)
        x, rep = rb.rbi_pcg_solve(A, f, cfg, msrb_hier=hier, mu=mu)
        assert abs(rep.iterations - int(g[f"{k}_iters"][m])) <= 1
        assert _rel(x, g[f"{k}_x"][m]) <= (1e-8 if tag == "ex1" else 1e-5)
        assert rep.config["preconditioner"] == "msrb"
        # (the thermal-block run stops at l_max in the reference as well: same count)
        assert rep.converged == (int(g[f"{k}_iters"][m]) < 60)
