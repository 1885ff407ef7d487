"""CUDA path (through the C ABI) vs the CPU oracle and the reference's golden vectors."""

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import problems as op
from oracle import solvers as so

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build
    build.build(verbose=False)


def _pkg():
    import paper_2311_13862_b200 as pkg
    return pkg


def _pair(blocks_or_smooth, n, m0):
    pkg = _pkg()
    if blocks_or_smooth == "smooth":
        ps, os_ = pkg.smooth_affine(6), op.smooth_affine(6)
    else:
        ps, os_ = pkg.thermal_block(blocks_or_smooth), op.thermal_block(blocks_or_smooth)
    levels = int(np.log2(n // m0)) + 1
    return pkg.ParametricProblem(ps, levels=levels, m0=m0), op.OracleProblem(os_, n, m0), os_


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ------------------------------------------------------------- operators

@pytest.mark.parametrize("case,n,m0", [((2, 2, 1), 16, 4), ((2, 2, 2), 16, 2), ("smooth", 16, 4),
                                        ((2, 1, 1), 32, 4)])
def test_apply_every_level(case, n, m0):
    pkg = _pkg()
    prob, oprob, ospec = _pair(case, n, m0)
    mus = op.sample_mus(ospec, 3, seed=11)
    ctx = pkg.mg_context_for(prob, mus)
    A = pkg.BatchOperator(ctx)
    rng = np.random.default_rng(0)
    for lvl in range(prob.levels):
        nl = prob.cells[lvl]
        xs = rng.standard_normal((3, (nl - 1) ** 3))
        y = A.apply(pkg.to_padded(xs, nl), level=lvl)
        got = pkg.from_padded(y, nl, 3)
        for m in range(3):
            ref = oprob.operator(mus[m], level=lvl) @ xs[m]
            assert _rel(got[m], ref) <= 1e-13, (lvl, m, _rel(got[m], ref))
        # ghosts stay zero
        blk = y[: 3 * nl ** 3].view(3, nl, nl, nl)
        assert float(blk[:, 0].abs().max()) == 0.0 and float(blk[:, :, 0].abs().max()) == 0.0


def test_transfers_match_prolongation():
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    prob, oprob, ospec = _pair((2, 2, 1), 16, 4)
    P = oprob.prolongations[-1]
    nf, nc = 16, 8
    rng = np.random.default_rng(1)
    rf = rng.standard_normal((2, (nf - 1) ** 3))
    ec = rng.standard_normal((2, (nc - 1) ** 3))
    bc = torch.zeros(pkg.padded_len(nc, 2), dtype=torch.float64, device="cuda")
    rft, ect = pkg.to_padded(rf, nf), pkg.to_padded(ec, nc)
    _native.call("rbws_restrict", nf, 2, rft.data_ptr(), bc.data_ptr(), 0)
    u = pkg.to_padded(rf, nf)
    _native.call("rbws_prolong_add", nf, 2, ect.data_ptr(), u.data_ptr(), 0)
    torch.cuda.synchronize()
    got_r, got_p = pkg.from_padded(bc, nc, 2), pkg.from_padded(u, nf, 2)
    for m in range(2):
        assert _rel(got_r[m], P.T @ rf[m]) <= 1e-14
        assert _rel(got_p[m], rf[m] + P @ ec[m]) <= 1e-14


def test_jacobi_sweep_matches_oracle():
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    prob, oprob, ospec = _pair((2, 2, 1), 16, 4)
    mus = op.sample_mus(ospec, 2, seed=5)
    ctx = pkg.mg_context_for(prob, mus)
    rng = np.random.default_rng(2)
    for lvl in (1, prob.levels - 1):
        nl = prob.cells[lvl]
        x = rng.standard_normal((2, (nl - 1) ** 3))
        b = rng.standard_normal((2, (nl - 1) ** 3))
        y = torch.zeros(pkg.padded_len(nl, 2), dtype=torch.float64, device="cuda")
        xt, bt = pkg.to_padded(x, nl), pkg.to_padded(b, nl)  # keep alive across the call
        _native.call("rbws_jacobi_sweep", ctx.handle, lvl, xt.data_ptr(), bt.data_ptr(),
                     y.data_ptr(), 0)
        got = pkg.from_padded(y, nl, 2)
        for m in range(2):
            A = oprob.operator(mus[m], level=lvl)
            ref = so.jacobi_sweep(A, A.diagonal(), x[m], b[m])
            assert _rel(got[m], ref) <= 1e-13


def test_vcycle_matches_reference_golden(golden):
    pkg = _pkg()
    prob, oprob, ospec = _pair((2, 2, 1), 16, 4)
    mu = golden["vcycle_tb221_n16_mu"]
    ctx = pkg.mg_context_for(prob, mu[None])
    out = pkg.mg_vcycle(pkg.to_padded(golden["vcycle_tb221_n16_in"], 16), ctx)
    got = pkg.from_padded(out, 16, 1)[0]
    assert _rel(got, golden["vcycle_tb221_n16_out"]) <= 1e-12


def test_vcycle_linearity_and_symmetry():
    pkg = _pkg()
    prob, oprob, ospec = _pair((2, 2, 2), 32, 4)
    mus = op.sample_mus(ospec, 2, seed=4)
    ctx = pkg.mg_context_for(prob, mus)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 31 ** 3))
    y = rng.standard_normal((2, 31 ** 3))
    Mx = pkg.from_padded(pkg.mg_vcycle(pkg.to_padded(x, 32), ctx), 32, 2)
    My = pkg.from_padded(pkg.mg_vcycle(pkg.to_padded(y, 32), ctx), 32, 2)
    Mx2 = pkg.from_padded(pkg.mg_vcycle(pkg.to_padded(-2.5 * x, 32), ctx), 32, 2)
    for m in range(2):
        assert _rel(Mx2[m], -2.5 * Mx[m]) <= 1e-12
        a, b = Mx[m] @ y[m], x[m] @ My[m]
        assert abs(a - b) <= 1e-10 * max(abs(a), abs(b))


# ------------------------------------------------------------- MGCG

@pytest.mark.parametrize("tag,case,n", [("tb211", (2, 1, 1), 16), ("tb221", (2, 2, 1), 32),
                                        ("tb222", (2, 2, 2), 16), ("smooth6", "smooth", 16)])
def test_mgcg_matches_reference_golden(golden, tag, case, n):
    """Solutions within 1e-8 rel. L2 and iteration counts within +-1 of the reference."""
    pkg = _pkg()
    prob, _, _ = _pair(case, n, 4)
    key = f"mgcg_{tag}_n{n}"
    mus = golden[key + "_mus"]
    delta = float(golden[key + "_delta"])
    ctx = pkg.mg_context_for(prob, mus)
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=delta, l_max=60)
    got = pkg.from_padded(x, n, len(mus))
    for m in range(len(mus)):
        assert abs(reps[m].iterations - int(golden[key + "_iters"][m])) <= 1
        assert _rel(got[m], golden[key + "_x"][m]) <= 1e-8
        assert reps[m].converged and reps[m].true_residual <= delta
        h_ref = golden[key + "_hist"][m]
        k = min(len(reps[m].history), 6)
        np.testing.assert_allclose(reps[m].history[:k], h_ref[:k], rtol=1e-7)


def test_mgcg_batch_matches_oracle_smooth32():
    pkg = _pkg()
    prob, oprob, ospec = _pair("smooth", 32, 4)
    mus = op.sample_mus(ospec, 3, seed=21)
    ctx = pkg.mg_context_for(prob, mus)
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-12, l_max=60)
    got = pkg.from_padded(x, 32, 3)
    for m in range(3):
        A, f = oprob.operator(mus[m]), oprob.rhs()
        xr, rr = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(oprob, mus[m]),
                               delta=1e-12, l_max=60)
        assert abs(reps[m].iterations - rr.iterations) <= 1
        assert _rel(got[m], xr) <= 1e-8


def test_mgcg_edge_cases():
    pkg = _pkg()
    prob, oprob, ospec = _pair((2, 1, 1), 16, 4)
    mus = op.sample_mus(ospec, 3, seed=2)
    ctx = pkg.mg_context_for(prob, mus)
    # l_max = 0: no iterations, history = [1]
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=0)
    assert all(r.iterations == 0 and r.history[0] == pytest.approx(1.0) for r in reps)
    # exact initial guess: zero iterations
    xs = np.stack([spla.spsolve(oprob.operator(m).tocsc(), oprob.rhs()) for m in mus])
    x, reps = pkg.mgcg_solve(None, prob.rhs(), pkg.to_padded(xs, 16), ctx, delta=1e-10)
    assert all(r.iterations == 0 for r in reps)
    # l_max caps iterations, not converged
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-30, l_max=3)
    assert all(r.iterations == 3 and not r.converged for r in reps)
    # zero rhs: absolute norms, stays at zero
    z = prob.zeros(1)
    x, reps = pkg.mgcg_solve(None, z, None, ctx, delta=1e-12)
    assert all(r.absolute_norms and r.iterations == 0 for r in reps)
    # outside bounds
    with pytest.raises(ValueError):
        pkg.mg_context_for(prob, np.array([[50.0, 1.0]]))


def test_mgcg_batch_of_one_and_context_reuse():
    pkg = _pkg()
    prob, oprob, ospec = _pair((2, 2, 1), 32, 4)
    mus = op.sample_mus(ospec, 4, seed=8)
    ctx = pkg.mg_context_for(prob, mus)
    xb, rb = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10)
    ctx = pkg.mg_context_for(prob, mus[2:3], ctx=ctx)
    x1, r1 = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10)
    assert r1[0].iterations == rb[2].iterations
    assert _rel(pkg.from_padded(x1, 32, 1)[0], pkg.from_padded(xb, 32, 4)[2]) <= 1e-12


# ------------------------------------------------------------- L1ROC

def _golden_model(golden, pkg, n=16):
    W = golden["l1roc_tb221_n16_W"]
    N = W.shape[1]
    basis = pkg.to_padded(W.T, n)
    return pkg.L1rocModel(n, basis, golden["l1roc_tb221_n16_T"], golden["l1roc_tb221_n16_colloc"],
                          golden["l1roc_tb221_n16_xs"], golden["l1roc_tb221_n16_xr"],
                          golden["l1roc_tb221_n16_chosen_mus"], golden["l1roc_tb221_n16_hist"])


def test_l1roc_online_matches_reference_golden(golden):
    pkg = _pkg()
    prob, _, _ = _pair((2, 2, 1), 16, 4)
    model = _golden_model(golden, pkg)
    test = golden["l1roc_tb221_n16_test"]
    ctx = pkg.mg_context_for(prob, test)
    u0, c = pkg.l1roc_online(model, pkg.BatchOperator(ctx), prob.rhs())
    got = pkg.from_padded(u0, 16, len(test))
    for m in range(len(test)):
        assert _rel(got[m], golden["l1roc_tb221_n16_u0"][m]) <= 1e-9
        np.testing.assert_allclose(c[m], golden["l1roc_tb221_n16_c"][m], rtol=1e-7, atol=1e-12)
    # RBI-MGCG refinement matches the reference's iteration counts and solutions
    cfg = pkg.MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=model.dim)
    x, reps = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), prob.rhs(), cfg, mg_ctx=ctx,
                                l1roc_model=model)
    got = pkg.from_padded(x, 16, len(test))
    for m in range(len(test)):
        assert abs(reps[m].iterations - int(golden["rbi_tb221_n16_iters"][m])) <= 1
        assert _rel(got[m], golden["rbi_tb221_n16_x"][m]) <= 1e-8


def test_l1roc_offline_matches_reference_golden(golden):
    pkg = _pkg()
    prob, _, _ = _pair((2, 2, 1), 16, 4)
    train = golden["l1roc_tb221_n16_train"]
    hf = pkg.HighFidelitySolver(prob, delta=1e-14, l_max=200)
    model = pkg.l1roc_offline(train, 6, hf, prob, seed=3)
    np.testing.assert_array_equal(model.collocation, golden["l1roc_tb221_n16_colloc"])
    np.testing.assert_array_equal(model.chosen_mus, golden["l1roc_tb221_n16_chosen_mus"])
    W = golden["l1roc_tb221_n16_W"]
    assert np.max(np.abs(model.basis_numpy() - W)) <= 1e-8 * np.max(np.abs(W))
    np.testing.assert_allclose(model.indicator_history, golden["l1roc_tb221_n16_hist"], rtol=1e-6)


def test_l1roc_saturation_matches_reference_golden(golden):
    pkg = _pkg()
    prob, _, _ = _pair((2, 1, 1), 16, 4)
    hf = pkg.HighFidelitySolver(prob, delta=1e-14, l_max=200)
    model = pkg.l1roc_offline(golden["l1roc_tb211_n16_train"], 8, hf, prob, seed=0)
    assert model.saturated
    np.testing.assert_array_equal(model.collocation, golden["l1roc_tb211_n16_colloc"])


def test_l1roc_rank_deficient_raises():
    pkg = _pkg()
    prob, _, ospec = _pair((2, 2, 1), 16, 4)
    n = 16
    # two identical basis columns -> rank deficient sampled matrix
    v = np.random.default_rng(0).standard_normal(15 ** 3)
    basis = pkg.to_padded(np.stack([v, v]), n)
    model = pkg.L1rocModel(n, basis, np.eye(2), np.array([0, 5, 9]), np.array([0, 5]),
                           np.array([9]), np.zeros((2, 4)), np.ones(2))
    ctx = pkg.mg_context_for(prob, op.sample_mus(ospec, 2, seed=1))
    with pytest.raises(pkg.DegenerateBasisError):
        pkg.l1roc_online(model, pkg.BatchOperator(ctx), prob.rhs())


def test_deim_known_answers():
    pkg = _pkg()
    n = 8
    v = np.zeros(7 ** 3)
    v[[0, 1, 2]] = [1.0, 3.0, 2.0]
    step = pkg.deim_extend(n, None, [], pkg.to_padded(v, n)[: pkg.padded_len(n, 1)])
    assert step.index == 1 and step.pivot == 3.0
    col = pkg.from_padded(step.column, n, 1)[0]
    np.testing.assert_allclose(col[:3], [1 / 3, 1.0, 2 / 3])
    step2 = pkg.deim_extend(n, None, [], pkg.to_padded(v, n)[: pkg.padded_len(n, 1)], exclude={1})
    assert step2.index == 2


# ------------------------------------------------------------- level kernels / full size

@pytest.mark.parametrize("case,n,m0", [((2, 2, 1), 16, 4), ((2, 2, 2), 32, 4), ("smooth", 16, 4)])
def test_level_kernels_every_mode(case, n, m0):
    """apply / residual / Jacobi / pre-smoothing residual on every smoothed level."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    prob, oprob, ospec = _pair(case, n, m0)
    mus = op.sample_mus(ospec, 5, seed=13)
    ctx = pkg.mg_context_for(prob, mus)
    rng = np.random.default_rng(7)
    for lvl in range(1, prob.levels):
        nl = prob.cells[lvl]
        x = rng.standard_normal((5, (nl - 1) ** 3))
        r = rng.standard_normal((5, (nl - 1) ** 3))
        xt, rt = pkg.to_padded(x, nl), pkg.to_padded(r, nl)
        for mode in range(4):
            ys = []
            for _ in range(2):
                y = torch.zeros_like(xt)
                _native.call("rbws_level_kernel", ctx.handle, lvl, mode, xt.data_ptr(),
                             rt.data_ptr(), y.data_ptr(), 0)
                ys.append(y)
            assert torch.equal(ys[0], ys[1]), "level kernel not deterministic"
            g = pkg.from_padded(ys[0], nl, 5)
            for m in range(5):
                A = oprob.operator(mus[m], level=lvl)
                d = A.diagonal()
                ref = [A @ x[m], r[m] - A @ x[m], so.jacobi_sweep(A, d, x[m], r[m]),
                       r[m] - A @ (0.7 * r[m] / d)][mode]
                assert _rel(g[m], ref) <= 1e-13, (lvl, mode, m)


def test_bench_config_properties_64():
    """configs[1]-shaped problem: every instance converges to tol; oracle agrees on a sample."""
    pkg = _pkg()
    prob, oprob, ospec = _pair((2, 2, 1), 64, 4)
    mus = op.sample_mus(ospec, 24, seed=2000)
    ctx = pkg.mg_context_for(prob, mus)
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    assert all(r.converged and r.true_residual <= 1e-10 for r in reps)
    got = pkg.from_padded(x, 64, len(mus))
    for m in (0, 11):
        A, f = oprob.operator(mus[m]), oprob.rhs()
        xr, rr = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(oprob, mus[m]),
                               delta=1e-10, l_max=60)
        assert abs(reps[m].iterations - rr.iterations) <= 1
        assert _rel(got[m], xr) <= 1e-8
    # the same batch solved twice is bitwise identical (deterministic reductions)
    x2, _ = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    assert torch.equal(x, x2)


def test_l1roc_online_matches_oracle_with_device_model():
    """GPU-trained model, GPU online stage vs the oracle's online stage on that model."""
    pkg = _pkg()
    prob, oprob, ospec = _pair((2, 2, 1), 32, 4)
    train = op.sample_mus(ospec, 64, seed=5)
    model = pkg.l1roc_offline(train, 8, pkg.HighFidelitySolver(prob), prob, seed=1)
    omodel = so.OracleL1rocModel(model.basis_numpy(), model.transform, model.collocation,
                                 model.solution_points, model.residual_points, model.chosen,
                                 model.indicator_history, model.saturated)
    test = op.sample_mus(ospec, 6, seed=6)
    ctx = pkg.mg_context_for(prob, test)
    u0, c = pkg.l1roc_online(model, pkg.BatchOperator(ctx), prob.rhs())
    got = pkg.from_padded(u0, 32, len(test))
    for m in range(len(test)):
        ur, cr, _ = so.l1roc_online(omodel, oprob.operator(test[m]), oprob.rhs())
        assert _rel(got[m], ur) <= 1e-9
        np.testing.assert_allclose(c[m], cr, rtol=1e-7, atol=1e-12)
    # prefix models (nested) agree with the oracle too
    sub = model.prefix(4)
    u4, _ = pkg.l1roc_online(sub, pkg.BatchOperator(ctx), prob.rhs())
    ur4, _, _ = so.l1roc_online(omodel.prefix(4), oprob.operator(test[0]), oprob.rhs())
    assert _rel(pkg.from_padded(u4, 32, len(test))[0], ur4) <= 1e-9


def test_mgcg_streaming_download_matches_device():
    """rbws_mgcg_solve_to_host: every instance's solution lands in pinned host memory
    (downloaded as soon as it stops iterating) and equals the device result."""
    pkg = _pkg()
    prob, _, ospec = _pair((2, 2, 1), 32, 4)
    mus = op.sample_mus(ospec, 9, seed=33)
    ctx = pkg.mg_context_for(prob, mus)
    n3 = 32 ** 3
    host = torch.full((9 * n3,), float("nan"), dtype=torch.float64).pin_memory()
    cs = torch.cuda.Stream()
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60,
                             out_host=host, copy_stream=cs)
    cs.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(host, x[:9 * n3].cpu())
    x2, reps2 = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    assert [r.iterations for r in reps] == [r.iterations for r in reps2]
    # l_max cap: nothing converges, everything is sent at the end
    host.fill_(float("nan"))
    x3, _ = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-30, l_max=2,
                           out_host=host, copy_stream=cs)
    cs.synchronize()
    assert torch.equal(host, x3[:9 * n3].cpu())


def test_host_pipeline_matches_device_solve():
    pkg = _pkg()
    prob, _, ospec = _pair((2, 2, 1), 32, 4)
    mus = op.sample_mus(ospec, 11, seed=34)
    ctx = pkg.mg_context_for(prob, mus)
    cfg = pkg.MethodConfig("mgcg", delta=1e-10, l_max=60)
    x, reps = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), prob.rhs(), cfg, mg_ctx=ctx)
    n3 = 32 ** 3
    host = torch.empty(11 * n3, dtype=torch.float64).pin_memory()
    pipe = pkg.HostPipeline(prob, cfg, sub_batch=4, tail=2)
    reps_p = pipe.solve(mus, host)
    torch.cuda.synchronize()
    assert [r.iterations for r in reps_p] == [r.iterations for r in reps]
    assert _rel(host.numpy(), x[:11 * n3].cpu().numpy()) <= 1e-13


def test_host_pipeline_back_to_back_async_calls():
    """sync=False calls overlap one call's downloads with the next call's solves; after
    waiting on the copy stream every output buffer holds its own call's solutions."""
    pkg = _pkg()
    prob, _, ospec = _pair((2, 2, 1), 32, 4)
    cfg = pkg.MethodConfig("mgcg", delta=1e-10, l_max=60)
    pipe = pkg.HostPipeline(prob, cfg, sizes=[5, 3])
    n3 = 32 ** 3
    outs, want = [], []
    for seed in (41, 42, 43):
        mus = op.sample_mus(ospec, 8, seed=seed)
        ctx = pkg.mg_context_for(prob, mus)
        x, _ = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), prob.rhs(), cfg, mg_ctx=ctx)
        want.append(x[:8 * n3].cpu().numpy())
        outs.append((mus, torch.empty(8 * n3, dtype=torch.float64).pin_memory()))
    for mus, buf in outs:
        pipe.solve(mus, buf, sync=False)
    pipe.copy_stream.synchronize()
    for (mus, buf), w in zip(outs, want):
        assert _rel(buf.numpy(), w) <= 1e-13


def test_configs2_shape_128_matches_oracle():
    """configs[2]-shaped problem (thermal 2x2x2, 128^3, tol 1e-12): batched and slab paths
    against the oracle on one parameter (north_star tolerance: 1e-8 rel. L2, +-1 iteration)."""
    pkg = _pkg()
    prob, oprob, ospec = _pair((2, 2, 2), 128, 4)
    mus = op.sample_mus(ospec, 3, seed=77)
    ctx = pkg.mg_context_for(prob, mus)
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-12, l_max=60)
    assert all(r.converged for r in reps)
    A, f = oprob.operator(mus[0]), oprob.rhs()
    xr, rr = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(oprob, mus[0]),
                           delta=1e-12, l_max=60)
    got = pkg.from_padded(x, 128, 3)[0]
    assert abs(reps[0].iterations - rr.iterations) <= 1
    assert _rel(got, xr) <= 1e-8
    xs, rs = pkg.slab_mgcg_solve(prob, mus[:1], nslabs=4, delta=1e-12)
    assert abs(rs.iterations - rr.iterations) <= 1
    assert _rel(pkg.from_padded(xs, 128, 1)[0], xr) <= 1e-8


def test_device_side_graph_loop_matches_host_loop():
    """PCG iterations as a conditional CUDA graph (device-side WHILE) give bitwise the
    host-driven loop's solutions, iteration counts and histories."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    prob, _, ospec = _pair((2, 2, 1), 32, 4)
    mus = op.sample_mus(ospec, 6, seed=51)
    ctx = pkg.mg_context_for(prob, mus)
    out = {}
    for g in (0, 1, 1):   # the second graph run reuses the cached executable
        _native.call("rbws_batch_set_graph", ctx.handle, g)
        x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-11, l_max=60)
        out.setdefault(g, []).append((x.clone(), [r.history for r in reps]))
    x0, h0 = out[0][0]
    for x1, h1 in out[1]:
        assert torch.equal(x0, x1) and h0 == h1
    # l_max cap inside the graph
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-30, l_max=5)
    assert all(r.iterations == 5 and not r.converged for r in reps)


def test_stored_weight_kernels_match_register_kernels(monkeypatch):
    """Coefficients whose z factors change on every plane use stored face weights (SCW);
    they reproduce the register-refresh kernels (smooth affine coefficient)."""
    pkg = _pkg()
    prob, oprob, ospec = _pair("smooth", 32, 4)
    mus = op.sample_mus(ospec, 3, seed=61)
    out = []
    for scw in ("1", "0"):
        monkeypatch.setenv("RBWS_SCW", scw)
        ctx = pkg.MgContext(prob, 3).setup(mus)
        x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-12, l_max=60)
        out.append((x.clone(), [r.history for r in reps]))
        del ctx
    # the post-smoothing takes w/diag from the 1/diag vector (one rounding apart)
    assert _rel(out[0][0].cpu().numpy(), out[1][0].cpu().numpy()) <= 1e-12
    for h0, h1 in zip(out[0][1], out[1][1]):
        assert len(h0) == len(h1)
        np.testing.assert_allclose(h0, h1, rtol=1e-9)


def test_l1roc_rank_test_follows_numpy_lstsq():
    """The online least squares declares rank deficiency exactly when numpy's lstsq
    (SVD, rcond = eps max(M, N); reference rb.py:174-179) reports rank < N: sampled
    matrices with a smallest singular value just above / below the threshold, and a
    well-conditioned one (the unpivoted-QR diagonal test disagreed)."""
    from paper_2311_13862_b200 import _native
    M, N = 7, 4
    rng = np.random.default_rng(11)
    U, _ = np.linalg.qr(rng.standard_normal((M, M)))
    V, _ = np.linalg.qr(rng.standard_normal((N, N)))
    rc = np.finfo(float).eps * max(M, N)
    svals = [[1.0, 0.5, 0.2, 0.1], [1.0, 1e-3, 1e-9, 0.3 * rc], [1.0, 1e-3, 1e-9, 3.0 * rc],
             [1.0, 1e-3, 1e-9, 1e-12], [1.0, 0.0, 0.5, 0.2]]
    Bs = [U[:, :N] @ np.diag(s) @ V.T for s in svals]
    Q = count = len(Bs)
    theta = torch.eye(count, dtype=torch.float64, device="cuda").contiguous()
    Bq = torch.as_tensor(np.stack(Bs), device="cuda").contiguous()
    bs = torch.as_tensor(rng.standard_normal((count, M)), device="cuda").contiguous()
    T = torch.eye(N, dtype=torch.float64, device="cuda")
    a = torch.zeros(count * N, dtype=torch.float64, device="cuda")
    c = torch.zeros_like(a)
    ind = torch.zeros(count, dtype=torch.float64, device="cuda")
    st = torch.zeros(count, dtype=torch.int32, device="cuda")
    _native.call("rbws_l1roc_online", count, Q, M, N, theta.data_ptr(), Bq.data_ptr(),
                 bs.data_ptr(), M, T.data_ptr(), a.data_ptr(), c.data_ptr(), ind.data_ptr(),
                 st.data_ptr(), 0)
    got = st.cpu().numpy()
    for m, B in enumerate(Bs):
        sol, _, rank, _ = np.linalg.lstsq(B, bs[m].cpu().numpy(), rcond=None)
        assert bool(got[m]) == (rank < N), (m, got[m], rank)
        if rank == N and np.linalg.cond(B) < 1e6:
            np.testing.assert_allclose(a.view(count, N)[m].cpu().numpy(), sol, rtol=1e-10)
