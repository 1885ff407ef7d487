"""example-2 on the B200 full-node path (csrc/planes.cu through the C ABI): operator
apply, transfers, plane-Jacobi / point-Jacobi V-cycles and batched MGCG against the
unmodified reference's goldens (tests/golden/golden_fem2.npz) and the oracle."""

from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

G = np.load(Path(__file__).parent / "golden" / "golden_fem2.npz")
CASES = (("n8m2", 3, 2), ("n16m4", 3, 4))
SMOOTHERS = (("planejacobi", "auto"), ("planez", "plane-z"), ("jacobi", "jacobi"))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build
    build.build(verbose=False)


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def case(request):
    from paper_2311_13862_b200 import fem
    from paper_2311_13862_b200.fem_fn import FnFemProblem
    tag, levels, m0 = request.param
    return f"fem2_{tag}", FnFemProblem(fem.example2(), levels=levels, m0=m0)


def _golden_op(k, lvl):
    ip = G[f"{k}_op{lvl}_indptr"]
    return sp.csr_matrix((G[f"{k}_op{lvl}_data"], G[f"{k}_op{lvl}_indices"], ip),
                         shape=(len(ip) - 1,) * 2)


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_apply_every_level(case):
    from paper_2311_13862_b200.fem_fn import mg_context_for
    k, p = case
    mus = G[f"{k}_mus"]
    ctx = mg_context_for(p, mus[:1], smoother="jacobi")
    rng = np.random.default_rng(1)
    for lvl in range(p.levels):
        A = _golden_op(k, lvl)
        v = rng.standard_normal((1, A.shape[0]))
        y = p.from_full(ctx.apply(p.to_full(v, lvl), lvl), lvl)
        assert _rel(y[0], A @ v[0]) <= 1e-14
        b = rng.standard_normal((1, A.shape[0]))
        r = p.from_full(ctx.apply(p.to_full(v, lvl), lvl, b=p.to_full(b, lvl)), lvl)
        assert _rel(r[0], b[0] - A @ v[0]) <= 1e-14


def test_transfers(case):
    """Restriction P^T r and prolongation u + P e against the host free-DoF P."""
    from paper_2311_13862_b200 import _native
    from paper_2311_13862_b200.fem_fn import _ptr
    k, p = case
    rng = np.random.default_rng(2)
    st = _native.stream_ptr()
    for lvl in range(1, p.levels):
        P = p.prolongations[lvl - 1]
        cc = p.cells[lvl - 1]
        r = rng.standard_normal((2, P.shape[0]))
        rt = p.to_full(r, lvl)
        bc = torch.empty(2, p.nodes(lvl - 1), dtype=torch.float64, device="cuda")
        _native.call("rbws_fn_restrict", 2, cc, _ptr(rt), _ptr(bc), _ptr(p._mask_dev[lvl - 1]), st)
        got = p.from_full(bc, lvl - 1)
        for i in range(2):
            assert _rel(got[i], P.T @ r[i]) <= 1e-15
        e = rng.standard_normal((2, P.shape[1]))
        u = rng.standard_normal((2, P.shape[0]))
        ut = p.to_full(u, lvl)
        _native.call("rbws_fn_prolong_add", 2, cc, _ptr(p.to_full(e, lvl - 1)), _ptr(ut),
                     _ptr(p._mask_dev[lvl]), st)
        full = ut.cpu().numpy()
        assert np.all(full[:, ~p.masks[lvl]] == 0.0)
        got = full[:, p.free_by_level[lvl]]
        for i in range(2):
            assert _rel(got[i], u[i] + P @ e[i]) <= 1e-15


@pytest.mark.parametrize("key,kind", SMOOTHERS, ids=[s[0] for s in SMOOTHERS])
def test_vcycle_matches_reference(case, key, kind):
    from paper_2311_13862_b200.fem_fn import mg_context_for
    k, p = case
    mus = G[f"{k}_mus"]
    ctx = mg_context_for(p, np.repeat(mus[:1], 3, axis=0), smoother=kind)
    b = np.repeat(G[f"{k}_vcyc_b"][None], 3, axis=0)
    v = p.from_full(ctx.vcycle(p.to_full(b)))
    ref = G[f"{k}_vcyc_{key}"]
    for i in range(3):
        assert _rel(v[i], ref) <= 1e-12
    # the same instance solved three times in one batch is bitwise repeatable
    assert np.array_equal(v[0], v[1]) and np.array_equal(v[0], v[2])


@pytest.mark.parametrize("key,kind", SMOOTHERS, ids=[s[0] for s in SMOOTHERS])
def test_batched_mgcg_matches_reference(case, key, kind):
    """Zero-init MGCG to 1e-10 for the golden parameters in ONE batch: the reference's
    iteration counts, histories and solutions per instance."""
    from paper_2311_13862_b200.fem_fn import mg_context_for, mgcg_solve
    k, p = case
    mus = G[f"{k}_mus"]
    ctx = mg_context_for(p, mus, smoother=kind)
    x, reps = mgcg_solve(ctx, p.rhs(mus), delta=1e-10, l_max=80)
    xs = p.from_full(x)
    np.testing.assert_array_equal(reps.iterations, G[f"{k}_{key}_iters"])
    for i in range(len(mus)):
        h = G[f"{k}_{key}_hist"][i]
        np.testing.assert_allclose(reps[i].history, h[~np.isnan(h)], rtol=1e-6)
        assert reps[i].converged
        assert _rel(xs[i], G[f"{k}_{key}_x"][i]) <= 1e-9
    # Dirichlet nodes stay exactly zero
    assert torch.all(x.reshape(len(mus), -1)[:, torch.as_tensor(~p.masks[-1])] == 0.0)


def test_plane_blocks_solved_exactly(case):
    """A plane-Jacobi sweep with omega = 1 from x = 0 solves every z-plane block exactly:
    the result equals the host's dense block solves of b."""
    from paper_2311_13862_b200 import _native
    from paper_2311_13862_b200.fem_fn import _ptr, mg_context_for
    k, p = case
    mu = G[f"{k}_mus"][1]
    import os
    os.environ["RBWS_BAND_SOLVE_T"] = "1"  # also build the transposed factors (opt-in path)
    try:
        ctx = mg_context_for(p, mu[None], smoother="plane-jacobi")
    finally:
        os.environ.pop("RBWS_BAND_SOLVE_T", None)
    A = p.operator_host(mu).toarray()
    rng = np.random.default_rng(3)
    b = rng.standard_normal((1, p.n_free))
    r = p.to_full(b)
    layers = p.free_by_level[-1] // (p.n + 1) ** 2
    ref = np.zeros(p.n_free)
    for z in np.unique(layers):
        idx = np.flatnonzero(layers == z)
        ref[idx] = np.linalg.solve(A[np.ix_(idx, idx)], b[0, idx])
    # gather-form kernel and the scatter-form kernel on the transposed factor
    for kind in ("gather", "scatter"):
        r = p.to_full(b)
        x = torch.zeros_like(r)
        if kind == "gather":
            _native.call("rbws_fn_band_solve", 1, p.n, 1, _ptr(ctx.bands[-1]), _ptr(r), _ptr(x),
                         1.0, 1, _native.stream_ptr())
        else:
            assert ctx.bandsT[-1] is not None
            _native.call("rbws_fn_band_solve_t", 1, p.n, 1, _ptr(ctx.bands[-1]),
                         _ptr(ctx.bandsT[-1]), _ptr(r), _ptr(x), 1.0, 1, _native.stream_ptr())
        got = p.from_full(x)[0]
        assert _rel(got, ref) <= 1e-12, kind


def test_larger_grid_against_oracle():
    """32^3 (4 levels, m0 = 4): batched plane-Jacobi MGCG against the oracle restatement
    (iteration counts, solutions)."""
    from oracle import fem as of
    from oracle import solvers as so
    from paper_2311_13862_b200 import fem
    from paper_2311_13862_b200.fem_fn import FnFemProblem, mg_context_for, mgcg_solve
    p = FnFemProblem(fem.example2(), levels=4, m0=4)
    op = of.OracleFemProblem(of.Example2(), levels=4, m0=4)
    rng = np.random.default_rng(11)
    b = fem.example2().bounds
    mus = b[:, 0] + rng.random((4, 7)) * (b[:, 1] - b[:, 0])
    x, reps = mgcg_solve(mg_context_for(p, mus), p.rhs(mus), delta=1e-10, l_max=80)
    xs = p.from_full(x)
    for i, mu in enumerate(mus):
        A, f = op.operator(mu), op.rhs(mu)
        xo, rep = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(op, mu, smoother="auto"),
                                delta=1e-10, l_max=80)
        assert reps.iterations[i] == rep.iterations
        assert _rel(xs[i], xo) <= 1e-9


def test_reference_api_dispatch():
    """A reference user's calls (ParametricProblem / mg_context_for / mgcg_solve) reach the
    full-node path for example-2 and give the reference's iteration counts."""
    import paper_2311_13862_b200 as rb
    from paper_2311_13862_b200.fem_fn import FnFemProblem
    k = "fem2_n16m4"
    prob = rb.ParametricProblem(rb.get_problem("example-2"), levels=3, m0=4)
    assert isinstance(prob, FnFemProblem)
    mus = G[f"{k}_mus"]
    ctx = rb.mg_context_for(prob, mus)
    assert ctx.smoother == "plane-jacobi"
    x, reps = rb.mgcg_solve(None, prob.rhs(mus), None, ctx, delta=1e-10, l_max=80)
    np.testing.assert_array_equal([r.iterations for r in reps], G[f"{k}_planejacobi_iters"])
    v = prob.from_full(rb.mg_vcycle(prob.to_full(G[f"{k}_vcyc_b"][None].repeat(3, 0)), ctx))
    assert _rel(v[0], G[f"{k}_vcyc_planejacobi"]) <= 1e-12


def test_shared_apply_is_bitwise_the_per_instance_apply(case):
    """rbws_fn_apply_shared (batch-shared term coefficients combined on the fly, the finest
    level's apply) equals rbws_fn_apply over the combined per-instance coefficients bit for
    bit, for a batch size that is not a multiple of the 4 instances per thread."""
    from paper_2311_13862_b200 import _native
    from paper_2311_13862_b200.fem_fn import _ptr, mg_context_for
    k, p = case
    b = p.spec.bounds
    rng = np.random.default_rng(4)
    mus = b[:, 0] + rng.random((7, 7)) * (b[:, 1] - b[:, 0])
    ctx = mg_context_for(p, mus, smoother="jacobi")
    lvl = p.levels - 1
    x = p.to_full(rng.standard_normal((7, p.n_free)))
    f = p.to_full(rng.standard_normal((7, p.n_free)))
    st = _native.stream_ptr()
    for mode, bb in ((0, None), (1, f)):
        y1, y2 = torch.empty_like(x), torch.empty_like(x)
        _native.call("rbws_fn_apply", 7, p.n, _ptr(ctx.coefA[lvl]), _ptr(x),
                     _ptr(bb) if bb is not None else None, _ptr(y1), mode, st)
        _native.call("rbws_fn_apply_shared", 7, ctx.theta.shape[1], p.n, _ptr(ctx.theta),
                     _ptr(p._coef[lvl]), _ptr(x), _ptr(bb) if bb is not None else None, _ptr(y2),
                     mode, st)
        assert torch.equal(y1, y2)


def test_mgcg_edge_cases(case):
    """krylov.py:49-67 semantics on the full-node path: l_max = 0 returns x0 with the true
    residual, a zero right-hand side switches to absolute norms and needs no iteration, an
    exact initial guess stops at k = 0, and non-positive tolerances / negative l_max raise."""
    from paper_2311_13862_b200.fem_fn import mg_context_for, mgcg_solve
    k, p = case
    mus = G[f"{k}_mus"]
    ctx = mg_context_for(p, mus)
    f = p.rhs(mus)
    x, reps = mgcg_solve(ctx, f, delta=1e-10, l_max=0)
    assert all(r.iterations == 0 for r in reps) and torch.all(x == 0)
    assert all(abs(r.true_residual - 1.0) < 1e-12 for r in reps)
    z = torch.zeros_like(f)
    x, reps = mgcg_solve(ctx, z, delta=1e-10, l_max=10)
    assert all(r.iterations == 0 and r.absolute_norms and r.converged for r in reps)
    xs, _ = mgcg_solve(ctx, f, delta=1e-12, l_max=80)
    x, reps = mgcg_solve(ctx, f, x0=xs, delta=1e-6, l_max=80)
    assert all(r.iterations == 0 for r in reps)
    assert torch.equal(x, xs)
    with pytest.raises(ValueError):
        mgcg_solve(ctx, f, delta=0.0)
    with pytest.raises(ValueError):
        mgcg_solve(ctx, f, l_max=-1)
