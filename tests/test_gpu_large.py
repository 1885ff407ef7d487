"""Parity at the BASELINE's large grids and for every finest-level kernel variant.

configs[3] (smooth affine, 256^3: stored face weights "SCW", 3-slot rings) and
configs[4] (thermal 2x2x2, 512^3: "DC" kernels with w/diag cached in shared memory,
512-thread CTAs, 2-slot post-smoothing ring) run kernel instantiations that the small
golden cases never reach.  The checker here is the matrix-free Kronecker oracle
(oracle/kron.py, pinned to the 3D-assembled oracle and the reference goldens by
tests/test_oracle_kron.py), which fits these sizes; the reference runs the same
mg_vcycle / mgcg_solve at any size (multigrid.py:205-232).

* level kernels (apply / residual / Jacobi / pre-smoothing residual, rbws_level_kernel)
  on the finest and the next level, compared plane window by plane window;
* one V-cycle at 256^3 against the oracle's V-cycle (fused pre-smoothing + restriction,
  prolongation fused into the post-smoothing, coarse Kronecker kernels, coarsest Cholesky);
* one zero-init MGCG at 256^3 against the oracle's (north_star: 1e-8 rel. L2, +-1 iteration);
* the DC kernels forced on at 64^3 and off at 256^3 against the default choice;
* fused vs separate pre-smoothing + restriction at 256^3 and 512^3;
* a 4-slab 512^3 solve against the batched (one-instance) 512^3 solve;
* RBI-MGCG at the bench configuration (configs[1]: 64^3, r = 20 from 1024 training
  parameters) against the oracle's online stage + MGCG on the same model.
"""

import numpy as np
import pytest

from oracle import kron
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
    yield
    from paper_2311_13862_b200 import _native
    _native.call("rbws_set_kernel_variant", 0, -1)
    torch.cuda.empty_cache()


def _pkg():
    import paper_2311_13862_b200 as pkg
    return pkg


def _specs(case):
    pkg = _pkg()
    if case == "smooth":
        return pkg.smooth_affine(6), op.smooth_affine(6)
    return pkg.thermal_block(case), op.thermal_block(case)


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _planes(t, n, inst, k0, k1):
    """Interior planes [k0-1, k1] of instance `inst` of a padded device vector as a
    zero-framed (k1-k0+2, n+1, n+1) host array (the oracle's apply_planes input)."""
    m = n - 1
    out = np.zeros((k1 - k0 + 2, m + 2, m + 2))
    lo, hi = max(k0 - 1, 0), min(k1, m - 1)          # interior planes present
    base = inst * n ** 3
    blk = t[base + (lo + 1) * n * n: base + (hi + 2) * n * n].view(hi - lo + 1, n, n)
    out[lo - (k0 - 1): hi - (k0 - 1) + 1, 1:m + 1, 1:m + 1] = blk[:, 1:, 1:].cpu().numpy()
    return out


def _windows(m):
    mid = m // 2
    return [(0, 3), (mid - 2, mid + 2), (m - 3, m)]


def _check_level_kernels(case, n, count, level_from_top=0, windows=None):
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    spec, ospec = _specs(case)
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    kp = kron.KronProblem(ospec, n, 4)
    mus = op.sample_mus(ospec, count, seed=101)
    ctx = pkg.mg_context_for(prob, mus)
    lvl = prob.levels - 1 - level_from_top
    nl = prob.cells[lvl]
    m = nl - 1
    g = torch.Generator(device="cuda").manual_seed(5)
    L = pkg.padded_len(nl, count)
    mask = torch.zeros(count, nl, nl, nl, dtype=torch.float64, device="cuda")
    mask[:, 1:, 1:, 1:] = 1.0
    x = torch.zeros(L, dtype=torch.float64, device="cuda")
    r = torch.zeros_like(x)
    x[: count * nl ** 3] = (torch.randn(count * nl ** 3, generator=g, device="cuda",
                                        dtype=torch.float64) * mask.view(-1))
    r[: count * nl ** 3] = (torch.randn(count * nl ** 3, generator=g, device="cuda",
                                        dtype=torch.float64) * mask.view(-1))
    del mask
    omega = 0.7
    ys = []
    for mode in range(4):
        y = torch.zeros_like(x)
        _native.call("rbws_level_kernel", ctx.handle, lvl, mode, x.data_ptr(), r.data_ptr(),
                     y.data_ptr(), 0)
        ys.append(y)
    torch.cuda.synchronize()
    for inst in range(count):
        for k0, k1 in (windows or _windows(m)):
            st = kp.stencil(mus[inst], lvl, k0, k1)
            xp = _planes(x, nl, inst, k0, k1)
            rp = _planes(r, nl, inst, k0, k1)[1:-1, 1:-1, 1:-1]
            d = st.coef[(0, 0, 0)]
            ax = st.apply_planes(xp)
            # pre-smoothing residual input w D^-1 r needs the diagonal one plane beyond the
            # window: take it from a one-plane-wider stencil
            wk0, wk1 = max(k0 - 1, 0), min(k1 + 1, m)
            dw = kp.stencil(mus[inst], lvl, wk0, wk1).coef[(0, 0, 0)]
            rw = _planes(r, nl, inst, wk0, wk1)[1:-1, 1:-1, 1:-1]
            uw = np.zeros((k1 - k0 + 2, m + 2, m + 2))
            uw[wk0 - (k0 - 1): wk1 - (k0 - 1), 1:m + 1, 1:m + 1] = omega * rw / dw
            refs = [ax, rp - ax, xp[1:-1, 1:-1, 1:-1] + omega * (rp - ax) / d,
                    rp - st.apply_planes(uw)]
            for mode in range(4):
                got = _planes(ys[mode], nl, inst, k0, k1)[1:-1, 1:-1, 1:-1]
                ref = refs[mode]
                err = np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)
                assert err <= 1e-13, (case, n, lvl, mode, inst, (k0, k1), err)
    return ctx


@pytest.mark.parametrize("case,n,count,top", [
    ("smooth", 256, 2, 0),          # configs[3]: SCW kernels, 3-slot rings
    ("smooth", 256, 2, 1),          # its 128^3 coarse level (stored 27-point coefficients)
    ((2, 2, 2), 256, 2, 0),         # DC pre-smoothing at N = 256
    ((2, 2, 2), 512, 1, 0),         # configs[4]: 512-thread CTAs, DC
    ((2, 2, 2), 512, 1, 1),         # its 256^3 coarse level (Kronecker kernel)
])
def test_level_kernels_large(case, n, count, top):
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    ctx = _check_level_kernels(case, n, count, top)
    if case == "smooth" and top == 0:
        assert _native.load().rbws_batch_stored_weights(ctx.handle) == 1
    del ctx
    torch.cuda.empty_cache()


def test_vcycle_256_matches_kron_oracle():
    """One V-cycle (configs[3] shape) for two instances vs the oracle's mg_vcycle."""
    pkg = _pkg()
    spec, ospec = _specs("smooth")
    n = 256
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    kp = kron.KronProblem(ospec, n, 4)
    mus = op.sample_mus(ospec, 2, seed=33)
    ctx = pkg.mg_context_for(prob, mus)
    rng = np.random.default_rng(3)
    b = rng.standard_normal((2, (n - 1) ** 3))
    out = pkg.mg_vcycle(pkg.to_padded(b, n), ctx)
    got = pkg.from_padded(out, n, 2)
    from paper_2311_13862_b200 import _native
    assert _native.load().rbws_batch_stored_weights(ctx.handle) == 1
    for m in range(2):
        ref = so.mg_vcycle(b[m], kron.mg_context_for(kp, mus[m]))
        assert _rel(got[m], ref) <= 1e-12, m
    del ctx, out
    torch.cuda.empty_cache()


def test_mgcg_256_matches_kron_oracle():
    """configs[3]: zero-init MGCG to 1e-12 on one 256^3 instance vs the oracle."""
    pkg = _pkg()
    spec, ospec = _specs("smooth")
    n = 256
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    kp = kron.KronProblem(ospec, n, 4)
    mu = op.sample_mus(ospec, 1, seed=44)
    ctx = pkg.mg_context_for(prob, mu)
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-12, l_max=60)
    got = pkg.from_padded(x, n, 1)[0]
    xr, rr = kron.mgcg_solve(kp, mu[0], delta=1e-12, l_max=60)
    assert abs(reps[0].iterations - rr.iterations) <= 1
    assert _rel(got, xr) <= 1e-8
    np.testing.assert_allclose(reps[0].history[:5], rr.history[:5], rtol=1e-8)
    del ctx, x
    torch.cuda.empty_cache()


def _vcycle_and_solve(prob, mus, delta, n):
    pkg = _pkg()
    ctx = pkg.MgContext(prob, len(mus)).setup(mus)
    rng = np.random.default_rng(9)
    b = pkg.to_padded(rng.standard_normal((len(mus), (n - 1) ** 3)), n)
    v = pkg.mg_vcycle(b, ctx)
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=delta, l_max=60)
    out = (v.clone(), x.clone(), [r.iterations for r in reps], [r.history for r in reps])
    del ctx, v, x, b
    torch.cuda.empty_cache()
    return out


def _compare_runs(a, b, tol):
    assert (torch.linalg.norm(a[0] - b[0]) / torch.linalg.norm(b[0])).item() <= tol
    assert (torch.linalg.norm(a[1] - b[1]) / torch.linalg.norm(b[1])).item() <= tol
    assert a[2] == b[2]
    for h0, h1 in zip(a[3], b[3]):
        np.testing.assert_allclose(h0, h1, rtol=1e-8)


@pytest.mark.parametrize("n,case,force", [(64, (2, 2, 1), 1), (32, (2, 2, 2), 1),
                                          (256, (2, 2, 2), 0)])
def test_dc_variant_matches_default(n, case, force):
    """The DC pre/post-smoothing kernels (auto only at N >= 256) forced on at small N and
    off at N = 256 give the default kernels' V-cycle, solutions and iteration counts."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    spec, ospec = _specs(case)
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    mus = op.sample_mus(ospec, 3 if n < 256 else 1, seed=55)
    delta = 1e-10
    try:
        _native.call("rbws_set_kernel_variant", 0, -1)
        base = _vcycle_and_solve(prob, mus, delta, n)
        _native.call("rbws_set_kernel_variant", 0, force)
        var = _vcycle_and_solve(prob, mus, delta, n)
    finally:
        _native.call("rbws_set_kernel_variant", 0, -1)
    _compare_runs(var, base, 1e-13)


@pytest.mark.parametrize("n,case", [(16, (2, 1, 1)), (64, (2, 2, 1)), (64, (2, 2, 2)),
                                    (128, (2, 2, 2)), (256, (2, 2, 2))])
def test_sw_variant_matches_transformed(n, case):
    """The scaled-weights pre-smoothing kernels (face weights x the neighbours' w/diag on the
    raw b, default for piecewise-constant coefficients) against the transformed-ring kernels
    (u = w D^-1 b staged, rbws_set_kernel_variant(1, 0)): V-cycle, solutions, iterations."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    spec, ospec = _specs(case)
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    mus = op.sample_mus(ospec, 3 if n < 256 else 1, seed=57)
    delta = 1e-10
    try:
        _native.call("rbws_set_kernel_variant", 1, 0)
        base = _vcycle_and_solve(prob, mus, delta, n)
        _native.call("rbws_set_kernel_variant", 1, -1)
        var = _vcycle_and_solve(prob, mus, delta, n)
    finally:
        _native.call("rbws_set_kernel_variant", 1, -1)
    _compare_runs(var, base, 1e-13)


@pytest.mark.parametrize("n,case,count", [(64, (2, 2, 1), 40), (64, (2, 2, 2), 37),
                                          (128, (2, 2, 2), 10)])
def test_fused_cg_update_pre_smoothing_matches_separate(n, case, count):
    """The CG update that also computes the next V-cycle's pre-smoothing residual and the x/z
    passes of its restriction (cgp.cu, the default at 64^3 with whole instances per CTA) against
    the separate kernels (rbws_set_kernel_variant(4, 0)): solutions, iteration counts,
    histories."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    spec, ospec = _specs(case)
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    mus = op.sample_mus(ospec, count, seed=60)
    delta = 1e-10
    try:
        _native.call("rbws_set_kernel_variant", 4, 0)
        base = _vcycle_and_solve(prob, mus, delta, n)
        _native.call("rbws_set_kernel_variant", 4, -1)
        var = _vcycle_and_solve(prob, mus, delta, n)
    finally:
        _native.call("rbws_set_kernel_variant", 4, -1)
    # (rounding-level differences: an instance whose residual sits at the tolerance may take
    # one more / fewer iteration)
    assert (torch.linalg.norm(var[0] - base[0]) / torch.linalg.norm(base[0])).item() <= 1e-12
    assert (torch.linalg.norm(var[1] - base[1]) / torch.linalg.norm(base[1])).item() <= 1e-9
    assert max(abs(a - b) for a, b in zip(var[2], base[2])) <= 1
    for h0, h1 in zip(var[3], base[3]):
        np.testing.assert_allclose(h0[:8], h1[:8], rtol=1e-8)
    print("fused CG update: max |dx| =", float((var[1] - base[1]).abs().max()))


@pytest.mark.parametrize("count", [37, 150])
def test_fused_cg_update_is_repeatable(count):
    """The fused CG update reads its neighbours' halo rows of r while they update theirs (out of
    place) and hands planes between warps through shared memory: repeated solves of the same
    batch must agree bitwise (a race would show up as run-to-run differences)."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    n = 64
    spec, ospec = _specs((2, 2, 1))
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    mus = op.sample_mus(ospec, count, seed=61)
    ctx = pkg.mg_context_for(prob, mus)
    runs = []
    for _ in range(3):
        x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
        assert _native.load().rbws_batch_cg_fused(ctx.handle) == 1
        runs.append((x.clone(), [r.iterations for r in reps], np.array([r.history for r in reps], dtype=object)))
    for x, it, _ in runs[1:]:
        assert torch.equal(x, runs[0][0])
        assert it == runs[0][1]
    del ctx, runs
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,case", [(16, (2, 1, 1)), (64, (2, 2, 1)), (64, "smooth"),
                                    (128, (2, 2, 2))])
def test_direct_p_update_matches_transformed(n, case):
    """The opt-in p-update kernel that forms the neighbours' p = s + beta p_old where it reads
    them (no transformed ring; rbws_set_kernel_variant(3, 1)) against the default
    transformed-ring kernel: same sums in the same order (observed bitwise)."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    spec, ospec = _specs(case)
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    mus = op.sample_mus(ospec, 3, seed=59)
    delta = 1e-10
    try:
        _native.call("rbws_set_kernel_variant", 3, 0)
        base = _vcycle_and_solve(prob, mus, delta, n)
        _native.call("rbws_set_kernel_variant", 3, 1)
        var = _vcycle_and_solve(prob, mus, delta, n)
    finally:
        _native.call("rbws_set_kernel_variant", 3, -1)
    _compare_runs(var, base, 1e-13)
    print("direct vs transformed p-update: max |dx| =", float((var[1] - base[1]).abs().max()))


@pytest.mark.parametrize("n,case,m0", [(16, (2, 1, 1), 4), (32, (2, 2, 1), 4), (64, (2, 2, 1), 4),
                                       (64, (2, 2, 2), 4), (32, (2, 2, 2), 2), (128, (2, 2, 2), 4)])
def test_coarse_tail_matches_per_level_kernels(n, case, m0):
    """The opt-in fused coarse tail (levels <= 16 cells + the coarsest solve in one kernel,
    vectors in shared memory; rbws_set_kernel_variant(2, 1)) against the per-level kernels:
    every sum is taken in the same order, so V-cycles and solves agree to rounding (observed
    bitwise)."""
    pkg = _pkg()
    from paper_2311_13862_b200 import _native
    spec, ospec = _specs(case)
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, m0), m0=m0)
    mus = op.sample_mus(ospec, 5, seed=58)
    delta = 1e-10
    try:
        _native.call("rbws_set_kernel_variant", 2, 0)
        base = _vcycle_and_solve(prob, mus, delta, n)
        _native.call("rbws_set_kernel_variant", 2, 1)
        var = _vcycle_and_solve(prob, mus, delta, n)
    finally:
        _native.call("rbws_set_kernel_variant", 2, -1)
    _compare_runs(var, base, 1e-13)
    print("tail vs per-level: max |dv| =", float((var[0] - base[0]).abs().max()))


@pytest.mark.parametrize("n,count", [(256, 2), (512, 1)])
def test_fused_restrict_matches_separate_large(monkeypatch, n, count):
    """Pre-smoothing fused with the x/z restriction vs the separate kernels (N = 256, 512)."""
    pkg = _pkg()
    spec, ospec = _specs((2, 2, 2))
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    mus = op.sample_mus(ospec, count, seed=66)
    monkeypatch.setenv("RBWS_FUSED_RESTRICT", "1")
    fused = _vcycle_and_solve(prob, mus, 1e-10, n)
    monkeypatch.setenv("RBWS_FUSED_RESTRICT", "0")
    sep = _vcycle_and_solve(prob, mus, 1e-10, n)
    _compare_runs(fused, sep, 1e-12)


def test_slab4_512_matches_batched_512():
    """configs[4]: the 512^3 instance on 4 z-slabs (halo exchanges, replicated coarse
    levels, all-gathered dot partials) vs the one-instance batched solve."""
    pkg = _pkg()
    spec, ospec = _specs((2, 2, 2))
    n = 512
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    mu = op.sample_mus(ospec, 1, seed=77)
    ctx = pkg.mg_context_for(prob, mu)
    x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    assert reps[0].converged
    xb = x.clone()
    del ctx, x
    torch.cuda.empty_cache()
    xs, rs = pkg.slab_mgcg_solve(prob, mu[0], nslabs=4, delta=1e-10)
    assert rs.converged
    assert abs(rs.iterations - reps[0].iterations) <= 1
    assert (torch.linalg.norm(xs - xb) / torch.linalg.norm(xb)).item() <= 1e-9
    del xs, xb
    torch.cuda.empty_cache()


def test_rbi_mgcg_bench_config_matches_oracle():
    """configs[1] (the bench workload): r = 20 greedy from 1024 training parameters on the
    GPU, then RBI-MGCG for a batch; solutions / iterations vs the oracle's online stage and
    MGCG on the same model (warmstart.py:88-117; north_star: 1e-8 rel. L2, +-1 iteration)."""
    pkg = _pkg()
    spec, ospec = _specs((2, 2, 1))
    n = 64
    prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
    train = pkg.sample_mus(spec, 1024, seed=1000)
    hf = pkg.HighFidelitySolver(prob, delta=1e-14, l_max=100)
    model = pkg.l1roc_offline(train, 20, hf, prob, seed=0, on_degenerate="stop")
    assert model.dim >= 10
    test = pkg.sample_mus(spec, 64, seed=2000)
    ctx = pkg.mg_context_for(prob, test)
    cfg = pkg.MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=model.dim)
    x, reps = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), prob.rhs(), cfg, mg_ctx=ctx,
                                l1roc_model=model)
    got = pkg.from_padded(x, n, len(test))
    assert all(r.converged for r in reps)
    omodel = so.OracleL1rocModel(model.basis_numpy(), model.transform, model.collocation,
                                 model.solution_points, model.residual_points, model.chosen,
                                 model.indicator_history, model.saturated)
    oprob = op.OracleProblem(ospec, n, 4)
    for m in (0, 17, 63):
        xr, rr = so.rbi_mgcg_solve(oprob, test[m], omodel, delta=1e-10, l_max=60)
        assert abs(reps[m].iterations - rr.iterations) <= 1, m
        assert _rel(got[m], xr) <= 1e-8, m
