"""The reference's own assembled problem example-1 (Q1 FEM, mu-dependent Dirichlet data)
on the CUDA path (stored-coefficient hierarchy, through the C ABI) vs the unmodified
reference's goldens (tests/golden/golden_fem.npz) and the oracle."""

from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

G = np.load(Path(__file__).parent / "golden" / "golden_fem.npz")
CASES = (("n16m4", 3, 4), ("n16m2", 4, 2), ("n32m4", 4, 4))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build
    build.build(verbose=False)


def _pkg():
    import paper_2311_13862_b200 as pkg
    return pkg


def canonical_points(idx, n):
    """example-1 is invariant under the y<->z swap and the point inversion through the cube
    centre, so DEIM's |residual| maxima tie across each orbit and which member a solver
    picks depends on the last bit of its arithmetic.  Map interior indices to the orbit's
    smallest member (a tie-invariant view of the collocation set)."""
    m = n - 1
    idx = np.asarray(idx, dtype=np.int64)
    i, j, k = idx % m, (idx // m) % m, idx // (m * m)
    orbit = [(i, j, k), (i, k, j), (m - 1 - i, m - 1 - j, m - 1 - k),
             (m - 1 - i, m - 1 - k, m - 1 - j)]
    return np.sort(np.min([a + m * (b + m * c) for a, b, c in orbit], axis=0))


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _golden_op(k, lvl):
    ip = G[f"{k}_op{lvl}_indptr"]
    return sp.csr_matrix((G[f"{k}_op{lvl}_data"], G[f"{k}_op{lvl}_indices"], ip),
                         shape=(len(ip) - 1,) * 2)


@pytest.fixture(scope="module")
def probs():
    pkg = _pkg()
    spec = pkg.get_problem("example-1")
    return {t: pkg.ParametricProblem(spec, levels=l, m0=m) for t, l, m in CASES}


@pytest.mark.parametrize("tag,levels,m0", CASES)
def test_fem_operators_rhs_vcycle(probs, tag, levels, m0):
    pkg = _pkg()
    p, k = probs[tag], f"fem_{tag}"
    assert type(p).__name__ == "FemProblem"
    mus = G[f"{k}_mus"]
    ctx = pkg.mg_context_for(p, mus)
    A = pkg.BatchOperator(ctx)
    rng = np.random.default_rng(1)
    for lvl in range(levels):
        n = p.cells[lvl]
        v = rng.standard_normal((len(mus), (n - 1) ** 3))
        y = pkg.from_padded(A.apply(pkg.to_padded(v, n), level=lvl), n, len(mus))
        if f"{k}_op{lvl}_data" in G:
            ref = _golden_op(k, lvl) @ v[0]
            assert _rel(y[0], ref) <= 1e-13, lvl
        else:
            vb = _pad_batch(pkg, G[f"{k}_op{lvl}_v"], n, len(mus))
            y0 = pkg.from_padded(A.apply(vb, level=lvl), n, len(mus))
            assert _rel(y0[0], G[f"{k}_op{lvl}_Av"]) <= 1e-13
        # every instance against its own host operator
        for m in range(len(mus)):
            assert _rel(y[m], p.operator_host(mus[m], lvl) @ v[m]) <= 1e-13
    f = pkg.from_padded(p.rhs(mus), p.n, len(mus))
    assert _rel(f, G[f"{k}_rhs"]) <= 1e-13
    # one V-cycle (instance 0 = the golden's mu)
    b = np.tile(G[f"{k}_vcyc_b"], (len(mus), 1))
    out = pkg.from_padded(pkg.mg_vcycle(pkg.to_padded(b, p.n), ctx), p.n, len(mus))
    assert _rel(out[0], G[f"{k}_vcyc"]) <= 1e-12


def _pad_batch(pkg, v, n, count):
    return pkg.to_padded(np.tile(v, (count, 1)), n)


@pytest.mark.parametrize("tag,levels,m0", CASES)
def test_fem_mgcg_matches_reference(probs, tag, levels, m0):
    """Zero-init MGCG to 1e-10: solutions within 1e-8 relative L2 and iteration counts
    within +-1 of the reference (north_star tolerance)."""
    pkg = _pkg()
    p, k = probs[tag], f"fem_{tag}"
    mus = G[f"{k}_mus"]
    ctx = pkg.mg_context_for(p, mus)
    x, reps = pkg.mgcg_solve(None, None, None, ctx, delta=1e-10, l_max=60)
    got = pkg.from_padded(x, p.n, len(mus))
    for m in range(len(mus)):
        assert _rel(got[m], G[f"{k}_mgcg_x"][m]) <= 1e-8
        assert abs(reps[m].iterations - G[f"{k}_mgcg_iters"][m]) <= 1
        assert reps[m].converged
        hist = G[f"{k}_mgcg_hist"][m][: reps[m].iterations + 1]
        assert np.allclose(reps[m].history[: len(hist)], hist, rtol=1e-6)


def test_fem_term_apply_and_streaming(probs):
    pkg = _pkg()
    p = probs["n16m4"]
    mus = G["fem_n16m4_mus"]
    n = p.n
    rng = np.random.default_rng(2)
    v = rng.standard_normal((3, (n - 1) ** 3))
    for q in range(p.spec.n_terms):
        y = pkg.from_padded(p.term_apply(q, pkg.to_padded(v, n), 3), n, 3)
        T = p.terms_by_level[-1][q]
        for m in range(3):
            assert _rel(y[m], T @ v[m]) <= 1e-13
    # streaming download of converged instances == device solutions (bitwise)
    ctx = pkg.mg_context_for(p, mus)
    x, _ = pkg.mgcg_solve(None, None, None, ctx, delta=1e-10, l_max=60)
    host = torch.zeros(len(mus) * n ** 3, dtype=torch.float64).pin_memory()
    cs = torch.cuda.Stream()
    x2, _ = pkg.mgcg_solve(None, None, None, ctx, delta=1e-10, l_max=60, out_host=host,
                           copy_stream=cs)
    cs.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(host, x[: len(mus) * n ** 3].cpu())
    assert torch.equal(x2, x)


def test_fem_example2_goes_to_the_full_node_path():
    """The padded stored-coefficient path refuses free boundary nodes; the factory sends
    example-2 to the full-node path (fem_fn.py, tests/test_gpu_fem_fn.py), which has no
    padded-layout hierarchy handle (asking for one fails loudly)."""
    pkg = _pkg()
    from paper_2311_13862_b200.fem import FemProblem
    from paper_2311_13862_b200.fem_fn import FnFemProblem
    with pytest.raises(NotImplementedError):
        FemProblem(pkg.get_problem("example-2"), levels=3, m0=2)
    p = pkg.ParametricProblem(pkg.get_problem("example-2"), levels=3, m0=2)
    assert isinstance(p, FnFemProblem)
    with pytest.raises(NotImplementedError):
        p.handle


def test_fem_l1roc_rbi_mgcg_matches_reference(probs):
    """Greedy L1ROC on the device (MGCG high fidelity at 1e-14, the reference ran LU) and
    RBI-MGCG on example-1 vs the unmodified reference: same chosen parameters, indicator
    history and collocation orbits (ties across the problem's symmetry, canonical_points),
    same basis span, warm-started solutions 1e-8 and iterations +-1."""
    pkg = _pkg()
    p, k = probs["n16m4"], "fem_n16m4"
    train = G[f"{k}_l1_train"]
    model = pkg.l1roc_offline(train, 6, pkg.HighFidelitySolver(p), p, seed=0)
    assert np.array_equal(canonical_points(model.collocation, p.n),
                          canonical_points(G[f"{k}_l1_colloc"], p.n))
    assert np.allclose(model.chosen_mus, G[f"{k}_l1_chosen"])
    assert np.allclose(model.indicator_history, G[f"{k}_l1_hist"], rtol=1e-6)
    W = model.basis_numpy()
    Wr = G[f"{k}_l1_basis"]
    proj = W @ np.linalg.lstsq(W, Wr, rcond=None)[0]
    assert np.linalg.norm(proj - Wr) <= 1e-8 * np.linalg.norm(Wr)
    mus = G[f"{k}_mus"]
    ctx = pkg.mg_context_for(p, mus)
    cfg = pkg.MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=model.dim)
    x, reps = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), p.rhs(mus), cfg, mg_ctx=ctx,
                                l1roc_model=model)
    got = pkg.from_padded(x, p.n, len(mus))
    for m in range(len(mus)):
        assert _rel(got[m], G[f"{k}_rbi_x"][m]) <= 1e-8
        assert abs(reps[m].iterations - G[f"{k}_rbi_iters"][m]) <= 1


def test_fem_unsupported_paths_fail_loudly(probs):
    """rbi-msrbcg runs on example-1 (tests/test_gpu_msrb.py); the full-node layout of example-2
    has no Gauss-Seidel sweep, so the multispace method is refused there with a clear error."""
    pkg = _pkg()
    spec2 = pkg.get_problem("example-2")
    p2 = pkg.ParametricProblem(spec2, levels=2, m0=4)
    mus = np.array(pkg.problems.lhs_sample(spec2.p, 2, spec2.bounds, seed=1))
    with pytest.raises(NotImplementedError):
        pkg.msrb_train(mus, 2, 1, None, p2)


def test_fem_gs_smoother_matches_reference(probs):
    """smoother="gs" (forward / backward Gauss-Seidel sweeps on the stored coefficients of
    every level) on example-1 vs the unmodified reference."""
    pkg = _pkg()
    p, k = probs["n16m4"], "fem_n16m4"
    mus = G[f"{k}_mus"]
    ctx = pkg.mg_context_for(p, mus, smoother="gs")
    x, reps = pkg.mgcg_solve(None, None, None, ctx, delta=1e-10, l_max=60)
    got = pkg.from_padded(x, p.n, len(mus))
    for m in range(len(mus)):
        assert _rel(got[m], G[f"{k}_gs_x"][m]) <= 1e-8
        assert abs(reps[m].iterations - G[f"{k}_gs_iters"][m]) <= 1


def test_fem_full_size_properties():
    """At the bench size (64^3, 64 instances): every instance converges with a true residual
    <= tol, the V-cycle is linear and symmetric (b1 . M b2 == b2 . M b1), and repeated solves
    are bitwise identical."""
    pkg = _pkg()
    spec = pkg.get_problem("example-1")
    p = pkg.ParametricProblem(spec, levels=5, m0=4)
    mus = np.array(pkg.problems.lhs_sample(spec.p, 64, spec.bounds, seed=9))
    ctx = pkg.mg_context_for(p, mus)
    x1, reps = pkg.mgcg_solve(None, None, None, ctx, delta=1e-10, l_max=60)
    assert all(r.converged and r.true_residual <= 1e-10 for r in reps)
    x2, _ = pkg.mgcg_solve(None, None, None, ctx, delta=1e-10, l_max=60)
    assert torch.equal(x1, x2)
    n, c = p.n, len(mus)
    rng = np.random.default_rng(4)
    b1 = rng.standard_normal((c, (n - 1) ** 3))
    b2 = rng.standard_normal((c, (n - 1) ** 3))
    M = lambda b: pkg.from_padded(pkg.mg_vcycle(pkg.to_padded(b, n), ctx), n, c)
    m1, m2, m12 = M(b1), M(b2), M(2.0 * b1 + b2)
    assert np.abs(m12 - (2.0 * m1 + m2)).max() <= 1e-11 * np.abs(m12).max()
    s12 = np.einsum("ij,ij->i", b1, m2)
    s21 = np.einsum("ij,ij->i", b2, m1)
    assert np.all(np.abs(s12 - s21) <= 1e-11 * np.abs(s12))


class _HostView:
    """The product's host-side operators through the oracle solver interface."""

    def __init__(self, p):
        self.p, self.prolongations, self.levels = p, p.prolongations, p.levels

    def operator(self, mu, level=None):
        return self.p.operator_host(mu, level)


def _five_term_spec(pkg):
    from paper_2311_13862_b200 import fem
    def blk(k):
        return lambda x, y, z: (((x * 5).astype(int) % 5) == k).astype(np.float64) + 0.1
    return fem.FemProblemSpec(
        pid="five-blocks", p=5, bounds=np.array([[0.5, 2.0]] * 5),
        diffusion_terms=tuple(fem.DiffusionTerm((lambda q: (lambda mu: mu[q]))(q), blk(q))
                              for q in range(5)),
        source=lambda x, y, z, mu: np.ones(np.broadcast(x, y, z).shape),
        dirichlet=lambda x, y, z, mu: x * mu[0], source_mu_dependent=False)


@pytest.mark.parametrize("nu", [1, 2])
def test_fem_five_terms_and_nu(nu):
    """Q = 5 (> 4: the finest level keeps per-instance coefficients) and nu = 1, 2 against
    the oracle solvers on the product's own host operators."""
    from oracle import solvers as so
    pkg = _pkg()
    spec = _five_term_spec(pkg)
    p = pkg.ParametricProblem(spec, levels=3, m0=4)
    mus = np.array([[0.6, 1.9, 1.0, 0.7, 1.3], [1.5, 0.5, 0.9, 2.0, 1.1]])
    ctx = pkg.mg_context_for(p, mus, nu=nu)
    x, reps = pkg.mgcg_solve(None, None, None, ctx, delta=1e-10, l_max=60)
    got = pkg.from_padded(x, p.n, len(mus))
    f = p.rhs_host(mus)
    hv = _HostView(p)
    for m, mu in enumerate(mus):
        A = p.operator_host(mu)
        xr, rr = so.mgcg_solve(A, f[m], np.zeros_like(f[m]), so.mg_context_for(hv, mu, nu=nu),
                               delta=1e-10, l_max=60)
        assert _rel(got[m], xr) <= 1e-8
        assert abs(reps[m].iterations - rr.iterations) <= 1


def test_fem_pcg_edge_cases(probs):
    """The stored-coefficient PCG on the reference's edge cases (krylov.py:42-109): l_max = 0,
    an exact initial guess, a zero right-hand side (absolute norms)."""
    pkg = _pkg()
    p = probs["n16m4"]
    mus = G["fem_n16m4_mus"]
    c = len(mus)
    ctx = pkg.mg_context_for(p, mus)
    f = p.rhs(mus)
    x, reps = pkg.mgcg_solve(None, f, None, ctx, delta=1e-10, l_max=0)
    assert all(r.iterations == 0 and len(r.history) == 1 and not r.converged for r in reps)
    assert float(x.abs().max()) == 0.0
    xs, _ = pkg.mgcg_solve(None, f, None, ctx, delta=1e-13, l_max=60)
    _, reps2 = pkg.mgcg_solve(None, f, xs, ctx, delta=1e-10, l_max=60)
    assert all(r.iterations == 0 and r.converged for r in reps2)
    z = torch.zeros_like(f)
    xz, reps3 = pkg.mgcg_solve(None, z, None, ctx, delta=1e-10, l_max=60)
    assert all(r.iterations == 0 and r.converged and r.absolute_norms for r in reps3)
    assert float(xz.abs().max()) == 0.0
