"""Generate golden vectors by running the REAL reference package.

Run in the build container (needs /root/reference; never on the GPU box):

    python tests/golden/make_golden.py          # golden_fd.npz
    python tests/golden/make_golden.py --gs     # golden_gs.npz (Gauss-Seidel smoother)
    python tests/golden/make_golden.py --msrb   # golden_msrb.npz (rbi-msrbcg)
    python tests/golden/make_golden.py --msrb-fem  # golden_msrb_fem.npz (rbi-msrbcg, example-1)
    python tests/golden/make_golden.py --fem    # golden_fem.npz (example-1, unmodified reference)
    python tests/golden/make_golden.py --fem2   # golden_fem2.npz (example-2, unmodified reference)
    python tests/golden/make_golden.py --experiment  # golden_experiment.npz (run_experiment loop)
    python tests/golden/make_golden.py --signatures  # ref_signatures.json (public API)

The reference (``/root/reference/pkg``) is copied to /tmp and its Cython
smoother extension built in place (reference setup.py), so the reference's
default compiled backend is the one exercised.  The BASELINE problems are
finite-volume operators the reference cannot assemble itself; they are fed
through the reference's own ``ProblemSpec``/``ParametricProblem`` API by
substituting its two assembly hooks (``grid.assemble_stiffness_kernel`` and
``grid.assemble_load``) with the oracle's FV term matrices.  Everything after
assembly — free-DoF slicing, prolongations, Galerkin coarsening
(grid.py:203-236), ``mg_context_for``/``mg_vcycle``/``mgcg_solve``
(multigrid.py), ``pcg_solve`` (krylov.py), ``l1roc_offline``/``l1roc_online``
(rb.py), ``HighFidelitySolver`` (hf.py) — is the unmodified reference code.

Outputs ``tests/golden/golden_fd.npz`` (small cases only).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg")
BUILD = Path("/tmp/rbws_ref_golden")


def _import_reference():
    if not (BUILD / "src/rbws").exists():
        shutil.copytree(REF, BUILD)
    if not list((BUILD / "src/rbws").glob("_smoothers*.so")):
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"],
                       cwd=BUILD, check=True, capture_output=True)
    sys.path.insert(0, str(BUILD / "src"))
    os.environ.pop("RBWS_KERNELS", None)
    import rbws
    assert rbws.BACKEND == "cython", rbws.BACKEND
    return rbws


class _FDKernel:
    """Marker standing in for a coefficient callable; carries (spec, q)."""

    def __init__(self, spec, q):
        self.spec, self.q = spec, q

    def __call__(self, x, y, z):  # pragma: no cover - never evaluated
        raise RuntimeError("FD terms are injected, not quadrature-assembled")


def reference_problem(rbws, fdspec, n, m0=4):
    """Build the reference ParametricProblem for an FD spec via its own API."""
    sys.path.insert(0, str(REPO))
    from oracle import problems as op
    import rbws.grid as rg
    from rbws.problems import DiffusionTerm, ProblemSpec

    terms = []
    for q in range(fdspec.n_terms):
        if fdspec.kind == "thermal-block":
            theta = (lambda mu, q=q: mu[q])
        else:
            theta = (lambda mu, q=q: 1.0 if q == 0 else mu[q - 1])
        terms.append(DiffusionTerm(theta=theta, kernel=_FDKernel(fdspec, q)))
    spec = ProblemSpec(pid=fdspec.pid, p=fdspec.p, bounds=np.asarray(fdspec.bounds),
                       diffusion_terms=tuple(terms),
                       source=lambda x, y, z, mu: np.zeros(np.broadcast(x, y, z).shape),
                       dirichlet=lambda x, y, z, mu: np.zeros(np.broadcast(x, y, z).shape),
                       source_mu_dependent=False)

    orig_k, orig_l = rg.assemble_stiffness_kernel, rg.assemble_load

    def fd_stiffness(nn, kernel, aniso=(1.0, 1.0, 1.0)):
        return op.assemble_term_full(kernel.spec, nn, kernel.q)

    def fd_load(nn, source, mu):
        return op.rhs_full(fdspec, nn)

    rg.assemble_stiffness_kernel, rg.assemble_load = fd_stiffness, fd_load
    try:
        levels = int(np.log2(n // m0)) + 1
        prob = rg.ParametricProblem(spec, levels=levels, m0=m0)
        prob.rhs(np.asarray([b[0] for b in fdspec.bounds]))  # populate cached load
    finally:
        rg.assemble_stiffness_kernel, rg.assemble_load = orig_k, orig_l
    return prob


def main():
    rbws = _import_reference()
    sys.path.insert(0, str(REPO))
    from oracle import problems as op
    from rbws.hf import HighFidelitySolver
    from rbws.multigrid import mg_context_for, mg_vcycle, mgcg_solve
    from rbws.rb import l1roc_offline
    from rbws.warmstart import MethodConfig, rbi_pcg_solve

    out = {}

    # 1. operators on every level (thermal block 2x1x1, n=8, m0=2 -> 3 levels)
    tb = op.thermal_block((2, 1, 1))
    prob = reference_problem(rbws, tb, 8, m0=2)
    mu = np.array([0.37, 4.2])
    for lvl in range(prob.mesh.levels):
        A = prob.operator(mu, level=lvl).toarray()
        out[f"ops_tb211_n8_l{lvl}"] = A
    out["ops_tb211_n8_mu"] = mu
    out["ops_tb211_n8_rhs"] = prob.rhs(mu)

    # 2. single V-cycle application on a seeded vector (thermal 2x2x1, n=16)
    tb4 = op.thermal_block((2, 2, 1))
    prob16 = reference_problem(rbws, tb4, 16, m0=4)
    mu = np.array([0.2, 3.0, 7.5, 0.9])
    ctx = mg_context_for(prob16, mu)
    v = np.random.default_rng(5).standard_normal(prob16.n_free)
    out["vcycle_tb221_n16_mu"] = mu
    out["vcycle_tb221_n16_in"] = v
    out["vcycle_tb221_n16_out"] = mg_vcycle(v, ctx)

    # 3. zero-init MGCG solves
    cases = [("tb211", tb, 16, 3, 1e-10), ("tb221", tb4, 32, 2, 1e-10),
             ("tb222", op.thermal_block((2, 2, 2)), 16, 2, 1e-12),
             ("smooth6", op.smooth_affine(6), 16, 2, 1e-12)]
    for tag, spec, n, cnt, delta in cases:
        p = reference_problem(rbws, spec, n, m0=4)
        mus = op.sample_mus(spec, cnt, seed=100 + n)
        xs, hists, its = [], [], []
        for m in mus:
            A, f = p.operator(m), p.rhs(m)
            c = mg_context_for(p, m)
            x, rep = mgcg_solve(A, f, np.zeros_like(f), c, delta=delta, l_max=60, mu=m)
            xs.append(x)
            hists.append(np.pad(rep.history, (0, 61 - len(rep.history)), constant_values=np.nan))
            its.append(rep.iterations)
        out[f"mgcg_{tag}_n{n}_mus"] = mus
        out[f"mgcg_{tag}_n{n}_x"] = np.array(xs)
        out[f"mgcg_{tag}_n{n}_hist"] = np.array(hists)
        out[f"mgcg_{tag}_n{n}_iters"] = np.array(its)
        out[f"mgcg_{tag}_n{n}_delta"] = np.array(delta)

    # 4. L1ROC offline (LU high fidelity, reference default) + online + RBI-MGCG
    p = reference_problem(rbws, tb4, 16, m0=4)
    train = op.sample_mus(tb4, 64, seed=1)
    test = op.sample_mus(tb4, 4, seed=8)
    hf = HighFidelitySolver(p, method="lu")
    model = l1roc_offline(list(train), 6, hf, p.operator, p.operator_rows, p.rhs, seed=3)
    out["l1roc_tb221_n16_train"] = train
    out["l1roc_tb221_n16_test"] = test
    out["l1roc_tb221_n16_W"] = model.basis
    out["l1roc_tb221_n16_T"] = model.transform
    out["l1roc_tb221_n16_colloc"] = model.collocation
    out["l1roc_tb221_n16_xs"] = model.solution_points
    out["l1roc_tb221_n16_xr"] = model.residual_points
    out["l1roc_tb221_n16_chosen_mus"] = model.chosen_mus
    out["l1roc_tb221_n16_hist"] = model.indicator_history
    out["l1roc_tb221_n16_saturated"] = np.array(model.saturated)
    # a saturating greedy (duplicate pick terminates early, rb.py:258-260)
    tb2 = op.thermal_block((2, 1, 1))
    p2 = reference_problem(rbws, tb2, 16, m0=4)
    tr2 = op.sample_mus(tb2, 32, seed=1)
    m2 = l1roc_offline(list(tr2), 8, HighFidelitySolver(p2, method="lu"), p2.operator,
                       p2.operator_rows, p2.rhs, seed=0)
    out["l1roc_tb211_n16_train"] = tr2
    out["l1roc_tb211_n16_W"] = m2.basis
    out["l1roc_tb211_n16_colloc"] = m2.collocation
    out["l1roc_tb211_n16_hist"] = m2.indicator_history
    out["l1roc_tb211_n16_saturated"] = np.array(m2.saturated)
    from rbws.rb import l1roc_online
    u0s, cs, xs, its, hists = [], [], [], [], []
    for m in test:
        A, f = p.operator(m), p.rhs(m)
        u0, c = l1roc_online(model, A, f)
        u0s.append(u0)
        cs.append(c)
        cfg = MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=model.dim)
        x, rep = rbi_pcg_solve(A, f, cfg, mg_ctx=mg_context_for(p, m), l1roc_model=model, mu=m)
        xs.append(x)
        its.append(rep.iterations)
        hists.append(np.pad(rep.history, (0, 61 - len(rep.history)), constant_values=np.nan))
    out["l1roc_tb221_n16_u0"] = np.array(u0s)
    out["l1roc_tb221_n16_c"] = np.array(cs)
    out["rbi_tb221_n16_x"] = np.array(xs)
    out["rbi_tb221_n16_iters"] = np.array(its)
    out["rbi_tb221_n16_hist"] = np.array(hists)

    dest = REPO / "tests/golden/golden_fd.npz"
    np.savez_compressed(dest, **out)
    print(f"wrote {dest} ({dest.stat().st_size/1e6:.2f} MB, {len(out)} arrays)")


def main_gs():
    """Gauss-Seidel smoother goldens (smoother="gs": forward GS before, backward after the
    coarse correction, multigrid.py:132-152) -> tests/golden/golden_gs.npz."""
    rbws = _import_reference()
    sys.path.insert(0, str(REPO))
    from oracle import problems as op
    from rbws.multigrid import mg_context_for, mg_vcycle, mgcg_solve

    out = {}
    tb4 = op.thermal_block((2, 2, 1))
    prob16 = reference_problem(rbws, tb4, 16, m0=4)
    mu = np.array([0.2, 3.0, 7.5, 0.9])
    v = np.random.default_rng(5).standard_normal(prob16.n_free)
    out["gs_vcycle_tb221_n16_mu"] = mu
    out["gs_vcycle_tb221_n16_in"] = v
    for nu in (1, 2):
        ctx = mg_context_for(prob16, mu, nu=nu, smoother="gs")
        out[f"gs_vcycle_tb221_n16_nu{nu}_out"] = mg_vcycle(v, ctx)
    cases = [("tb221", tb4, 16, 2, 1e-10), ("smooth6", op.smooth_affine(6), 16, 2, 1e-12),
             ("tb222", op.thermal_block((2, 2, 2)), 32, 1, 1e-10)]
    for tag, spec, n, cnt, delta in cases:
        p = reference_problem(rbws, spec, n, m0=4)
        mus = op.sample_mus(spec, cnt, seed=300 + n)
        xs, hists, its = [], [], []
        for m in mus:
            A, f = p.operator(m), p.rhs(m)
            c = mg_context_for(p, m, smoother="gs")
            x, rep = mgcg_solve(A, f, np.zeros_like(f), c, delta=delta, l_max=60, mu=m)
            xs.append(x)
            hists.append(np.pad(rep.history, (0, 61 - len(rep.history)), constant_values=np.nan))
            its.append(rep.iterations)
        out[f"gs_mgcg_{tag}_n{n}_mus"] = mus
        out[f"gs_mgcg_{tag}_n{n}_x"] = np.array(xs)
        out[f"gs_mgcg_{tag}_n{n}_hist"] = np.array(hists)
        out[f"gs_mgcg_{tag}_n{n}_iters"] = np.array(its)
        out[f"gs_mgcg_{tag}_n{n}_delta"] = np.array(delta)
    dest = REPO / "tests/golden/golden_gs.npz"
    np.savez_compressed(dest, **out)
    print(f"wrote {dest} ({dest.stat().st_size/1e6:.2f} MB, {len(out)} arrays)")


def main_msrb():
    """rbi-msrbcg goldens (msrb_train + MsrbPreconditioner through the reference's
    rbi_pcg_solve) -> tests/golden/golden_msrb.npz."""
    rbws = _import_reference()
    sys.path.insert(0, str(REPO))
    from oracle import problems as op
    from rbws.hf import HighFidelitySolver
    from rbws.msrb import msrb_train
    from rbws.warmstart import MethodConfig, rbi_pcg_solve

    out = {}
    tb4 = op.thermal_block((2, 2, 1))
    p = reference_problem(rbws, tb4, 16, m0=4)
    train = op.sample_mus(tb4, 48, seed=11)
    test = op.sample_mus(tb4, 3, seed=12)
    N, K = 10, 8
    hf = HighFidelitySolver(p, method="lu")
    hier = msrb_train(list(train), N, K, hf, p.operator, p.rhs)
    out["msrb_tb221_n16_train"] = train
    out["msrb_tb221_n16_test"] = test
    out["msrb_tb221_n16_NK"] = np.array([N, K])
    out["msrb_tb221_n16_init"] = hier.init_basis.basis
    out["msrb_tb221_n16_init_eig"] = hier.init_basis.eigenvalues
    for k, W in enumerate(hier.bases):
        out[f"msrb_tb221_n16_basis{k}"] = W
    xs, its, hists = [], [], []
    for m in test:
        A, f = p.operator(m), p.rhs(m)
        cfg = MethodConfig("rbi-msrbcg", delta=1e-10, l_max=60, N=N, K_max=K)
        x, rep = rbi_pcg_solve(A, f, cfg, msrb_hier=hier, mu=m)
        xs.append(x)
        its.append(rep.iterations)
        hists.append(np.pad(rep.history, (0, 61 - len(rep.history)), constant_values=np.nan))
    out["msrb_tb221_n16_x"] = np.array(xs)
    out["msrb_tb221_n16_iters"] = np.array(its)
    out["msrb_tb221_n16_hist"] = np.array(hists)
    dest = REPO / "tests/golden/golden_msrb.npz"
    np.savez_compressed(dest, **out)
    print(f"wrote {dest} ({dest.stat().st_size/1e6:.2f} MB, {len(out)} arrays)")


def main_msrb_fem():
    """rbi-msrbcg on the reference's own assembled problem example-1 (unmodified reference,
    no hooks: per-parameter right-hand sides with lifted Dirichlet data) ->
    tests/golden/golden_msrb_fem.npz."""
    rbws = _import_reference()
    from rbws.grid import ParametricProblem
    from rbws.hf import HighFidelitySolver
    from rbws.msrb import msrb_train
    from rbws.problems import get_problem
    from rbws.sampling import lhs_sample
    from rbws.warmstart import MethodConfig, rbi_pcg_solve

    out = {}
    spec = get_problem("example-1")
    p = ParametricProblem(spec, levels=3, m0=4)
    train = lhs_sample(spec.p, 24, spec.bounds, seed=21)
    test = lhs_sample(spec.p, 3, spec.bounds, seed=22)
    N, K = 6, 4
    hf = HighFidelitySolver(p, method="lu")
    hier = msrb_train(list(train), N, K, hf, p.operator, p.rhs)
    k0 = "msrb_ex1_n16"
    out[f"{k0}_train"] = np.asarray(train)
    out[f"{k0}_test"] = np.asarray(test)
    out[f"{k0}_NK"] = np.array([N, K])
    out[f"{k0}_init"] = hier.init_basis.basis
    out[f"{k0}_init_eig"] = hier.init_basis.eigenvalues
    for k, W in enumerate(hier.bases):
        out[f"{k0}_basis{k}"] = W
    xs, its, hists = [], [], []
    for m in test:
        A, f = p.operator(m), p.rhs(m)
        cfg = MethodConfig("rbi-msrbcg", delta=1e-10, l_max=60, N=N, K_max=K)
        x, rep = rbi_pcg_solve(A, f, cfg, msrb_hier=hier, mu=m)
        xs.append(x)
        its.append(rep.iterations)
        hists.append(np.pad(rep.history, (0, 61 - len(rep.history)), constant_values=np.nan))
    out[f"{k0}_x"] = np.array(xs)
    out[f"{k0}_iters"] = np.array(its)
    out[f"{k0}_hist"] = np.array(hists)
    dest = REPO / "tests/golden/golden_msrb_fem.npz"
    np.savez_compressed(dest, **out)
    print(f"wrote {dest} ({dest.stat().st_size/1e6:.2f} MB, {len(out)} arrays)", its)


def main_fem():
    """The reference's own assembled problem example-1 (Q1 FEM, Dirichlet, p = 2) through
    its unmodified API -> tests/golden/golden_fem.npz: per-level operators (CSR) and
    right-hand sides, a V-cycle, zero-init MGCG and L1ROC RBI-MGCG solves."""
    rbws = _import_reference()
    from rbws.grid import ParametricProblem
    from rbws.hf import HighFidelitySolver
    from rbws.multigrid import mg_context_for, mg_vcycle, mgcg_solve
    from rbws.problems import get_problem
    from rbws.rb import l1roc_offline
    from rbws.sampling import lhs_sample
    from rbws.warmstart import MethodConfig, rbi_pcg_solve

    out = {}
    spec = get_problem("example-1")
    rng = np.random.default_rng(5)
    mus = np.array([[0.3, 0.25], [1.7, 0.8], [1.0, 0.5], [0.05, 0.95]])
    for tag, levels, m0 in (("n16m4", 3, 4), ("n16m2", 4, 2), ("n32m4", 4, 4)):
        p = ParametricProblem(spec, levels=levels, m0=m0)
        k = f"fem_{tag}"
        out[f"{k}_mus"] = mus
        mu = mus[0]
        for lvl in range(p.mesh.levels):
            A = p.operator(mu, level=lvl).tocsr()
            if tag == "n32m4" and lvl == p.mesh.levels - 1:
                v = rng.standard_normal(A.shape[0])
                out[f"{k}_op{lvl}_v"] = v
                out[f"{k}_op{lvl}_Av"] = A @ v
                continue
            A.sort_indices()
            out[f"{k}_op{lvl}_data"] = A.data
            out[f"{k}_op{lvl}_indices"] = A.indices.astype(np.int64)
            out[f"{k}_op{lvl}_indptr"] = A.indptr.astype(np.int64)
        out[f"{k}_rhs"] = np.array([p.rhs(m) for m in mus])
        ctx = mg_context_for(p, mu)
        b = rng.standard_normal(p.n_free)
        out[f"{k}_vcyc_b"] = b
        out[f"{k}_vcyc"] = mg_vcycle(b, ctx)
        xs, its, hists = [], [], []
        for m in mus:
            A, f = p.operator(m), p.rhs(m)
            x, rep = mgcg_solve(A, f, np.zeros_like(f), mg_context_for(p, m), delta=1e-10,
                                l_max=60)
            xs.append(x)
            its.append(rep.iterations)
            hists.append(np.pad(rep.history, (0, 61 - len(rep.history)), constant_values=np.nan))
        out[f"{k}_mgcg_x"] = np.array(xs)
        out[f"{k}_mgcg_iters"] = np.array(its)
        out[f"{k}_mgcg_hist"] = np.array(hists)
        if tag != "n16m4":
            continue
        # Gauss-Seidel V-cycle smoother (forward before / backward after, multigrid.py:137-138)
        xs, its = [], []
        for m in mus:
            A, f = p.operator(m), p.rhs(m)
            x, rep = mgcg_solve(A, f, np.zeros_like(f), mg_context_for(p, m, smoother="gs"),
                                delta=1e-10, l_max=60)
            xs.append(x)
            its.append(rep.iterations)
        out[f"{k}_gs_x"] = np.array(xs)
        out[f"{k}_gs_iters"] = np.array(its)
        # L1ROC greedy (reference default LU high fidelity) + RBI-MGCG warm-started solves
        train = np.array(lhs_sample(spec.p, 24, spec.bounds, seed=3))
        model = l1roc_offline(list(train), 6, HighFidelitySolver(p), p.operator,
                              p.operator_rows, p.rhs, seed=0)
        out[f"{k}_l1_train"] = train
        out[f"{k}_l1_basis"] = model.basis
        out[f"{k}_l1_transform"] = model.transform
        out[f"{k}_l1_colloc"] = model.collocation
        out[f"{k}_l1_chosen"] = model.chosen_mus
        out[f"{k}_l1_hist"] = model.indicator_history
        xs, its = [], []
        for m in mus:
            A, f = p.operator(m), p.rhs(m)
            cfg = MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=model.dim)
            x, rep = rbi_pcg_solve(A, f, cfg, mg_ctx=mg_context_for(p, m), l1roc_model=model)
            xs.append(x)
            its.append(rep.iterations)
        out[f"{k}_rbi_x"] = np.array(xs)
        out[f"{k}_rbi_iters"] = np.array(its)
    dest = REPO / "tests/golden/golden_fem.npz"
    np.savez_compressed(dest, **out)
    print(f"wrote {dest} ({dest.stat().st_size/1e6:.2f} MB, {len(out)} arrays)")


def main_fem2():
    """The reference's example-2 (zero-flux face x = 1, anisotropic piecewise-constant
    coefficient, mu-dependent source, plane smoothers) through its unmodified API ->
    tests/golden/golden_fem2.npz: per-level operators, right-hand sides, V-cycles with
    the plane-Jacobi (default) and plane-z smoothers, zero-init MGCG solves."""
    rbws = _import_reference()
    from rbws.grid import ParametricProblem
    from rbws.multigrid import mg_context_for, mg_vcycle, mgcg_solve
    from rbws.problems import get_problem

    out = {}
    spec = get_problem("example-2")
    rng = np.random.default_rng(7)
    mus = np.array([[0.1, 1.0, 0.5, 0.4, 0.6, 0.5, 0.25],
                    [0.9, 0.2, 0.3, 0.55, 0.45, 0.42, 0.5],
                    [0.5, 0.5, 1.0, 0.6, 0.4, 0.6, 0.33]])
    for tag, levels, m0 in (("n8m2", 3, 2), ("n16m4", 3, 4)):
        p = ParametricProblem(spec, levels=levels, m0=m0)
        k = f"fem2_{tag}"
        out[f"{k}_mus"] = mus
        out[f"{k}_free"] = p.free_by_level[-1].astype(np.int64)
        for lvl in range(p.mesh.levels):
            A = p.operator(mus[0], level=lvl).tocsr()
            A.sort_indices()
            out[f"{k}_op{lvl}_data"] = A.data
            out[f"{k}_op{lvl}_indices"] = A.indices.astype(np.int64)
            out[f"{k}_op{lvl}_indptr"] = A.indptr.astype(np.int64)
        out[f"{k}_rhs"] = np.array([p.rhs(m) for m in mus])
        b = rng.standard_normal(p.n_free)
        out[f"{k}_vcyc_b"] = b
        for sm in ("plane-jacobi", "plane-z", "jacobi"):
            ctx = mg_context_for(p, mus[0], smoother=sm if sm != "plane-jacobi" else "auto")
            assert ctx.smoother_kind == sm
            key = sm.replace("-", "")
            out[f"{k}_vcyc_{key}"] = mg_vcycle(b, ctx)
            xs, its, hists = [], [], []
            for m in mus:
                A, f = p.operator(m), p.rhs(m)
                x, rep = mgcg_solve(A, f, np.zeros_like(f),
                                    mg_context_for(p, m, smoother=sm), delta=1e-10, l_max=80)
                xs.append(x)
                its.append(rep.iterations)
                hists.append(np.pad(rep.history, (0, 81 - len(rep.history)),
                                    constant_values=np.nan))
            out[f"{k}_{key}_x"] = np.array(xs)
            out[f"{k}_{key}_iters"] = np.array(its)
            out[f"{k}_{key}_hist"] = np.array(hists)
    dest = REPO / "tests/golden/golden_fem2.npz"
    np.savez_compressed(dest, **out)
    print(f"wrote {dest} ({dest.stat().st_size/1e6:.2f} MB, {len(out)} arrays)")


EXPERIMENTS = {
    # tag: (problem, levels, m0, n_train, n_test, rb_dims, deltas)
    "ex1": ("example-1", 3, 4, 16, 3, (4, 6), (1e-10, 1e-12)),
    "ex2": ("example-2", 3, 4, 12, 3, (4,), (1e-10,)),
}


def main_experiment():
    """The reference's own experiment driver, unmodified (experiment.py:108-172: LHS train /
    test sets, the LU-backed L1ROC greedy, per-parameter mg_context_for + rbi_pcg_solve for
    mgcg and rbi-mgcg) -> tests/golden/golden_experiment.npz.  The loop's calls are recorded
    through wrappers around the names it imports (training / test sets, the trained model,
    every solve's solution and report); nothing inside the loop is changed.  The compat layer
    (paper_2311_13862_b200/compat.py) replays the same loop on the GPU against these."""
    rbws = _import_reference()
    import rbws.experiment as ex

    out = {}
    for tag, (pid, levels, m0, n_train, n_test, dims, deltas) in EXPERIMENTS.items():
        rec = {"lhs": [], "model": None, "solves": []}
        orig_lhs, orig_off, orig_rbi = ex.lhs_sample, ex.l1roc_offline, ex.rbi_pcg_solve

        def lhs(*a, **k):
            pts = orig_lhs(*a, **k)
            rec["lhs"].append(np.array(pts))
            return pts

        def off(*a, **k):
            rec["model"] = orig_off(*a, **k)
            return rec["model"]

        def rbi(A, f, mcfg, **k):
            x, rep = orig_rbi(A, f, mcfg, **k)
            rec["solves"].append((mcfg.method, mcfg.N, mcfg.delta, x, rep))
            return x, rep

        ex.lhs_sample, ex.l1roc_offline, ex.rbi_pcg_solve = lhs, off, rbi
        try:
            cfg = ex.ExperimentConfig(problem=pid, levels=levels, m0=m0, n_train=n_train,
                                      n_test=n_test, seed=0, methods=("mgcg", "rbi-mgcg"),
                                      rb_dims=dims, deltas=deltas, l_max=60)
            ex.run_experiment(cfg)
        finally:
            ex.lhs_sample, ex.l1roc_offline, ex.rbi_pcg_solve = orig_lhs, orig_off, orig_rbi
        k = f"exp_{tag}"
        out[f"{k}_train"], out[f"{k}_test"] = rec["lhs"]
        m = rec["model"]
        out[f"{k}_colloc"] = m.collocation
        out[f"{k}_chosen"] = m.chosen_mus
        out[f"{k}_hist"] = m.indicator_history
        out[f"{k}_basis"] = m.basis
        keys = []
        for i, (method, N, delta, x, rep) in enumerate(rec["solves"]):
            keys.append(f"{method}|{N}|{delta!r}")
            out[f"{k}_x{i}"] = x
            out[f"{k}_it{i}"] = np.array(rep.iterations)
            out[f"{k}_h{i}"] = np.array(rep.history)
        out[f"{k}_keys"] = np.array(keys)
    dest = REPO / "tests/golden/golden_experiment.npz"
    np.savez_compressed(dest, **out)
    print(f"wrote {dest} ({dest.stat().st_size/1e6:.2f} MB, {len(out)} arrays)")


SIGNATURE_NAMES = ["ParametricProblem", "mg_context_for", "mg_vcycle", "mgcg_solve", "pcg_solve",
                   "cg_solve", "rbi_pcg_solve", "make_initial_guess", "initial_residual",
                   "MethodConfig", "l1roc_offline", "l1roc_online", "HighFidelitySolver",
                   "msrb_train", "lhs_sample", "get_problem"]


def main_signatures():
    """Parameter names / defaults of the reference's public solver API ->
    tests/golden/ref_signatures.json (the compat layer's signature pin)."""
    import inspect
    import json
    rbws = _import_reference()
    out = {}
    for name in SIGNATURE_NAMES:
        obj = getattr(rbws, name)
        if inspect.isclass(obj):
            obj = obj.__init__
        out[name] = [[p.name, None if p.default is inspect._empty else repr(p.default)]
                     for p in inspect.signature(obj).parameters.values() if p.name != "self"]
    dest = REPO / "tests/golden/ref_signatures.json"
    dest.write_text(json.dumps(out, indent=1))
    print(f"wrote {dest}")


if __name__ == "__main__":
    if "--signatures" in sys.argv:
        main_signatures()
        sys.exit(0)
    if "--experiment" in sys.argv:
        main_experiment()
        sys.exit(0)
    if "--fem2" in sys.argv:
        main_fem2()
        sys.exit(0)
    if "--fem" in sys.argv:
        main_fem()
        sys.exit(0)
    if "--msrb-fem" in sys.argv:
        main_msrb_fem()
        sys.exit(0)
    if "--msrb" in sys.argv:
        main_msrb()
        sys.exit(0)
    if "--gs" in sys.argv:
        main_gs()
        sys.exit(0)
    main()
