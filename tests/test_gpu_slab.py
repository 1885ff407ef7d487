"""Slab-decomposed single-instance MGCG (configs[4] path) vs the CPU oracle.

All slabs live in one process on one GPU (halo planes by device copies): the
same native solver, kernels and exchange schedule as the one-process-per-GPU
NCCL run, whose only difference is the transport of the halo planes and the
all-gather of the dot-product partials.  Tolerance: north_star's 1e-8 relative
L2 and iteration counts within +-1 of the oracle (reference algorithm).
"""

import numpy as np
import pytest

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


def _pair(case, n, m0):
    pkg = _pkg()
    if case == "smooth":
        ps, os_ = pkg.smooth_affine(6), op.smooth_affine(6)
    else:
        ps, os_ = pkg.thermal_block(case), op.thermal_block(case)
    levels = int(np.log2(n // m0)) + 1
    return pkg.ParametricProblem(ps, levels=levels, m0=m0), op.OracleProblem(os_, n, m0), os_


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _oracle(oprob, mu, x0=None, delta=1e-10, l_max=60):
    A, f = oprob.operator(mu), oprob.rhs()
    x0 = np.zeros_like(f) if x0 is None else x0
    return so.mgcg_solve(A, f, x0, so.mg_context_for(oprob, mu), delta=delta, l_max=l_max)


@pytest.mark.parametrize("case,n,m0,nslabs", [
    ((2, 2, 2), 32, 4, 1), ((2, 2, 2), 32, 4, 2), ((2, 2, 2), 32, 4, 4),
    ((2, 2, 2), 64, 4, 2),   # two distributed coarse levels (32, 16)
    ((2, 2, 2), 64, 4, 4),   # distributed 32-level, replicated below
    ((2, 2, 1), 64, 4, 8),   # 8 planes per slab, everything coarser replicated
    ("smooth", 32, 4, 2),    # 14 z-groups: 27-coefficient coarse kernel
])
def test_slab_mgcg_matches_oracle(case, n, m0, nslabs):
    pkg = _pkg()
    prob, oprob, ospec = _pair(case, n, m0)
    mu = op.sample_mus(ospec, 1, seed=40 + nslabs)[0]
    delta = 1e-10
    x, rep = pkg.slab_mgcg_solve(prob, mu[None], nslabs=nslabs, delta=delta, l_max=60)
    xr, rr = _oracle(oprob, mu, delta=delta)
    got = pkg.from_padded(x, n, 1)[0]
    assert rep.converged and rep.true_residual <= delta
    assert abs(rep.iterations - rr.iterations) <= 1, (rep.iterations, rr.iterations)
    assert _rel(got, xr) <= 1e-8, _rel(got, xr)
    k = min(len(rep.history), len(rr.history), 6)
    np.testing.assert_allclose(rep.history[:k], rr.history[:k], rtol=1e-7)


def test_slab_counts_independent_of_decomposition():
    """Same instance on 1, 2, 4, 8 slabs: identical iteration counts, solutions to 1e-12."""
    pkg = _pkg()
    prob, _, ospec = _pair((2, 2, 2), 64, 4)
    mu = op.sample_mus(ospec, 1, seed=7)
    ref = None
    for ns in (1, 2, 4, 8):
        x, rep = pkg.slab_mgcg_solve(prob, mu, nslabs=ns, delta=1e-11)
        v = pkg.from_padded(x, 64, 1)[0]
        if ref is None:
            ref, it = v, rep.iterations
        else:
            assert rep.iterations == it
            assert _rel(v, ref) <= 1e-12


def test_slab_matches_batched_path():
    pkg = _pkg()
    prob, _, ospec = _pair((2, 2, 1), 64, 4)
    mu = op.sample_mus(ospec, 1, seed=3)
    ctx = pkg.mg_context_for(prob, mu)
    xb, rb = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    xs, rs = pkg.slab_mgcg_solve(prob, mu, nslabs=4, delta=1e-10)
    assert rs.iterations == rb[0].iterations
    assert _rel(pkg.from_padded(xs, 64, 1)[0], pkg.from_padded(xb, 64, 1)[0]) <= 1e-12


def test_slab_prolonged_warm_start():
    """x0 = P e_c (a coarse-grid solution prolonged, as configs[4]'s RB warm start)."""
    pkg = _pkg()
    prob, oprob, ospec = _pair((2, 2, 2), 64, 4)
    cprob, coprob, _ = _pair((2, 2, 2), 32, 4)
    mu = op.sample_mus(ospec, 1, seed=5)
    xc, _ = _oracle(coprob, mu[0], delta=1e-6)
    ec = pkg.to_padded(xc, 32)
    s = pkg.SlabSolver(prob, nslabs=2)
    s.setup(mu)
    s.load("f", prob.rhs())
    s.prolong_x(ec)
    x0 = torch.zeros(pkg.padded_len(64, 1), dtype=torch.float64, device="cuda")
    s.store(x0)
    P = op.prolongation_full(32)
    full = np.zeros(33 ** 3)
    m = 31
    full.reshape(33, 33, 33)[1:32, 1:32, 1:32] = xc.reshape(m, m, m)
    want = (P @ full).reshape(65, 65, 65)[1:64, 1:64, 1:64].ravel()
    assert _rel(pkg.from_padded(x0, 64, 1)[0], want) <= 1e-14
    rep = s.solve(delta=1e-10)
    xr, rr = _oracle(oprob, mu[0], x0=want, delta=1e-10)
    xs = torch.zeros_like(x0)
    s.store(xs)
    assert abs(rep.iterations - rr.iterations) <= 1
    assert _rel(pkg.from_padded(xs, 64, 1)[0], xr) <= 1e-8


def test_slab_edge_cases():
    pkg = _pkg()
    prob, _, ospec = _pair((2, 1, 1), 32, 4)
    mu = op.sample_mus(ospec, 1, seed=9)
    s = pkg.SlabSolver(prob, nslabs=2).setup(mu)
    s.load("f", prob.rhs())
    s.load("x", prob.zeros(1))
    rep = s.solve(delta=1e-10, l_max=0)
    assert rep.iterations == 0 and rep.history[0] == pytest.approx(1.0)
    rep = s.solve(delta=1e-30, l_max=3)
    assert rep.iterations == 3 and not rep.converged
    s.load("f", prob.zeros(1))
    s.load("x", prob.zeros(1))
    rep = s.solve(delta=1e-12)
    assert rep.absolute_norms and rep.iterations == 0
    with pytest.raises(ValueError):
        pkg.SlabSolver(prob, nslabs=3)   # planes per slab must be even
    with pytest.raises(ValueError):
        pkg.SlabSolver(prob, nslabs=16)  # fewer than 4 planes per slab


def test_slab_nccl_loopback_transport_is_bitwise_identical():
    """Halo planes and dot partials through NCCL (send/recv to this rank, all-gather)
    give bitwise the device-copy result: the multi-process code path on one GPU."""
    pkg = _pkg()
    prob, _, ospec = _pair((2, 2, 2), 64, 4)
    mu = op.sample_mus(ospec, 1, seed=13)
    xa, ra = pkg.slab_mgcg_solve(prob, mu, nslabs=4, delta=1e-10, transport="copy")
    xb, rb_ = pkg.slab_mgcg_solve(prob, mu, nslabs=4, delta=1e-10, transport="nccl")
    assert rb_.config["transport"] == "nccl"
    assert ra.iterations == rb_.iterations and ra.history == rb_.history
    assert torch.equal(xa, xb)
