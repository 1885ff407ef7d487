"""rbi-msrbcg on the GPU (POD bases, iteration-indexed MSRB preconditioner) against the
reference's own golden vectors (tests/golden/golden_msrb.npz)."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_msrb.npz"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build
    build.build(verbose=False)


@pytest.fixture(scope="module")
def gm():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="module")
def trained(gm):
    import paper_2311_13862_b200 as pkg
    prob = pkg.ParametricProblem(pkg.thermal_block((2, 2, 1)), levels=3, m0=4)
    N, K = (int(v) for v in gm["msrb_tb221_n16_NK"])
    hf = pkg.HighFidelitySolver(prob, delta=1e-14, l_max=100)
    hier = pkg.msrb_train(gm["msrb_tb221_n16_train"], N, K, hf, prob)
    return pkg, prob, hier


def _free(pkg, rows, n):
    """(N, n^3) padded rows -> (M, N) free-DoF columns (reference ordering)."""
    N = rows.shape[0]
    buf = torch.zeros(pkg.padded_len(n, N), dtype=torch.float64, device="cuda")
    buf[: N * n ** 3] = rows.reshape(-1)
    return pkg.from_padded(buf, n, N).T


def _span_err(A, B):
    return np.linalg.norm(A - B @ (B.T @ A), 2)


def test_msrb_bases_match_reference(gm, trained):
    pkg, prob, hier = trained
    np.testing.assert_allclose(hier.init_basis.eigenvalues[:10],
                               gm["msrb_tb221_n16_init_eig"][:10], rtol=1e-8)
    W0 = _free(pkg, hier.init_basis.basis, 16)
    assert W0.shape == gm["msrb_tb221_n16_init"].shape
    assert _span_err(W0, gm["msrb_tb221_n16_init"]) <= 1e-7
    assert len(hier.bases) == int(gm["msrb_tb221_n16_NK"][1])
    for k, W in enumerate(hier.bases):
        assert _span_err(_free(pkg, W, 16), gm[f"msrb_tb221_n16_basis{k}"]) <= 1e-5, k


def test_rbi_msrbcg_matches_reference(gm, trained):
    pkg, prob, hier = trained
    test = gm["msrb_tb221_n16_test"]
    ctx = pkg.mg_context_for(prob, test)
    N, K = (int(v) for v in gm["msrb_tb221_n16_NK"])
    cfg = pkg.MethodConfig("rbi-msrbcg", delta=1e-10, l_max=60, N=N, K_max=K)
    x, reps = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), prob.rhs(), cfg, mg_ctx=ctx,
                                msrb_hier=hier)
    got = pkg.from_padded(x, 16, len(test))
    for m in range(len(test)):
        assert abs(reps[m].iterations - int(gm["msrb_tb221_n16_iters"][m])) <= 1
        h = gm["msrb_tb221_n16_hist"][m]
        np.testing.assert_allclose(reps[m].history[:8], h[:8], rtol=1e-5)
        ref = gm["msrb_tb221_n16_x"][m]
        assert np.linalg.norm(got[m] - ref) <= 1e-5 * np.linalg.norm(ref)
        assert reps[m].config["preconditioner"] == "msrb"


def test_basis_dot_kernel_matches_matmul():
    """rbws_basis_dot (W^T v of the MSRB correction) against a plain fp64 torch matmul,
    shared (stride 0) and per-instance right-hand sides, N above one 8-vector chunk."""
    from paper_2311_13862_b200 import _native
    g = torch.Generator(device="cuda").manual_seed(3)
    n3, count, N = 33 * 33 * 33 + 17, 13, 11
    W = torch.randn(N, n3, generator=g, device="cuda", dtype=torch.float64)
    v = torch.randn(count, n3, generator=g, device="cuda", dtype=torch.float64)
    for vv, stride in ((v, n3), (v[:1].expand(count, n3), 0)):
        out = torch.empty(count, N, dtype=torch.float64, device="cuda")
        _native.call("rbws_basis_dot", n3, count, W.data_ptr(), n3, N, vv.data_ptr(), stride,
                     out.data_ptr(), 0)
        ref = vv @ W.T
        assert torch.allclose(out, ref, rtol=1e-12, atol=1e-10)
        out2 = torch.empty_like(out)
        _native.call("rbws_basis_dot", n3, count, W.data_ptr(), n3, N, vv.data_ptr(), stride,
                     out2.data_ptr(), 0)
        assert torch.equal(out, out2)  # fixed-order partial sums


# ---- rbi-msrbcg on the reference's assembled problem example-1 (stored-coefficient hierarchy,
# per-parameter right-hand sides): goldens from the unmodified reference,
# make_golden.py --msrb-fem
GOLDEN_FEM = Path(__file__).resolve().parent / "golden" / "golden_msrb_fem.npz"


@pytest.fixture(scope="module")
def trained_fem():
    import paper_2311_13862_b200 as pkg
    g = dict(np.load(GOLDEN_FEM))
    prob = pkg.ParametricProblem(pkg.get_problem("example-1"), levels=3, m0=4)
    N, K = (int(v) for v in g["msrb_ex1_n16_NK"])
    hf = pkg.HighFidelitySolver(prob, delta=1e-14, l_max=100)
    hier = pkg.msrb_train(g["msrb_ex1_n16_train"], N, K, hf, prob)
    return pkg, prob, hier, g


def test_msrb_example1_bases_match_reference(trained_fem):
    pkg, prob, hier, g = trained_fem
    np.testing.assert_allclose(hier.init_basis.eigenvalues[:6], g["msrb_ex1_n16_init_eig"][:6],
                               rtol=1e-8)
    assert _span_err(_free(pkg, hier.init_basis.basis, 16), g["msrb_ex1_n16_init"]) <= 1e-7
    assert len(hier.bases) == int(g["msrb_ex1_n16_NK"][1])
    for k, W in enumerate(hier.bases):
        assert _span_err(_free(pkg, W, 16), g[f"msrb_ex1_n16_basis{k}"]) <= 1e-5, k


def test_rbi_msrbcg_example1_matches_reference(trained_fem):
    pkg, prob, hier, g = trained_fem
    test = g["msrb_ex1_n16_test"]
    ctx = pkg.mg_context_for(prob, test)
    N, K = (int(v) for v in g["msrb_ex1_n16_NK"])
    cfg = pkg.MethodConfig("rbi-msrbcg", delta=1e-10, l_max=60, N=N, K_max=K)
    x, reps = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), prob.rhs(test), cfg, mg_ctx=ctx,
                                msrb_hier=hier)
    got = pkg.from_padded(x, 16, len(test))
    for m in range(len(test)):
        assert abs(reps[m].iterations - int(g["msrb_ex1_n16_iters"][m])) <= 1
        np.testing.assert_allclose(reps[m].history[:8], g["msrb_ex1_n16_hist"][m][:8], rtol=1e-5)
        ref = g["msrb_ex1_n16_x"][m]
        assert np.linalg.norm(got[m] - ref) <= 1e-8 * np.linalg.norm(ref)
        assert reps[m].converged


def test_msrbcg_native_edge_cases(trained):
    """The native loop's argument checks and degenerate runs: l_max = 0 (initial guess only),
    no bases (sweep-only preconditioner), a converged initial guess."""
    pkg, prob, hier = trained
    from paper_2311_13862_b200.msrb import MsrbHierarchy, rbi_msrbcg_solve
    mus = pkg.sample_mus(prob.spec, 2, seed=4)
    x0, r0 = rbi_msrbcg_solve(prob, mus, hier, delta=1e-10, l_max=0)
    assert all(r.iterations == 0 for r in r0)
    bare = MsrbHierarchy(hier.init_basis, (), hier.N, 0)
    x1, r1 = rbi_msrbcg_solve(prob, mus, bare, delta=1e-6, l_max=200)
    assert all(r.converged for r in r1)
    x2, r2 = rbi_msrbcg_solve(prob, mus, hier, delta=1e-6, l_max=200)
    assert all(r.converged for r in r2)
    with pytest.raises(ValueError):
        rbi_msrbcg_solve(prob, mus, hier, delta=0.0)
