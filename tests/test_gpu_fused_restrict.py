"""Finest pre-smoothing residual fused with the x/z passes of the restriction (FM_PREX +
restrict_y_kernel) against the separate kernels: V-cycles to rounding, identical MGCG
iteration counts, on whole-instance CTAs (large batch) and on z-chunked CTAs (small batch:
every chunk recomputes the odd plane below it)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build
    build.build(verbose=False)


def _ctx(pkg, prob, mus, fused):
    old = os.environ.get("RBWS_FUSED_RESTRICT")
    os.environ["RBWS_FUSED_RESTRICT"] = "1" if fused else "0"
    try:
        return pkg.mg_context_for(prob, mus)
    finally:
        if old is None:
            del os.environ["RBWS_FUSED_RESTRICT"]
        else:
            os.environ["RBWS_FUSED_RESTRICT"] = old


@pytest.mark.parametrize("count", [64, 4])
def test_fused_restriction_matches_separate_kernels(count):
    import paper_2311_13862_b200 as pkg
    from paper_2311_13862_b200 import _native
    spec = pkg.thermal_block((2, 2, 2))
    prob = pkg.ParametricProblem(spec, levels=5, m0=4)   # 64^3
    mus = pkg.sample_mus(spec, count, seed=31)
    n = prob.n
    b = pkg.to_padded(np.random.default_rng(5).standard_normal((count, (n - 1) ** 3)), n)
    out = {}
    for fused in (True, False):
        ctx = _ctx(pkg, prob, mus, fused)
        v = pkg.from_padded(pkg.mg_vcycle(b, ctx), n, count)
        assert bool(_native.load().rbws_batch_fused_restrict(ctx.handle)) == fused
        x, reps = pkg.mgcg_solve(None, None, None, ctx, delta=1e-10, l_max=60)
        out[fused] = (v, pkg.from_padded(x, n, count), [r.iterations for r in reps])
    (v1, x1, it1), (v0, x0, it0) = out[True], out[False]
    assert np.linalg.norm(v1 - v0) <= 1e-13 * np.linalg.norm(v0)
    assert it1 == it0
    assert np.linalg.norm(x1 - x0) <= 1e-10 * np.linalg.norm(x0)
