"""RBI-MGCG (L1ROC warm start + MGCG) on the reference's assembled problems through the
batched product API, and HostPipeline for them, against the reference's own outputs
(golden_experiment.npz: the unmodified run_experiment on example-1 / example-2, LU greedy).

example-2 keeps its free x = 1 face in the full-node layout (fem_fn.py): the greedy's
DEIM points, term projections (A_q W)[X, :] and warm starts run on (c+1)^3-node vectors
(rb.FullNodeLayout); reference rb.py:190-293, warmstart.py:88-117."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_experiment.npz"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build
    build.build(verbose=False)


def _pkg():
    import paper_2311_13862_b200 as pkg
    return pkg


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _golden_rbi(g, k, N, delta):
    keys = list(g[f"{k}_keys"])
    idx = [i for i, key in enumerate(keys) if key == f"rbi-mgcg|{N}|{delta!r}"]
    return np.array([g[f"{k}_x{i}"] for i in idx]), [int(g[f"{k}_it{i}"]) for i in idx]


@pytest.mark.parametrize("tag,pid,N,delta", [("ex2", "example-2", 4, 1e-10),
                                             ("ex1", "example-1", 6, 1e-12)])
def test_batched_rbi_matches_reference_experiment(tag, pid, N, delta):
    pkg = _pkg()
    g = np.load(GOLDEN)
    k = f"exp_{tag}"
    prob = pkg.ParametricProblem(pkg.get_problem(pid), levels=3, m0=4)
    hf = pkg.HighFidelitySolver(prob, delta=1e-14, l_max=200)
    model = pkg.l1roc_offline(g[f"{k}_train"], N, hf, prob, seed=0)
    np.testing.assert_array_equal(model.chosen_mus, g[f"{k}_chosen"][:N])
    np.testing.assert_allclose(model.indicator_history, g[f"{k}_hist"][:N], rtol=1e-6)
    B = model.basis_numpy()
    assert B.shape == (prob.n_free, N)
    test = g[f"{k}_test"]
    ctx = pkg.mg_context_for(prob, test)
    f = prob.rhs(test)
    cfg = pkg.MethodConfig("rbi-mgcg", delta=delta, l_max=60, N=N)
    x, reps = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), f, cfg, mg_ctx=ctx, l1roc_model=model)
    xr, itr = _golden_rbi(g, k, N, delta)
    if tag == "ex2":
        got = prob.from_full(x)
    else:
        got = pkg.from_padded(x, prob.n, len(test))
    for m in range(len(test)):
        assert abs(reps[m].iterations - itr[m]) <= 1, (m, reps[m].iterations, itr[m])
        assert _rel(got[m], xr[m]) <= 1e-8, (m, _rel(got[m], xr[m]))


@pytest.mark.parametrize("pid", ["example-2", "example-1"])
def test_host_pipeline_assembled_matches_device_solve(pid):
    """HostPipeline on assembled problems (per-parameter rhs uploaded inside the call)
    gives the device-resident batched solve's solutions and iteration counts."""
    pkg = _pkg()
    spec = pkg.get_problem(pid)
    prob = pkg.ParametricProblem(spec, levels=3, m0=4)
    train = np.array(pkg.lhs_sample(spec.p, 12, spec.bounds, seed=1))
    model = pkg.l1roc_offline(train, 4, pkg.HighFidelitySolver(prob), prob, seed=0)
    mus = np.array(pkg.lhs_sample(spec.p, 10, spec.bounds, seed=2))
    cfg = pkg.MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=model.dim)
    pipe = pkg.HostPipeline(prob, cfg, model, sub_batch=4)
    buf = torch.empty(len(mus) * pipe.stride, dtype=torch.float64, pin_memory=True)
    reps = pipe.solve(mus, buf)
    torch.cuda.synchronize()
    ctx = pkg.mg_context_for(prob, mus)
    x, rr = pkg.rbi_pcg_solve(pkg.BatchOperator(ctx), prob.rhs(mus), cfg, mg_ctx=ctx,
                              l1roc_model=model)
    want = x.reshape(-1)[: len(mus) * pipe.stride].cpu().numpy()
    assert _rel(buf.numpy(), want) <= 1e-13
    assert [r.iterations for r in reps] == [r.iterations for r in rr]
