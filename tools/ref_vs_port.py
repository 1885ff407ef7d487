"""Build-container check (needs /root/reference; never on the GPU box): the unmodified
reference package's RBI-MGCG per parameter vs the oracle port that bench.py's reference arm
times, on the configs[1] problem (64^3 thermal 2x2x1, FD terms through the reference's own
ParametricProblem via make_golden's assembly hooks), same model, same parameters, one core.

    python tools/ref_vs_port.py [--n 64] [--count 6]
"""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests" / "golden"))
import numpy as np
from threadpoolctl import threadpool_limits

import make_golden as mg
from oracle import problems as op
from oracle import solvers as so

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--count", type=int, default=6)
args = ap.parse_args()
rbws = mg._import_reference()
from rbws.multigrid import mg_context_for
from rbws.rb import L1rocModel
from rbws.warmstart import MethodConfig, rbi_pcg_solve

spec = op.thermal_block((2, 2, 1))
with threadpool_limits(1):
    t0 = time.perf_counter()
    rprob = mg.reference_problem(rbws, spec, args.n, 4)
    oprob = op.OracleProblem(spec, args.n, 4)
    print(f"assembly (reference + oracle) {time.perf_counter() - t0:.1f}s", flush=True)
    train = op.sample_mus(spec, 64, seed=1000)

    def hf(mu):
        A, f = oprob.operator(mu), oprob.rhs()
        return so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(oprob, mu), 1e-14, 100)[0]

    om = so.l1roc_offline(list(train), 10, hf, oprob.operator, oprob.operator_rows, oprob.rhs,
                          seed=0, on_degenerate="stop")
    rm = L1rocModel(om.basis, om.transform, om.collocation, om.solution_points,
                    om.residual_points, train[om.chosen], om.indicator_history, om.saturated)
    test = op.sample_mus(spec, args.count, seed=2000)
    cfg = MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=om.dim)
    tr, tp, it_r, it_p = 0.0, 0.0, [], []
    for mu in test:
        A, f = rprob.operator(mu), rprob.rhs(mu)          # assembly outside the timing
        t1 = time.perf_counter()
        _, rep = rbi_pcg_solve(A, f, cfg, mg_ctx=mg_context_for(rprob, mu), l1roc_model=rm)
        tr += time.perf_counter() - t1
        it_r.append(rep.iterations)
        t1 = time.perf_counter()
        _, rep2 = so.rbi_mgcg_solve(oprob, mu, om, delta=1e-10, l_max=60)
        tp += time.perf_counter() - t1
        it_p.append(rep2.iterations)
    print(f"reference package: {args.count / tr:.3f} solves/s, iterations {it_r}")
    print(f"oracle port:       {args.count / tp:.3f} solves/s, iterations {it_p}")
