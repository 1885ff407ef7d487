"""Probe the end-to-end pipeline: sub-batch size vs copy overlap (development tool)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as rb
n, B = 64, 1024
spec = rb.thermal_block((2, 2, 1))
prob = rb.ParametricProblem(spec, levels=rb.problems.levels_for(n, 4), m0=4)
train = rb.sample_mus(spec, 1024, seed=1000)
test = rb.sample_mus(spec, B, seed=2000)
hf = rb.HighFidelitySolver(prob, delta=1e-14, l_max=100)
model = rb.l1roc_offline(train, 20, hf, prob, seed=0, on_degenerate="stop")
del hf
torch.cuda.empty_cache()
method = rb.MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=model.dim)
hbuf = torch.empty(B * n ** 3, dtype=torch.float64, pin_memory=True)
def timeit(fn, reps=2):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3
x = torch.empty(rb.padded_len(n, B), dtype=torch.float64, device='cuda')
print("d2h 2.1GB copy ms", timeit(lambda: hbuf.copy_(x[:B * n ** 3], non_blocking=True)))
for sub in (512, 256):
    pipe = rb.HostPipeline(prob, method, model, sub_batch=sub)
    print(sub, "pipeline ms", timeit(lambda: pipe.solve(test, hbuf)))
    ctx = pipe.ctx[0]; f = prob.rhs(); xb = pipe.x[0]
    def nocopy():
        for c0 in range(0, B, sub):
            rb.mg_context_for(prob, test[c0:c0 + sub], ctx=ctx)
            rb.rbi_pcg_solve(rb.BatchOperator(ctx), f, method, mg_ctx=ctx, l1roc_model=model, x0_out=xb)
    print(sub, "no-copy ms", timeit(nocopy))
    del pipe, ctx, xb
    torch.cuda.empty_cache()
