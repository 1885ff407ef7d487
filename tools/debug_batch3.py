import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as pkg
from paper_2311_13862_b200 import _native
n = 64; B = int(sys.argv[1])
spec = pkg.thermal_block((2, 2, 1))
prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
mus = pkg.sample_mus(spec, B, seed=2000)
ctx = pkg.mg_context_for(prob, mus)
ctx1 = pkg.MgContext(prob, 1)
for lvl in range(1, prob.levels):
    nl = prob.cells[lvl]
    x = torch.randn(pkg.padded_len(nl, B), dtype=torch.float64, device='cuda')
    blk = x[: B * nl**3].view(B, nl, nl, nl); blk[:, 0] = 0; blk[:, :, 0] = 0; blk[:, :, :, 0] = 0
    x[B * nl**3:] = 0
    b = x * 0.5 + 1.0
    blk = b[: B * nl**3].view(B, nl, nl, nl); blk[:, 0] = 0; blk[:, :, 0] = 0; blk[:, :, :, 0] = 0
    b[B * nl**3:] = 0
    y = torch.zeros_like(x)
    _native.call("rbws_jacobi_sweep", ctx.handle, lvl, x.data_ptr(), b.data_ptr(), y.data_ptr(), 0)
    fin = torch.isfinite(y[: B * nl**3].view(B, -1)).all(dim=1).cpu().numpy()
    print("jacobi level", lvl, "finite", fin.sum(), "/", B, np.flatnonzero(~fin)[:8], flush=True)
b = torch.randn(pkg.padded_len(n, B), dtype=torch.float64, device='cuda')
blk = b[: B * n**3].view(B, n, n, n); blk[:, 0] = 0; blk[:, :, 0] = 0; blk[:, :, :, 0] = 0; b[B*n**3:] = 0
o = pkg.mg_vcycle(b, ctx)
for m in (0, 1, 500, B - 1):
    ctx1.setup(mus[m:m+1])
    b1 = torch.zeros(pkg.padded_len(n, 1), dtype=torch.float64, device='cuda'); b1[: n**3] = b[m*n**3:(m+1)*n**3]
    o1 = pkg.mg_vcycle(b1, ctx1)
    print("vcycle", m, float((o1[: n**3] - o[m*n**3:(m+1)*n**3]).abs().max()), flush=True)
