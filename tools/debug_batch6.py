import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as pkg
spec = pkg.thermal_block((2, 2, 1))
n = int(sys.argv[1]); nu = int(sys.argv[2])
prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
for B in [int(v) for v in sys.argv[3].split(',')]:
    mus = pkg.sample_mus(spec, B, seed=2000)
    ctx = pkg.mg_context_for(prob, mus, nu=nu)
    b = torch.randn(pkg.padded_len(n, B), dtype=torch.float64, device='cuda')
    blk = b[: B * n**3].view(B, n, n, n); blk[:, 0] = 0; blk[:, :, 0] = 0; blk[:, :, :, 0] = 0; b[B*n**3:] = 0
    o = pkg.mg_vcycle(b, ctx)
    fin = torch.isfinite(o[: B * n**3].view(B, -1)).all(dim=1).cpu().numpy()
    print("n", n, "nu", nu, "B", B, "finite", fin.sum(), np.flatnonzero(~fin)[:6], flush=True)
