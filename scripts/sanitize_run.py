"""Small end-to-end run for compute-sanitizer: every kernel family and schedule once, checked vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import ProjQR, ProjClassic, ExtrapLS, ExtrapSparse
from paper_2009_10863_b200 import InitialGuess
from workloads import Grid, manufactured_step

g = Grid(23, 2)  # N = 529: odd, ragged
for M in (1, 3, 8, 17, 30):
    for method, ora_cls in (("proj_qr", ProjQR), ("proj_classic", ProjClassic)):
        for fused in (True, False):
            ora, ig = ora_cls(g.N, M), InitialGuess(g.N, method, M, fused=fused)
            worst = 0.0
            for n in range(M + 4):
                b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
                x0 = torch.zeros(g.N, dtype=torch.float64, device="cuda")
                ig.form_guess(torch.from_numpy(b).cuda(), x0)
                ref = ora.form_guess(b, np.zeros(g.N))
                worst = max(worst, np.linalg.norm(x0.cpu().numpy() - ref) / max(np.linalg.norm(ref), 1e-300))
                ora.update(x, Ax)
                ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
            ig.close()
            print(method, M, "fused" if fused else "split", f"{worst:.1e}", flush=True)
            assert worst < 1e-11
for method, cls in (("extrap_ls", ExtrapLS), ("extrap_sparse", ExtrapSparse)):
    for M, p in ((4, 2), (16, 3), (30, 5)):
        ora, ig = cls(g.N, M, p), InitialGuess(g.N, method, M, p)
        for n in range(M + 3):
            b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
            x0 = torch.zeros(g.N, dtype=torch.float64, device="cuda")
            ig.form_guess(None, x0)
            ref = ora.form_guess(b, np.zeros(g.N))
            assert np.linalg.norm(x0.cpu().numpy() - ref) <= 1e-11 * max(np.linalg.norm(ref), 1.0)
            ora.update(x)
            ig.update(torch.from_numpy(x).cuda())
        ig.close()
        print(method, M, p, "ok", flush=True)
print("SANITIZE RUN OK")
