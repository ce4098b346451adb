"""Small end-to-end run for compute-sanitizer: every kernel family and schedule once, checked vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import ProjQR, ProjClassic, ExtrapLS, ExtrapSparse
from paper_2009_10863_b200 import InitialGuess
from workloads import Grid, manufactured_step

g = Grid(23, 2)  # N = 529: odd, ragged
for M in (1, 3, 8, 12, 17, 30):
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
# multi-trip size (360,000 DOFs): the dynamically claimed pass-3 tail, the Givens planner's
# handed-off trips, the launch-epoch barrier counters; batch and host-buffer batch calls
from paper_2009_10863_b200 import ig_form_guess_batch, ig_form_guess_batch_host, ig_update_batch, ig_update_batch_host

gb = Grid(600, 2)
ora_q, ora_e = ProjQR(gb.N, 8), ExtrapLS(gb.N, 8, 3)
hq, he = InitialGuess(gb.N, "proj_qr", 8), InitialGuess(gb.N, "extrap_ls", 8, 3)
worst = 0.0
for n in range(12):
    b, x, Ax = (t.numpy() for t in manufactured_step(gb, n, dt=1e-2))
    if n % 2 == 0:
        x0s = [torch.zeros(gb.N, dtype=torch.float64, device="cuda") for _ in range(2)]
        ig_form_guess_batch([hq, he], [torch.from_numpy(b).cuda(), None], x0s)
        got = [t.cpu().numpy() for t in x0s]
    else:
        x0s = [torch.zeros(gb.N, dtype=torch.float64).pin_memory() for _ in range(2)]
        ig_form_guess_batch_host([hq, he], [torch.from_numpy(b).pin_memory(), None], x0s)
        got = [t.numpy() for t in x0s]
    for o, gval in zip((ora_q, ora_e), got):
        ref = o.form_guess(b, np.zeros(gb.N))
        worst = max(worst, np.linalg.norm(gval - ref) / max(np.linalg.norm(ref), 1e-300))
    ora_q.update(x, Ax)
    ora_e.update(x)
    if n % 2 == 0:
        ig_update_batch([hq, he], [torch.from_numpy(x).cuda()] * 2, [torch.from_numpy(Ax).cuda(), None])
    else:
        ig_update_batch_host([hq, he], [torch.from_numpy(x).pin_memory()] * 2, [torch.from_numpy(Ax).pin_memory(), None])
hq.close()
he.close()
print("multi-trip batch", f"{worst:.1e}", flush=True)
assert worst < 1e-11
# device-resident extrapolation windows + one captured multi-field step (ring kernels, graph replay)
from paper_2009_10863_b200 import CapturedStep

s = torch.cuda.Stream()
specs = [("proj_qr", 6, 0), ("extrap_ls", 6, 2), ("extrap_sparse", 8, 2)]
oras = [ProjQR(g.N, 6), ExtrapLS(g.N, 6, 2), ExtrapSparse(g.N, 8, 2)]
hs = [InitialGuess(g.N, m, M, p, stream=s) for m, M, p in specs]
for h in hs[1:]:
    h.set_device_ring(True)
bufs = [[torch.zeros(g.N, dtype=torch.float64, device="cuda") for _ in specs] for _ in range(4)]
torch.cuda.synchronize()
with CapturedStep(s) as step:
    ig_form_guess_batch(hs, bufs[0], bufs[1])
    ig_update_batch(hs, bufs[2], bufs[3])
worst = 0.0
for n in range(10):
    b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
    with torch.cuda.stream(s):
        for f in range(len(specs)):
            bufs[0][f].copy_(torch.from_numpy(b))
            bufs[1][f].zero_()
            bufs[2][f].copy_(torch.from_numpy(x))
            bufs[3][f].copy_(torch.from_numpy(Ax))
    step.replay()
    s.synchronize()
    for f, o in enumerate(oras):
        ref = o.form_guess(b, np.zeros(g.N))
        worst = max(worst, np.linalg.norm(bufs[1][f].cpu().numpy() - ref) / max(np.linalg.norm(ref), 1e-300))
        o.update(x, Ax)
step.close()
for h in hs:
    h.close()
print("captured step", f"{worst:.1e}", flush=True)
assert worst < 1e-11
print("SANITIZE RUN OK")
