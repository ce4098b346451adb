"""Per-phase timing of k_update_fused from a -DIG_TRACE=1 build (globaltimer stamps per CTA)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2009_10863_b200 import InitialGuess
from paper_2009_10863_b200._lib import lib
from workloads.gen import manufactured_step_slab
n, M = 128, 8
N = n ** 3
pool = [manufactured_step_slab(n, n, 0, 1, k, device="cuda") for k in range(14)]
ig = InitialGuess(N, "proj_qr", M)
he = InitialGuess(N, "extrap_ls", M, 3)
x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
x0e = torch.zeros(N, dtype=torch.float64, device="cuda")
for k in range(14):  # the bench step: QR form, QR update (traced), EXTRAP form, EXTRAP push
    b, x, Ax = pool[k]
    ig.form_guess(b, x0)
    ig.update(x, Ax)
    if k < 13:
        he.form_guess(None, x0e)
        he.update(x)
torch.cuda.synchronize()
L = lib()
L.ig_debug_trace_read.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * (1024 * 12))()
assert L.ig_debug_trace_read(buf, 1024 * 12) == 0
raw = np.array(buf[:148 * 12], dtype=np.float64).reshape(148, 12)
t = raw[:, [8, 0, 1, 2, 3, 4, 5, 6, 7]]
last = int(np.argmax(raw[:, 7]))  # the CTA that ran the epilogue
t0 = t[:, 0].min()
t = (t - t0) / 1e3  # us
names = ["CTA begin", "pdl_wait out", "pass1 done", "barrier1 out", "reduce1 done", "pass2 done", "barrier2 out", "pass3 done",
         "exit (last: epilogue done)"]
for j, nm in enumerate(names):
    print(f"{nm:14s} min {t[:, j].min():8.1f} med {np.median(t[:, j]):8.1f} max {t[:, j].max():8.1f} us")
e = (raw[last, [6, 9, 7]] - t0) / 1e3
print(f"epilogue CTA {last}: pass3 done {e[0]:.1f}, after grid_exit {e[1]:.1f}, done {e[2]:.1f} us")
pl = (raw[0, [10, 11]] - t0) / 1e3
print(f"R update + Givens plan (CTA 0 warp 0, during pass 3): {pl[0]:.1f} -> {pl[1]:.1f} us ({pl[1] - pl[0]:.1f} us)")
