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
x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
for k in range(14):
    b, x, Ax = pool[k]
    ig.form_guess(b, x0)
    ig.update(x, Ax)
torch.cuda.synchronize()
L = lib()
L.ig_debug_trace_read.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * (1024 * 8))()
assert L.ig_debug_trace_read(buf, 1024 * 8) == 0
t = np.array(buf[:148 * 8], dtype=np.float64).reshape(148, 8)[:, :7]
t0 = t[:, 0].min()
t = (t - t0) / 1e3  # us
names = ["start", "pass1 done", "barrier1 out", "reduce1 done", "pass2 done", "barrier2 out", "pass3 done"]
for j, nm in enumerate(names):
    print(f"{nm:14s} min {t[:, j].min():8.1f} med {np.median(t[:, j]):8.1f} max {t[:, j].max():8.1f} us")
