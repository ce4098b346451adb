"""Per-phase timing of k_update_fused and k_form_fused from a -DIG_TRACE=1 build (globaltimer
stamps per CTA, SM id per CTA).  python -m paper_2009_10863_b200.build --trace, then run this."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2009_10863_b200 import InitialGuess
from paper_2009_10863_b200._lib import lib
from workloads.gen import manufactured_step_slab
n = int(os.environ.get("TRACE_N", "128"))  # grid points per direction (n^3 DOFs); default C2
M = int(os.environ.get("TRACE_M", "8"))
N = n ** 3
S = M + 6
pool = [manufactured_step_slab(n, n, 0, 1, k, device="cuda") for k in range(S)]
ig = InitialGuess(N, "proj_qr", M)
he = InitialGuess(N, "extrap_ls", M, min(3, M - 1))
x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
x0e = torch.zeros(N, dtype=torch.float64, device="cuda")
for k in range(S):  # the bench step: QR form, QR update (traced), EXTRAP form, EXTRAP push
    b, x, Ax = pool[k]
    ig.form_guess(b, x0)
    ig.update(x, Ax)
    if k < S - 1:
        he.form_guess(None, x0e)
        he.update(x)
torch.cuda.synchronize()
L = lib()
L.ig_debug_trace_read.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * (1024 * 16))()
assert L.ig_debug_trace_read(buf, 1024 * 16) == 0
allrows = np.array(buf[:148 * 16], dtype=np.float64).reshape(148, 16)
plan_row = allrows[147]  # QR grids: the last CTA is the planner (streams nothing)
raw = allrows[:147]
t = raw[:, [8, 0, 1, 2, 3, 4, 5, 6, 7]]
last = 0  # CTA 0 writes the control block (no exit barrier)
t0 = t[:, 0].min()
t = (t - t0) / 1e3  # us
names = ["CTA begin", "pdl_wait out", "pass1 done", "barrier1 out", "reduce1 done", "pass2 done", "barrier2 out", "pass3 done",
         "exit (last: epilogue done)"]
for j, nm in enumerate(names):
    print(f"{nm:14s} min {t[:, j].min():8.1f} med {np.median(t[:, j]):8.1f} max {t[:, j].max():8.1f} us")
e = (raw[last, [6, 9, 7]] - t0) / 1e3
print(f"CTA 0 (planner + control block): pass3 done {e[0]:.1f}, epilogue start {e[1]:.1f}, done {e[2]:.1f} us")
pl = (plan_row[[8, 10, 14, 13, 11]] - t0) / 1e3
print(f"planner CTA: begin {pl[0]:.1f}, staged R {pl[1]:.1f}, plan prefix done {pl[2]:.1f}, saw barrier 2 {pl[3]:.1f}, "
      f"R + plan suffix done {pl[4]:.1f} us (after barrier 2: {pl[4] - pl[3]:.1f} us)")

# ---- k_form_fused of the same (last) step
L.ig_debug_trace_read_form.argtypes = [C.c_void_p, C.c_int]
assert L.ig_debug_trace_read_form(buf, 1024 * 16) == 0
rf = np.array(buf[:148 * 16], dtype=np.float64).reshape(148, 16)
tf = (rf[:, [8, 0, 1, 2, 3, 4, 7]] - rf[:, 8].min()) / 1e3
print("k_form_fused:")
for j, nm in enumerate(["CTA begin", "pdl_wait out", "pass1 done", "barrier out", "reduce done", "pass2 done", "exit"]):
    print(f"  {nm:14s} min {tf[:, j].min():8.1f} med {np.median(tf[:, j]):8.1f} max {tf[:, j].max():8.1f} us")

# per-SM systematic imbalance? pass-1 duration of the CTA on each SM in both kernels
sm_u = raw[:, 12].astype(int)
sm_f = rf[:, 12].astype(int)
du = {s: (raw[i, 1] - raw[i, 0]) / 1e3 for i, s in enumerate(sm_u)}
df = {s: (rf[i, 1] - rf[i, 0]) / 1e3 for i, s in enumerate(sm_f)}
common = sorted((set(du) & set(df)) - {int(plan_row[12])})
a = np.array([du[s] for s in common]); b = np.array([df[s] for s in common])
print(f"pass-1 duration per SM: update {a.mean():.1f}+-{a.std():.2f} us, form {b.mean():.1f}+-{b.std():.2f} us, "
      f"corr over {len(common)} SMs = {np.corrcoef(a, b)[0, 1]:.2f}")
slow = sorted(common, key=lambda s: -du[s])[:8]
print("slowest SMs (update pass 1):", slow, "form ranks:", [sorted(common, key=lambda s: -df[s]).index(s) for s in slow])
