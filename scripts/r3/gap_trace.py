"""Kernel-boundary gaps of back-to-back QR calls (form -> update -> form) from a -DIG_TRACE=1 build:
last CTA exit of one persistent kernel -> first CTA begin / pdl_wait out of the next (globaltimer).
TRACE_N (n^3 DOFs), TRACE_M; IG_LAUNCH selects cooperative (default) or plain launches."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2009_10863_b200 import InitialGuess
from paper_2009_10863_b200._lib import lib
from workloads.gen import manufactured_step_slab
n = int(os.environ.get("TRACE_N", "100")); M = int(os.environ.get("TRACE_M", "30")); N = n ** 3
S = M + 4
pool = [manufactured_step_slab(n, n, 0, 1, k, device="cuda") for k in range(S)]
ig = InitialGuess(N, "proj_qr", M)
x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
L = lib()
L.ig_debug_trace_read.argtypes = [C.c_void_p, C.c_int]
L.ig_debug_trace_read_form.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * (1024 * 16))()
def rows(read):
    assert read(buf, 1024 * 16) == 0
    return np.array(buf[:148 * 16], dtype=np.float64).reshape(148, 16)
res = []
for rep in range(3):
    for k in range(S):
        b, x, Ax = pool[k]
        ig.form_guess(b, x0)
        ig.update(x, Ax)
    b, x, Ax = pool[0]
    ig.form_guess(b, x0)      # form(S-1) ... update(S-1) traced below
    ig.update(x, Ax)
    torch.cuda.synchronize()
    f1 = rows(L.ig_debug_trace_read_form); u = rows(L.ig_debug_trace_read)
    ig.form_guess(b, x0)      # the form right after the traced update
    torch.cuda.synchronize()
    f2 = rows(L.ig_debug_trace_read_form)
    # form: slot 8 begin, 0 pdl out, 7 exit; update: 8 begin, 0 pdl out, 7 exit (planner row 147: 11 done)
    fend = f1[:, 7].max(); ubeg = u[:, 8].min(); upd = u[:, 0].min(); uend = max(u[:147, 7].max(), u[147, 11])
    f2beg = f2[:, 8].min(); f2pd = f2[:, 0].min()
    r = dict(form_us=(fend - f1[:, 8].min()) / 1e3, upd_us=(uend - ubeg) / 1e3,
             gap_form_to_update_begin=(ubeg - fend) / 1e3, gap_form_to_update_pdlout=(upd - fend) / 1e3,
             gap_update_to_form_begin=(f2beg - uend) / 1e3, gap_update_to_form_pdlout=(f2pd - uend) / 1e3,
             upd_begin_spread=(u[:147, 8].max() - ubeg) / 1e3, form_begin_spread=(f2[:, 8].max() - f2beg) / 1e3)
    res.append(r)
print(f"N={N} M={M} IG_LAUNCH={os.environ.get('IG_LAUNCH', 'default')}")
for kk in res[0]:
    print(f"  {kk:28s} " + " ".join(f"{r[kk]:8.2f}" for r in res))
