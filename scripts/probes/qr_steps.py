"""Run QR(M) form+update steps on random vectors (N, M from argv) -- a target for ncu captures."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2009_10863_b200 import InitialGuess  # noqa: E402

N, M, S = int(float(sys.argv[1])), int(sys.argv[2]), int(sys.argv[3])
pool = M + 2
g = torch.Generator(device="cuda").manual_seed(10863 + M)
X = [torch.randn(N, dtype=torch.float64, device="cuda", generator=g) for _ in range(pool)]
AX = [torch.randn(N, dtype=torch.float64, device="cuda", generator=g) for _ in range(pool)]
x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
h = InitialGuess(N, "proj_qr", M)
for k in range(S):
    h.form_guess(AX[(k + 1) % pool], x0)
    h.update(X[k % pool], AX[k % pool])
torch.cuda.synchronize()
print("d", h.d)
