"""Dump the QR(M) guesses of a short seeded sequence (for bitwise A/B of library variants):
python scripts/r3/dump_guesses.py N M out.npy"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import hashlib, numpy as np, torch
from paper_2009_10863_b200 import InitialGuess
from workloads.gen import manufactured_step_slab
N, M, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
n = round(N ** (1 / 3)); N = n ** 3
ig = InitialGuess(N, "proj_qr", M)
x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
h = hashlib.sha256()
for k in range(M + 6):
    b, x, Ax = manufactured_step_slab(n, n, 0, 1, k, device="cuda")
    ig.form_guess(b, x0)
    h.update(x0.cpu().numpy().tobytes())
    ig.update(x, Ax)
print(N, M, h.hexdigest(), ig.stats()["d"])
