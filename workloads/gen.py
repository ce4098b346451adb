"""Seeded synthetic workloads (device-agnostic torch fp64; CPU for the oracle, CUDA for bench).

Shapes follow BASELINE.json ``configs`` (SURVEY.md §8(d) "Synthetic inputs"):

* grid: unit interval/square/cube, n points per direction, h = 1/(n+1), interior
  unknowns only, lexicographic order with the LAST axis fastest (so the 3D
  vector is contiguous z-slabs -> contiguous DOF ranges shard by z).
* operator (harness only): A = -Delta_h + sigma I, homogeneous Dirichlet,
  3/5/7-point stencil (1D/2D/3D).  SPD.
* smooth field u(x, t) ("smooth" family, SPEC S:362 style forcing):
      prod_j sin(pi x_j) (1 + 0.3 sin 2 pi t) + exp(-|x - c(t)|^2 / 0.02)
      + sum_{k<K} a_k(t) prod_j sin(q_kj pi x_j),   a_k = cos(omega_k t + phi_k)
  with c(t) translating at speed 0.4, K = 8 modes (3D) / 4 (1D, 2D) drawn once
  from ``numpy.random.default_rng(SEED)``.
* noise: counter-hash xi_n(i) = splitmix64(seed, n, i) mapped exactly to [-1, 1).
* manufactured step n (open loop, no solver needed):
      b_n = A u(t_n),   x_n = u(t_n) + eta xi_n (eta = 1e-8 max|u|, mimics a
      CG-tolerance solve),   Ax_n = A x_n.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

SEED = 10863
_MASK64 = (1 << 64) - 1


def _s64(v: int) -> int:
    """Python int (mod 2^64) -> the int64 with the same bit pattern."""
    v &= _MASK64
    return v - (1 << 64) if v >= (1 << 63) else v


_GOLD = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)
_C3 = _s64(0xD1B54A32D192ED03)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor (bit pattern as uint64)."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def counter_uniform(seed: int, step: int, n: int, device="cpu", offset: int = 0) -> torch.Tensor:
    """xi(i) in [-1, 1), i = offset..offset+n-1: splitmix64 of (seed, step, i); exact dyadic values."""
    key = _s64(seed * 0x9E3779B97F4A7C15 + step * 0xD1B54A32D192ED03)
    i = torch.arange(offset + 1, offset + n + 1, dtype=torch.int64, device=device)
    z = i * _GOLD + key  # wraps mod 2^64
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    z = z ^ _lsr(z, 31)
    u53 = _lsr(z, 11).to(torch.float64)  # exact: < 2^53
    return u53 * (2.0 ** -52) - 1.0


@dataclass(frozen=True)
class Grid:
    """n^dim interior points of the unit interval/square/cube; sigma is the Helmholtz shift."""

    n: int
    dim: int
    sigma: float = 1.0

    @property
    def N(self) -> int:
        return self.n ** self.dim

    @property
    def h(self) -> float:
        return 1.0 / (self.n + 1)

    @property
    def shape(self):
        return (self.n,) * self.dim


def helmholtz_diag(g: Grid) -> float:
    """Diagonal of A = -Delta_h + sigma I: 2 dim / h^2 + sigma (Jacobi preconditioner)."""
    return 2.0 * g.dim / g.h ** 2 + g.sigma


def helmholtz_apply(g: Grid, x: torch.Tensor) -> torch.Tensor:
    """y = A x, A = -Delta_h + sigma I, homogeneous Dirichlet (harness operator; PAPER.md:237 'b~ <- A x~')."""
    u = x.reshape(g.shape)
    y = helmholtz_diag(g) * u
    inv_h2 = 1.0 / g.h ** 2
    for ax in range(g.dim):
        n = g.n
        lo = [slice(None)] * g.dim
        hi = [slice(None)] * g.dim
        lo[ax] = slice(0, n - 1)
        hi[ax] = slice(1, n)
        y[tuple(lo)] -= inv_h2 * u[tuple(hi)]
        y[tuple(hi)] -= inv_h2 * u[tuple(lo)]
    return y.reshape(-1)


def _modes(dim: int):
    rng = np.random.default_rng(SEED)
    K = 8 if dim == 3 else 4
    q = rng.integers(1, 5, size=(K, dim))
    omega = rng.uniform(0.5, 3.0, size=K)
    phi = rng.uniform(0.0, 2.0 * math.pi, size=K)
    return q, omega, phi


def _coords(g: Grid, device, offset: int = 0, count: int | None = None):
    """Coordinates of DOFs offset..offset+count-1 (lexicographic, last axis fastest)."""
    count = g.N - offset if count is None else count
    idx = torch.arange(offset, offset + count, dtype=torch.int64, device=device)
    xs = []
    rem = idx
    for _ in range(g.dim):
        xs.append(((rem % g.n) + 1).to(torch.float64) * g.h)
        rem = rem // g.n
    return xs[::-1]  # axis 0 slowest


def smooth_field(g: Grid, t: float, device="cpu", offset: int = 0, count: int | None = None) -> torch.Tensor:
    """u(x, t) of the 'smooth' family on DOFs offset..offset+count-1."""
    X = _coords(g, device, offset, count)
    env = torch.ones_like(X[0])
    for xj in X:
        env = env * torch.sin(math.pi * xj)
    u = env * (1.0 + 0.3 * math.sin(2.0 * math.pi * t))
    c = [0.3 + 0.4 * t, 0.5 + 0.1 * math.sin(2.0 * math.pi * t), 0.5 + 0.1 * math.cos(2.0 * math.pi * t)]
    r2 = torch.zeros_like(X[0])
    for j, xj in enumerate(X):
        r2 = r2 + (xj - c[j]) ** 2
    u = u + torch.exp(-r2 / 0.02)
    q, omega, phi = _modes(g.dim)
    for k in range(q.shape[0]):
        a = math.cos(omega[k] * t + phi[k])
        m = torch.full_like(X[0], a)
        for j, xj in enumerate(X):
            m = m * torch.sin(float(q[k, j]) * math.pi * xj)
        u = u + m
    return u


def manufactured_step(g: Grid, n: int, dt: float = 1e-3, eta_rel: float = 1e-8, device="cpu",
                      seed: int = SEED):
    """Open-loop step n: (b_n, x_n, Ax_n) with b_n = A u(t_n), x_n = u + eta xi_n, Ax_n = A x_n."""
    u = smooth_field(g, n * dt, device)
    eta = eta_rel * float(u.abs().max())
    x = u + eta * counter_uniform(seed, n, g.N, device)
    b = helmholtz_apply(g, u)
    Ax = helmholtz_apply(g, x)
    return b, x, Ax


def prescribed_rhs(g: Grid, n: int, dt: float = 1e-3, device="cpu") -> torch.Tensor:
    """Closed-loop RHS b_n = f(., t_n) with f the smooth family (independent of any solver output)."""
    return smooth_field(g, n * dt, device)


def manufactured_step_slab(n_xy: int, nz_local: int, rank: int, world: int, n: int, dt: float = 1e-3,
                           eta_rel: float = 1e-8, sigma: float = 1.0, device="cpu", seed: int = SEED):
    """Rank `rank`'s z-slab of a global n_xy x n_xy x (nz_local*world) manufactured step (weak
    scaling: every rank holds nz_local planes)."""
    return manufactured_step_zrange(n_xy, nz_local * world, rank * nz_local, (rank + 1) * nz_local, n, dt,
                                    eta_rel, sigma, device, seed)


def manufactured_step_zrange(n_xy: int, nz_global: int, z0: int, z1: int, n: int, dt: float = 1e-3,
                             eta_rel: float = 1e-8, sigma: float = 1.0, device="cpu", seed: int = SEED):
    """z-planes [z0, z1) of a global n_xy x n_xy x nz_global manufactured step (strong scaling: a
    fixed global grid split into contiguous plane ranges of any sizes).

    The field and noise are those of the global grid restricted to the slab (contiguous DOF
    range); the harness operator is the 7-point Helmholtz stencil of the slab with
    homogeneous Dirichlet faces (block-diagonal across ranks: a valid SPD operator, no halo
    exchange needed for synthetic timing inputs).
    """
    nzg = nz_global
    nz_local = z1 - z0
    count = n_xy * n_xy * nz_local
    offset = z0 * n_xy * n_xy
    idx = torch.arange(offset, offset + count, dtype=torch.int64, device=device)
    xs = [((idx // (n_xy * n_xy)) + 1).to(torch.float64) / (nzg + 1),
          (((idx // n_xy) % n_xy) + 1).to(torch.float64) / (n_xy + 1),
          ((idx % n_xy) + 1).to(torch.float64) / (n_xy + 1)]
    u = _field_at(xs, n * dt, 3)
    eta = eta_rel * (2.3 + _modes(3)[0].shape[0])  # analytic bound of |u|: identical on every rank
    x = u + eta * counter_uniform(seed, n, count, device, offset=offset)
    gl = _SlabGrid(n_xy, nz_local, sigma)
    return gl.apply(u), x, gl.apply(x)


def _field_at(X, t: float, dim: int) -> torch.Tensor:
    env = torch.ones_like(X[0])
    for xj in X:
        env = env * torch.sin(math.pi * xj)
    u = env * (1.0 + 0.3 * math.sin(2.0 * math.pi * t))
    c = [0.3 + 0.4 * t, 0.5 + 0.1 * math.sin(2.0 * math.pi * t), 0.5 + 0.1 * math.cos(2.0 * math.pi * t)]
    r2 = torch.zeros_like(X[0])
    for j, xj in enumerate(X):
        r2 = r2 + (xj - c[j]) ** 2
    u = u + torch.exp(-r2 / 0.02)
    q, omega, phi = _modes(dim)
    for k in range(q.shape[0]):
        m = torch.full_like(X[0], math.cos(omega[k] * t + phi[k]))
        for j, xj in enumerate(X):
            m = m * torch.sin(float(q[k, j]) * math.pi * xj)
        u = u + m
    return u


@dataclass(frozen=True)
class _SlabGrid:
    n_xy: int
    nz: int
    sigma: float

    def apply(self, x: torch.Tensor) -> torch.Tensor:
        h = 1.0 / (self.n_xy + 1)
        u = x.reshape(self.nz, self.n_xy, self.n_xy)
        y = (6.0 / h ** 2 + self.sigma) * u
        inv = 1.0 / h ** 2
        for ax in range(3):
            n = u.shape[ax]
            lo = [slice(None)] * 3
            hi = [slice(None)] * 3
            lo[ax] = slice(0, n - 1)
            hi[ax] = slice(1, n)
            y[tuple(lo)] -= inv * u[tuple(hi)]
            y[tuple(hi)] -= inv * u[tuple(lo)]
        return y.reshape(-1)
