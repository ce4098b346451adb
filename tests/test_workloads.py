"""The seeded input generators (workloads/) against independent constructions."""

import numpy as np
import scipy.sparse as sp
import torch

from workloads import Grid, counter_uniform, helmholtz_apply, manufactured_step


def _splitmix_ref(seed, step, n):
    with np.errstate(over="ignore"):
        key = np.uint64((seed * 0x9E3779B97F4A7C15 + step * 0xD1B54A32D192ED03) & ((1 << 64) - 1))
        z = np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + key
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0


def test_counter_hash_matches_uint64_reference():
    for seed, step in [(10863, 0), (1, 5), (123456789, 987654)]:
        np.testing.assert_array_equal(counter_uniform(seed, step, 4097).numpy(), _splitmix_ref(seed, step, 4097))
    u = counter_uniform(10863, 3, 1 << 16).numpy()
    assert u.min() >= -1.0 and u.max() < 1.0 and abs(u.mean()) < 0.02


def test_offset_slices_concatenate():
    full = counter_uniform(7, 2, 1000)
    parts = torch.cat([counter_uniform(7, 2, 300, offset=0), counter_uniform(7, 2, 700, offset=300)])
    assert torch.equal(full, parts)


def _dense_helmholtz(g: Grid):
    n, h = g.n, g.h
    T = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]) / h ** 2
    I = sp.identity(n)
    if g.dim == 1:
        L = T
    elif g.dim == 2:
        L = sp.kron(T, I) + sp.kron(I, T)
    else:
        L = sp.kron(sp.kron(T, I), I) + sp.kron(sp.kron(I, T), I) + sp.kron(sp.kron(I, I), T)
    return (L + g.sigma * sp.identity(g.N)).tocsr()


def test_stencil_matches_kron_laplacian():
    rng = np.random.default_rng(0)
    for g in (Grid(17, 1), Grid(9, 2, 0.5), Grid(6, 3, 0.0)):
        x = rng.standard_normal(g.N)
        y = helmholtz_apply(g, torch.from_numpy(x)).numpy()
        np.testing.assert_allclose(y, _dense_helmholtz(g) @ x, rtol=1e-13, atol=1e-9)


def test_manufactured_step_shapes_and_consistency():
    g = Grid(8, 3)
    b, x, Ax = manufactured_step(g, 4)
    assert b.shape == x.shape == Ax.shape == (g.N,)
    np.testing.assert_allclose(Ax.numpy(), _dense_helmholtz(g) @ x.numpy(), rtol=1e-12, atol=1e-9)
    # x solves A x = b to the synthetic "solver tolerance" eta ~ 1e-8
    assert 0 < np.linalg.norm(Ax - b) / np.linalg.norm(b) < 1e-5
