"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no partition, no kernel, no reduction):
it only draws point clouds, matvec vectors and sampled row sets with numpy PCG64, following
the recipe in DESIGN.md §"Input recipe" (BASELINE.json configs[0..4]).

Config k (1-based, matching BASELINE.json configs[k-1]):

  1  n=8192      uniform [0,1]^3                                  Coulomb           q=64   id_tol 1e-6
  2  n=1048576   uniform [0,1]^3                                  Coulomb           q=200  id_tol 1e-8
  3  n=262144    unit sphere surface (normalised Gaussians)       Gaussian h=0.5    q=128  id_tol 1e-6
  4  n=4194304   2-D mixture of 16 Gaussians (sigma .02, clipped)  Matern-3/2 l=0.1  q=256  id_tol 1e-6
  5  n=262144    5-D mixture of 8 Gaussians (sigma .3)            Gaussian h=1.0    q=256  id_tol 1e-4

Every config can be drawn at a reduced n (same distribution, same seed) for the small parity cases.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 20601885

KERNEL_COULOMB = 1
KERNEL_GAUSSIAN = 2
KERNEL_MATERN32 = 3
KERNEL_LAPLACE = 4
KERNEL_BUMP = 5
KERNEL_COSDOT = 6  # Table 1 kappa_3 = cos(x . y)
KERNEL_MQSHIFT = 7  # sqrt(1 + c |x - y + a|^2), non-symmetric; params (c, a_0, ..., a_{d-1})

# (n, d, kernel_id, kernel_params, leaf_size, id_tol, tau, name)
CONFIGS = {
    1: dict(n=8192, d=3, kernel=KERNEL_COULOMB, params=(), q=64, id_tol=1e-6, tau=0.5,
            name="cube8k_coulomb_1e-6"),
    2: dict(n=1 << 20, d=3, kernel=KERNEL_COULOMB, params=(), q=200, id_tol=1e-8, tau=0.5,
            name="cube1M_coulomb_1e-8"),
    3: dict(n=1 << 18, d=3, kernel=KERNEL_GAUSSIAN, params=(0.5,), q=128, id_tol=1e-6, tau=0.5,
            name="sphere256k_gauss0.5_1e-6"),
    4: dict(n=1 << 22, d=2, kernel=KERNEL_MATERN32, params=(0.1,), q=256, id_tol=1e-6, tau=0.5,
            name="mix2d_4M_matern0.1_1e-6"),
    5: dict(n=1 << 18, d=5, kernel=KERNEL_GAUSSIAN, params=(1.0,), q=256, id_tol=1e-4, tau=0.5,
            name="mix5d_256k_gauss1.0_1e-4"),
    # not a BASELINE config: the non-symmetric family (the paper's shifted multiquadric of P:711-716,
    # c = 100, here with a = [0, 0.3] so the shift lies inside the data's extent) on uniform 2-D points
    6: dict(n=1 << 20, d=2, kernel=KERNEL_MQSHIFT, params=(100.0, 0.0, 0.3), q=128, id_tol=1e-6, tau=0.5,
            name="mq2d_1M_shifted_multiquadric_1e-6"),
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def points(config: int, n: int | None = None, seed_offset: int = 0) -> np.ndarray:
    """Point cloud of `config` (n x d, fp64, C-contiguous, point-major). `n` overrides the size;
    `seed_offset` draws an independent instance (multi-GPU weak scaling)."""
    c = CONFIGS[config]
    n = c["n"] if n is None else int(n)
    rng = _rng(SEED_BASE + config + seed_offset)
    if config in (1, 2):
        x = rng.random((n, 3))
    elif config == 6:
        x = rng.random((n, 2))
    elif config == 3:
        g = rng.standard_normal((n, 3))
        x = g / np.linalg.norm(g, axis=1, keepdims=True)
    elif config == 4:
        centres = 0.1 + 0.8 * rng.random((16, 2))
        comp = np.arange(n) % 16
        x = np.clip(centres[comp] + 0.02 * rng.standard_normal((n, 2)), 0.0, 1.0)
    elif config == 5:
        centres = -1.0 + 2.0 * rng.random((8, 5))
        comp = np.arange(n) % 8
        x = centres[comp] + 0.3 * rng.standard_normal((n, 5))
    else:
        raise ValueError(config)
    return np.ascontiguousarray(x, dtype=np.float64)


def matvec_vector(config: int, n: int) -> np.ndarray:
    """x ~ N(0, I) for the relative matvec error (seed + 1000)."""
    return _rng(SEED_BASE + config + 1000).standard_normal(n)


def sample_rows(config: int, n: int, count: int = 1024) -> np.ndarray:
    """Seeded rows (original order) on which dense K.x is evaluated when n > 16384 (seed + 2000)."""
    if n <= 16384:
        return np.arange(n, dtype=np.int64)
    return np.sort(_rng(SEED_BASE + config + 2000).choice(n, count, replace=False)).astype(np.int64)


def uniform_cube(n: int, d: int, seed: int) -> np.ndarray:
    return np.ascontiguousarray(_rng(seed).random((n, d)), dtype=np.float64)


def clustered(n: int, d: int, seed: int, k: int = 4, sigma: float = 0.05) -> np.ndarray:
    """Mixture of k isotropic Gaussians: adaptive (non-uniform) trees for the small cases."""
    rng = _rng(seed)
    c = rng.random((k, d))
    comp = rng.integers(0, k, n)
    return np.ascontiguousarray(c[comp] + sigma * rng.standard_normal((n, d)), dtype=np.float64)


def equispaced_1d(n: int) -> np.ndarray:
    """n equispaced points i/(n-1) on [0,1] (the 1-D layout of the paper's Fig. 4)."""
    return (np.arange(n, dtype=np.float64) / (n - 1)).reshape(n, 1).copy()


def three_spheres(n: int, seed: int) -> np.ndarray:
    """The "3-sphere" dataset of PAPER §6: points on the surfaces of three intersecting unit
    spheres whose centres form an equilateral triangle of side 1 (reading: side exactly 1, the sphere
    of each point uniform over the three, directions normalised Gaussians).  Used by the section-6.3
    memory comparison (n = 20000)."""
    rng = _rng(seed)
    centres = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.5, np.sqrt(3.0) / 2.0, 0.0]])
    comp = rng.integers(0, 3, n)
    g = rng.standard_normal((n, 3))
    x = centres[comp] + g / np.linalg.norm(g, axis=1, keepdims=True)
    return np.ascontiguousarray(x, dtype=np.float64)
