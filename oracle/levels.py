"""TEST INFRASTRUCTURE (oracle) — numpy restatements of the reference's outer
refinement pieces, used only by tests/ to pin the golden fixtures; the product
path (libparorb_b200.so) never imports or calls this module.

  prolongate          grid.cpp:151-203   separable linear interpolation n -> 2n+1
                                         per axis (axes 0, 1, 2 in order) with
                                         linear extrapolation past the ends
  refine              grid.cpp:137-149   refine_uniform
  initialize_raw      optimizer.cpp:156-197 (before the orthonormalisation):
                                         Gaussians at the atoms, Rng widths and
                                         1e-2 uniform noise, in the reference's
                                         draw order
"""
from __future__ import annotations

import numpy as np

from paper_1510_07230_b200.rng import Rng


def refine(n):
    return tuple(2 * int(x) + 1 for x in n)


def _prolong_axis(cur: np.ndarray, axis: int) -> np.ndarray:
    """One pass of grid.cpp:166-200 along `axis` of a 3D array."""
    c = np.moveaxis(cur, axis, 0)
    n = c.shape[0]
    m = 2 * n + 1

    def line(i):
        if i < 0:
            return 2.0 * c[0] - c[1] if n >= 2 else c[0]
        if i >= n:
            return 2.0 * c[n - 1] - c[n - 2] if n >= 2 else c[n - 1]
        return c[i]

    out = np.empty((m,) + c.shape[1:])
    for j in range(m):
        out[j] = line((j - 1) // 2) if j % 2 == 1 else 0.5 * (line(j // 2 - 1) + line(j // 2))
    return np.moveaxis(out, 0, axis)


def prolongate(u: np.ndarray, n) -> np.ndarray:
    """u: (ng,) on grid n (axis 2 fastest) -> (ng_fine,) on refine(n)."""
    cur = np.asarray(u, dtype=np.float64).reshape(tuple(n))
    for axis in range(3):
        cur = _prolong_axis(cur, axis)
    return cur.reshape(-1)


def initialize_raw(n, extent, atoms, n_orbitals: int, seed: int) -> np.ndarray:
    """The fields initialize_orbitals orthonormalises (attempt 0 seed)."""
    h = [extent[a] / (n[a] + 1) for a in range(3)]
    k0, k1, k2 = np.meshgrid(*[np.arange(n[a]) for a in range(3)], indexing="ij")
    xyz = [(k0.reshape(-1) + 1) * h[0], (k1.reshape(-1) + 1) * h[1], (k2.reshape(-1) + 1) * h[2]]
    ng = int(np.prod(n))
    rng = Rng(seed)
    out = np.empty((n_orbitals, ng))
    for i in range(n_orbitals):
        c = atoms[i % len(atoms)][:3] if len(atoms) else [0.5 * e for e in extent]
        width = rng.uniform(0.5, 2.0)
        r2 = (xyz[0] - c[0]) ** 2
        r2 = r2 + (xyz[1] - c[1]) ** 2
        r2 = r2 + (xyz[2] - c[2]) ** 2
        f = np.exp(-r2 / (2.0 * width * width))
        noise = np.array([1e-2 * rng.uniform(-1.0, 1.0) for _ in range(ng)])
        out[i] = f + noise
    return out
