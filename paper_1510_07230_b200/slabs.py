"""Slab decomposition of the grid along axis 0, host side.

Mirrors the engine's partition (csrc/engine.cu, Engine::Engine): rank r of S
owns planes [z0, z0 + nz) with nz = n0 // S (+1 for the first n0 % S ranks).
The collectives per operator are:
  * H u / Laplacian: one-plane halo per side per orbital (send first plane to
    rank-1, last plane to rank+1), zero beyond the global box;
  * Gram / Sigma / per-orbital scalars: local partial sums + all-reduce(sum);
  * Poisson: all-gather of the local 4 pi rho slabs, replicated full-grid solve.
`sharded_laplacian` / `sharded_gram` restate that data flow with
torch.distributed so the multi-rank logic is testable on CPU (gloo).
"""
from __future__ import annotations

import numpy as np


def slab_bounds(n0: int, size: int, rank: int) -> tuple[int, int]:
    base, rem = divmod(n0, size)
    nz = base + (1 if rank < rem else 0)
    z0 = rank * base + min(rank, rem)
    return z0, nz


def local_laplacian(u_local: np.ndarray, halo_lo, halo_hi, n1: int, n2: int, h) -> np.ndarray:
    """7-point Dirichlet Laplacian of a slab (N, nz*n1*n2) given neighbour
    planes (N, n1*n2) or None at the global boundary (grid.cpp:94-122 order)."""
    N = u_local.shape[0]
    nz = u_local.shape[1] // (n1 * n2)
    f = u_local.reshape(N, nz, n1, n2)
    lo = np.zeros((N, 1, n1, n2)) if halo_lo is None else halo_lo.reshape(N, 1, n1, n2)
    hi = np.zeros((N, 1, n1, n2)) if halo_hi is None else halo_hi.reshape(N, 1, n1, n2)
    g = np.concatenate([lo, f, hi], axis=1)
    out = (g[:, :-2] - 2.0 * f + g[:, 2:]) / h[0] ** 2
    p1 = np.pad(f, ((0, 0), (0, 0), (1, 1), (0, 0)))
    out = out + (p1[:, :, :-2] - 2.0 * f + p1[:, :, 2:]) / h[1] ** 2
    p2 = np.pad(f, ((0, 0), (0, 0), (0, 0), (1, 1)))
    out = out + (p2[:, :, :, :-2] - 2.0 * f + p2[:, :, :, 2:]) / h[2] ** 2
    return out.reshape(N, -1)


def exchange_halos(u_local: np.ndarray, plane: int, rank: int, size: int, dist):
    """Send first/last plane to the axis-0 neighbours; returns (lo, hi) or None."""
    import torch

    lo = hi = None
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(u_local[:, :plane])), rank - 1))
        lo_t = torch.empty((u_local.shape[0], plane), dtype=torch.float64)
        reqs.append(dist.irecv(lo_t, rank - 1))
    if rank + 1 < size:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(u_local[:, -plane:])), rank + 1))
        hi_t = torch.empty((u_local.shape[0], plane), dtype=torch.float64)
        reqs.append(dist.irecv(hi_t, rank + 1))
    for r in reqs:
        r.wait()
    if rank > 0:
        lo = lo_t.numpy()
    if rank + 1 < size:
        hi = hi_t.numpy()
    return lo, hi


def sharded_laplacian(u_local, n1, n2, h, rank, size, dist):
    lo, hi = exchange_halos(u_local, n1 * n2, rank, size, dist)
    return local_laplacian(u_local, lo, hi, n1, n2, h)


def sharded_gram(a_local, b_local, weight, dist):
    import torch

    g = torch.from_numpy(weight * a_local @ b_local.T)
    dist.all_reduce(g)
    return g.numpy()


def gather_full(field_local, n0, plane, rank, size, dist):
    """All-gather of per-rank slabs into the full field (uneven splits padded)."""
    import torch

    nz_max = slab_bounds(n0, size, 0)[1]
    buf = np.zeros(nz_max * plane)
    buf[: field_local.size] = field_local
    out = [torch.empty(nz_max * plane, dtype=torch.float64) for _ in range(size)]
    dist.all_gather(out, torch.from_numpy(buf))
    parts = [out[r].numpy()[: slab_bounds(n0, size, r)[1] * plane] for r in range(size)]
    return np.concatenate(parts)
