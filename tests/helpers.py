"""Shared parity helpers (test-only)."""
import numpy as np


def _orthonormal_rows(w: np.ndarray, weight: float) -> np.ndarray:
    q, _ = np.linalg.qr((np.sqrt(weight) * w).T)
    return q.T


def projector_distance(w1: np.ndarray, w2: np.ndarray, weight: float) -> float:
    """||P1 - P2||_F of the subspaces spanned by the weighted orbitals sqrt(w) W
    (test_manifold.cpp:90-104), as sqrt(2) * ||B - (B A^T) A||_F with A, B the
    orthonormalised rows — never forms an N_g x N_g matrix and
    avoids the cancellation of sqrt(2N - 2||A B^T||^2). Raw opt_par_mod steps
    leave W slightly non-orthonormal, hence the re-orthonormalisation."""
    a = _orthonormal_rows(w1, weight)
    b = _orthonormal_rows(w2, weight)
    m = b @ a.T
    return float(np.sqrt(2.0) * np.linalg.norm(b - m @ a))
