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


# ---- size-independent fingerprints (oracle/ref_harness/trace_ref.cpp, Sketch)

_M1 = np.uint64(0xD1B54A32D192ED03)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def sketch_signs(seed: int, p0: int, p1: int, m: int) -> np.ndarray:
    """X(p, a) = +-1 for p in [p0, p1), a < m: the splitmix64 finaliser of
    seed ^ ((p * m + a) * M1), sign from the top bit — bit-identical to
    trace_ref.cpp:sketch_sign."""
    key = (np.arange(p0, p1, dtype=np.uint64)[:, None] * np.uint64(m)
           + np.arange(m, dtype=np.uint64)[None, :])
    with np.errstate(over="ignore"):
        z = np.uint64(seed) ^ (key * _M1)
        z ^= z >> np.uint64(30)
        z *= _M2
        z ^= z >> np.uint64(27)
        z *= _M3
        z ^= z >> np.uint64(31)
    return np.where((z >> np.uint64(63)) != 0, -1.0, 1.0)


_SIGN_CACHE: dict = {}


def _signs_cached(ng: int, m: int, seed: int) -> np.ndarray:
    """The whole N_g x m sign matrix as int8 (exact), cached: the GPU parity tests
    sketch several blocks of the same shape."""
    key = (ng, m, seed)
    if key not in _SIGN_CACHE:
        _SIGN_CACHE.clear()
        x = np.empty((ng, m), dtype=np.int8)
        for p0 in range(0, ng, 1 << 18):
            p1 = min(ng, p0 + (1 << 18))
            x[p0:p1] = sketch_signs(seed, p0, p1, m)
        _SIGN_CACHE[key] = x
    return _SIGN_CACHE[key]


def sketch_block(w: np.ndarray, weight: float, m: int = 64, seed: int = 7,
                 chunk: int = 1 << 17) -> np.ndarray:
    """S = sqrt(w) * W X (N x m) for an orbital-major block W (N x N_g)."""
    n, ng = w.shape
    x = _signs_cached(ng, m, seed)
    s = np.zeros((n, m))
    for p0 in range(0, ng, chunk):
        p1 = min(ng, p0 + chunk)
        s += w[:, p0:p1] @ x[p0:p1].astype(np.float64)
    return np.sqrt(weight) * s


def sample_points(ng: int, k: int) -> np.ndarray:
    """p_j = (j * 2654435761) mod N_g (trace_ref.cpp:sample_points)."""
    return (np.arange(k, dtype=np.uint64) * np.uint64(2654435761) % np.uint64(ng)).astype(np.int64)


def sketch_projector_distance(s1: np.ndarray, g1: np.ndarray, s2: np.ndarray, g2: np.ndarray) -> float:
    """Estimate of ||P1 - P2||_F from two sketches S_k = sqrt(w) W_k X and Grams
    G_k = w W_k W_k^T: X^T P_k X = S_k^T G_k^-1 S_k, and for Rademacher X every
    off-diagonal entry of X^T (P1 - P2) X has mean square ||P1 - P2||_F^2, so the
    mean over the m(m-1) off-diagonal entries is an unbiased estimate (relative
    spread ~ sqrt(2 / (m (m - 1))) ~ 2% at m = 64)."""
    q1 = s1.T @ np.linalg.solve(g1, s1)
    q2 = s2.T @ np.linalg.solve(g2, s2)
    d = q1 - q2
    m = d.shape[0]
    off = d[~np.eye(m, dtype=bool)]
    return float(np.sqrt(np.mean(off * off)))
