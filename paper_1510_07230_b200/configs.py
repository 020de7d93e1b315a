"""BASELINE.json configurations as seeded synthetic problems.

Resolutions of the spec conflicts fixed here and in DESIGN.md:

* C3: the reference box is [0, L]^3 with interior points at (k+1)h, h = L/(n+1)
  (grid.hpp:11-14, grid.cpp:33); molecules are centred at L/2 on every axis and
  "64^3" means 64 interior points.
* C4: nuclei are the reference's softened Coulomb wells, softening a = 1 bohr
  (energy.cpp:78-99, energy.hpp:16).
* C5: the start block is i.i.d. N(0,1) from `Rng(seed)` drawn orbital-major,
  then orthonormalised (tests/problems.hpp:59-68); seed 42.
* C6: one BASELINE "outer iteration" is one InnerLoop iteration with n_org = 1
  (optimizer.cpp:358-576), so `max_inner` = 50/50/40/20.
* C7: cluster geometry: positions are drawn first (x, y, z uniforms per
  candidate, rejected when closer than 2.0 bohr to an accepted atom), then one
  uniform per atom for Z; the sub-box is centred in the computational box;
  the sum of Z is then adjusted by the deterministic rule in `_adjust_charges`.
  N is the orbital count the config names (the reference decouples N from the
  charges, energy.hpp:24-32).
* C8: config 5 uses L = 20 n / 64 and V(r) = sum_k A_k exp(-|r - c_k|^2 / 8),
  A_k ~ U(-5, 0), c_k uniform in the box.

Occupation defaults to 1 (the unmodified reference, gate A); 2 is gate B.
"""
from __future__ import annotations

import dataclasses
import json
import math
from typing import Any

from .rng import Rng

DEFAULT_START_SEED = 42


@dataclasses.dataclass
class ProblemSpec:
    name: str
    n: tuple[int, int, int]
    extent: tuple[float, float, float]
    atoms: list[tuple[float, float, float, float, float]]  # x, y, z, Z, softening
    n_orbitals: int
    hartree: bool = True
    xc: bool = True
    occupation: float = 1.0
    start_seed: int = DEFAULT_START_SEED
    max_inner: int = 50
    algorithm: str = "opt_par_mod"
    params: dict[str, Any] = dataclasses.field(default_factory=dict)
    # C5 only: Gaussian wells (cx, cy, cz, amplitude, width) as the local potential
    wells: list[tuple[float, float, float, float, float]] | None = None

    @property
    def num_points(self) -> int:
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def spacing(self) -> tuple[float, float, float]:
        return tuple(self.extent[a] / (self.n[a] + 1) for a in range(3))  # grid.cpp:33

    def optimizer_params(self) -> dict[str, Any]:
        p = {"max_inner": self.max_inner, "n_org": 1, "n_diag": 100}
        p.update(self.params)
        return p

    def trace_ref_spec(self, threads: int = 1, start: dict | None = None) -> dict:
        """Spec understood by oracle/ref_harness/trace_ref.cpp (test infrastructure)."""
        return {
            "n": list(self.n),
            "extent": list(self.extent),
            "atoms": [list(a) for a in self.atoms],
            "n_orbitals": self.n_orbitals,
            "hartree": self.hartree,
            "xc": self.xc,
            "start": start or {"kind": "random_orthonormal", "seed": self.start_seed},
            "algorithm": self.algorithm,
            "params": self.optimizer_params(),
            "threads": threads,
        }

    def to_json(self) -> str:
        return json.dumps(dataclasses.asdict(self))


def _place_atoms(rng: Rng, count: int, lo: float, hi: float, min_sep: float):
    pos: list[tuple[float, float, float]] = []
    tries = 0
    while len(pos) < count:
        tries += 1
        if tries > 1_000_000:
            raise RuntimeError("atom placement did not converge")
        c = (rng.uniform(lo, hi), rng.uniform(lo, hi), rng.uniform(lo, hi))
        if all(math.dist(c, q) >= min_sep for q in pos):
            pos.append(c)
    return pos


def _draw_charges(rng: Rng, count: int, values, probs):
    out = []
    for _ in range(count):
        u = rng.uniform()
        acc = 0.0
        z = values[-1]
        for v, p in zip(values, probs):
            acc += p
            if u < acc:
                z = v
                break
        out.append(z)
    return out


def _adjust_charges(z: list[int], allowed: list[int], target: int) -> list[int]:
    """Re-balance drawn charges so sum(Z) equals `target` (or, if no mix of
    `allowed` values on len(z) atoms sums to it exactly, the smallest reachable
    sum above it). Among all per-value counts with that sum, pick the one
    closest (L1) to the drawn counts, ties broken by the lexicographically
    smallest count vector; then re-label the lowest-index atoms of each
    surplus value with the deficit values in ascending order. Deterministic;
    DESIGN.md (C7)."""
    import itertools

    allowed = sorted(allowed)
    m = len(z)
    drawn = [z.count(v) for v in allowed]
    best = None
    for counts in itertools.product(range(m + 1), repeat=len(allowed) - 1):
        last = m - sum(counts)
        if last < 0:
            continue
        c = list(counts) + [last]
        total = sum(v * k for v, k in zip(allowed, c))
        if total < target:
            continue
        key = (total - target, sum(abs(a - b) for a, b in zip(c, drawn)), c)
        if best is None or key < best:
            best = key
    want = best[2]
    z = list(z)
    surplus = {v: drawn[i] - want[i] for i, v in enumerate(allowed)}
    deficit = [v for v in allowed for _ in range(max(0, -surplus[v]))]
    k = 0
    for i, v in enumerate(z):
        if surplus[v] > 0 and k < len(deficit):
            surplus[v] -= 1
            z[i] = deficit[k]
            k += 1
    return z


def config1() -> ProblemSpec:
    """BASELINE configs[0]: O + 2 H, N = 5, 64^3 in a 20 bohr box, 50 iterations."""
    L = 20.0
    c = L / 2
    atoms = [(c, c, c, 8.0, 1.0), (c + 1.43, c + 1.11, c, 1.0, 1.0), (c - 1.43, c + 1.11, c, 1.0, 1.0)]
    return ProblemSpec("C1", (64, 64, 64), (L, L, L), atoms, 5, max_inner=50)


def config2(seed: int = 20002) -> ProblemSpec:
    """BASELINE configs[1]: 20 nuclei in a 24 bohr sub-box of a 32 bohr box, 96^3."""
    L, sub = 32.0, 24.0
    lo = (L - sub) / 2
    rng = Rng(seed)
    pos = _place_atoms(rng, 20, lo, lo + sub, 2.0)
    z = _draw_charges(rng, 20, [1, 6], [0.5, 0.5])
    total = sum(z) + (sum(z) % 2)  # round sum(Z) up to even
    atoms = [(x, y, w, float(q), 1.0) for (x, y, w), q in zip(pos, z)]
    return ProblemSpec("C2", (96, 96, 96), (L, L, L), atoms, total // 2, max_inner=50)


def config3(seed: int = 20003) -> ProblemSpec:
    """BASELINE configs[2]: 60 nuclei, sum(Z) = 256, N = 128, 128^3 in 40 bohr."""
    L, sub = 40.0, 30.0
    lo = (L - sub) / 2
    rng = Rng(seed)
    pos = _place_atoms(rng, 60, lo, lo + sub, 2.0)
    z = _adjust_charges(_draw_charges(rng, 60, [1, 6, 8], [0.5, 0.35, 0.15]), [1, 6, 8], 256)
    atoms = [(x, y, w, float(q), 1.0) for (x, y, w), q in zip(pos, z)]
    return ProblemSpec("C3", (128, 128, 128), (L, L, L), atoms, 128, max_inner=40)


def config4(seed: int = 20004) -> ProblemSpec:
    """BASELINE configs[3]: 240 nuclei, N = 512, 192^3 in 60 bohr (>= 2 GPUs)."""
    L, sub = 60.0, 48.0
    lo = (L - sub) / 2
    rng = Rng(seed)
    pos = _place_atoms(rng, 240, lo, lo + sub, 2.0)
    z = _adjust_charges(_draw_charges(rng, 240, [1, 6], [0.5, 0.5]), [1, 6], 1024)
    atoms = [(x, y, w, float(q), 1.0) for (x, y, w), q in zip(pos, z)]
    return ProblemSpec("C4", (192, 192, 192), (L, L, L), atoms, 512, max_inner=20)


def config5(n: int, n_orbitals: int, seed: int = 20005) -> ProblemSpec:
    """BASELINE configs[4] sweep point: smooth seeded potential of 32 Gaussians."""
    L = 20.0 * n / 64
    rng = Rng(seed + 7919 * n)
    wells = []
    for _ in range(32):
        c = (rng.uniform(0.0, L), rng.uniform(0.0, L), rng.uniform(0.0, L))
        amp = rng.uniform(-5.0, 0.0)
        wells.append((c[0], c[1], c[2], amp, 2.0))
    return ProblemSpec(f"C5-{n}-{n_orbitals}", (n, n, n), (L, L, L), [], n_orbitals,
                       hartree=False, xc=False, max_inner=1, wells=wells)


def small_molecule(n: int = 16, n_orbitals: int = 4, L: float = 8.0, **kw) -> ProblemSpec:
    """Scaled-down C1 (same chemistry, fewer points) for fast parity tests."""
    c = L / 2
    atoms = [(c, c, c, 8.0, 1.0), (c + 1.43, c + 1.11, c, 1.0, 1.0), (c - 1.43, c + 1.11, c, 1.0, 1.0)]
    spec = ProblemSpec(f"mol{n}", (n, n, n), (L, L, L), atoms, n_orbitals, max_inner=kw.pop("max_inner", 12))
    for k, v in kw.items():
        setattr(spec, k, v)
    return spec


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4}


def by_name(name: str) -> ProblemSpec:
    return CONFIGS[name]()
