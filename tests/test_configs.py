"""Seeded BASELINE configurations and the portable generator (host logic)."""
import math

import numpy as np

from paper_1510_07230_b200 import configs
from paper_1510_07230_b200.rng import Rng


def test_rng_matches_reference_bits(port):
    """rng.hpp:13-41: the Python restatement and the C restatement draw the same
    mt19937_64 bits and the same Box-Muller normals."""
    r = Rng(42)
    py = np.array([r.normal() for _ in range(1001)])
    assert np.array_equal(py, port.random_normals(42, 1001))
    r2 = Rng(5489)
    assert r2.next_u64() == 14514284786278117030  # std::mt19937_64 default-seed first output


def test_config1_geometry():
    s = configs.config1()
    assert s.n == (64, 64, 64) and s.n_orbitals == 5 and s.max_inner == 50
    assert math.isclose(s.spacing[0], 20.0 / 65)
    o, h1, h2 = s.atoms
    assert o[:4] == (10.0, 10.0, 10.0, 8.0) and h1[3] == h2[3] == 1.0
    assert math.isclose(h1[0] - o[0], 1.43) and math.isclose(h2[0] - o[0], -1.43)


def test_cluster_configs_deterministic_and_valid():
    for fn, natoms, total, n_orb in ((configs.config2, 20, None, None), (configs.config3, 60, 256, 128),
                                     (configs.config4, 240, 1025, 512)):
        a, b = fn(), fn()
        assert a.atoms == b.atoms
        assert len(a.atoms) == natoms
        pos = np.array([x[:3] for x in a.atoms])
        d = np.sqrt(((pos[:, None] - pos[None]) ** 2).sum(-1)) + np.eye(natoms) * 1e9
        assert d.min() >= 2.0
        assert (pos > 0).all() and (pos < a.extent[0]).all()
        zsum = sum(x[3] for x in a.atoms)
        if total:
            assert zsum == total and a.n_orbitals == n_orb
        else:
            assert a.n_orbitals == (zsum + zsum % 2) // 2


def test_config5_potential_wells():
    s = configs.config5(64, 64)
    assert len(s.wells) == 32 and s.extent[0] == 20.0
    assert all(-5.0 <= w[3] <= 0.0 and w[4] == 2.0 for w in s.wells)
