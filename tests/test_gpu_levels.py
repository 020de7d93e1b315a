"""Outer refinement on the GPU (optimizer.cpp:638-669, grid.cpp:137-212,
optimizer.cpp:156-197) against fixtures of the unmodified reference."""
import json
import os

import numpy as np
import pytest

from paper_1510_07230_b200 import configs

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _spec(name):
    meta = json.load(open(os.path.join(GOLDEN, name + ".json")))
    return meta, configs.ProblemSpec(**{k: (tuple(v) if k in ("n", "extent") else v)
                                        for k, v in meta["spec"].items()})


@pytest.mark.parametrize("name", ["prolong_init_mol8", "prolong_skew"])
def test_prolongate_bitwise(native, name):
    meta, spec = _spec(name)
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    coarse = native.engine_for(spec)
    nf, ext = native.refine_grid(spec.n, spec.extent)
    fine = native.Engine(nf, ext, spec.n_orbitals)
    cb, fb = coarse.block_from(g["u0"]), fine.alloc()
    coarse.prolongate(cb, fine, fb)
    assert np.array_equal(fine.download(fb), g["prolong"])
    coarse.close()
    fine.close()


def test_prolongate_rejects_non_refined(native):
    a = native.Engine((5, 5, 5), (4.0, 4.0, 4.0), 2)
    b = native.Engine((10, 11, 11), (4.0, 4.0, 4.0), 2)
    with pytest.raises(native.InvalidArgument):
        a.prolongate(a.alloc(), b, b.alloc())
    a.close()
    b.close()


def test_initialize_orbitals(native):
    meta, spec = _spec("prolong_init_mol8")
    u0 = np.load(os.path.join(GOLDEN, "prolong_init_mol8.npz"))["u0"]
    e = native.engine_for(spec)
    w = e.alloc()
    e.initialize_orbitals(spec.atoms, meta["start"]["seed"], w)
    got = e.download(w)
    # exp() differs from the host libm by at most an ulp; the Rng draws are the reference's bits
    assert np.abs(got - u0).max() < 1e-12
    e.close()


def test_solve_levels_vs_reference(native):
    meta, spec = _spec("levels_mol8")
    res, e, blk = native.solve_levels(spec, meta["outer_levels"], meta["seed"], algorithm=spec.algorithm,
                                      **spec.optimizer_params())
    ref = meta["records"]
    assert [(r["level"], r["iter"]) for r in res.records] == [(r["level"], r["iter"]) for r in ref]
    for a, b in zip(res.records, ref):
        assert abs(a["energy"] - float(b["energy"])) < 1e-8
        assert a["backtracks"] == b["backtracks"]
    assert res.outcome == meta["summary"]["outcome"]
    assert abs(res.energy["total"] - meta["summary"]["energy"]["total"]) < 1e-8
    assert abs(res.final_grad_norm - meta["summary"]["final_grad_norm"]) < 1e-6
    w_ref = np.load(os.path.join(GOLDEN, "levels_mol8_w.npz"))["w"]
    w = e.download(blk)
    assert w.shape == w_ref.shape
    wq = np.prod([L / (n + 1) for L, n in zip(e.extent, e.n)])
    m = wq * w_ref @ w.T  # <W_ref^T W>
    assert np.sqrt(2.0) * np.linalg.norm(np.sqrt(wq) * (w - m.T @ w_ref)) < 1e-6  # projector distance
    e.close()
