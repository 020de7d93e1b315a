"""Slab-sharded engine with several ranks in one process on one
GPU (PO_COMM_THREADS: one host thread per rank; halo planes, Gram and scalar
all-reduces and the Poisson RHS all-gather are host-synchronised copies, so no
kernel waits on another rank). Every rank's result must match the
single-domain oracle: the decomposition changes results only at round-off."""
import threading

import numpy as np
import pytest

from paper_1510_07230_b200 import configs
from helpers import projector_distance

pytestmark = pytest.mark.gpu


def run_ranks(native, spec, size, body):
    grp = native.thread_group(size)
    out = [None] * size
    errs = []

    def worker(r):
        try:
            e = native.engine_for(spec, r, size, native.PO_COMM_THREADS, grp, device=0)
            out[r] = body(e, r)
            e.close()
        except Exception as ex:  # surfaced below
            errs.append(ex)

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    native.thread_group_destroy(grp)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("size", [2, 3])
def test_sharded_operators(port, native, size):
    spec = configs.small_molecule(14, 4, L=8.0)
    u0 = port.random_orthonormal(spec)
    plane = spec.n[1] * spec.n[2]
    st = port.build_hamiltonian(spec, u0)
    hu_ref = port.apply_hamiltonian(spec, st["v_local"], u0)
    g_ref = port.gram(spec, u0, u0, same=True)
    en_ref, kin_ref, _ = port.total_energy(spec, u0, st)

    def body(e, r):
        sl = slice(e.z0 * plane, (e.z0 + e.nz) * plane)
        u = e.block_from(np.ascontiguousarray(u0[:, sl]))
        eh, exc, _ = e.build_hamiltonian(u)
        hu = e.alloc()
        sig, kin, ext = e.apply_hamiltonian(u, hu)
        return dict(sl=sl, vh=e.get_field(native.PO_VH), hu=e.download(hu), kin=kin,
                    gram=e.gram(u, u), eh=eh, exc=exc, tot=e.total_energy(u))

    res = run_ranks(native, spec, size, body)
    covered = np.zeros(spec.num_points, bool)
    for x in res:
        covered[x["sl"]] = True
        assert np.max(np.abs(x["vh"] - st["v_h"][x["sl"]])) < 1e-8 * np.abs(st["v_h"]).max()
        assert np.max(np.abs(x["hu"] - hu_ref[:, x["sl"]])) < 1e-10 * np.abs(hu_ref).max()
        assert np.allclose(x["kin"], kin_ref, rtol=1e-11)
        assert np.max(np.abs(x["gram"] - g_ref)) < 1e-13
        assert abs(x["tot"]["total"] - en_ref["total"]) < 1e-9
    assert covered.all()
    # all ranks hold identical replicated quantities (bitwise)
    for x in res[1:]:
        assert np.array_equal(x["gram"], res[0]["gram"]) and x["eh"] == res[0]["eh"]


@pytest.mark.parametrize("size", [2, 3])
def test_sharded_solver(port, native, size):
    spec = configs.small_molecule(14, 4, L=8.0, max_inner=10)
    spec.algorithm = "opt_par"
    u0 = port.random_orthonormal(spec)
    ref = port.solve(spec, u0=u0, trace_eigs=False)
    plane = spec.n[1] * spec.n[2]

    def body(e, r):
        sl = slice(e.z0 * plane, (e.z0 + e.nz) * plane)
        w = e.block_from(np.ascontiguousarray(u0[:, sl]))
        got = e.solve(w, algorithm="opt_par", max_inner=10, n_org=1, n_diag=100)
        return dict(sl=sl, got=got, w=e.download(w))

    res = run_ranks(native, spec, size, body)
    w = np.zeros_like(u0)
    for x in res:
        w[:, x["sl"]] = x["w"]
        assert len(x["got"].records) == len(ref["records"])
        for a, b in zip(x["got"].records, ref["records"]):
            assert abs(a["energy"] - b["energy"]) < 1e-6 and a["backtracks"] == b["backtracks"]
    assert projector_distance(ref["w"], w, np.prod(spec.spacing)) < 1e-6
