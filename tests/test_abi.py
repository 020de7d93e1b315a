"""The drop-in C ABI (include/parorb_gpu.h): the library loads on a host with
no GPU, exports every declared symbol, and its host-only entry points behave
like the reference (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "parorb_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(po_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(native):
    lib = C.CDLL(native.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding declares a signature for every exported symbol
    assert set(native.EXPORTED_SYMBOLS) <= set(names)
    assert set(names) <= set(native.EXPORTED_SYMBOLS), set(names) - set(native.EXPORTED_SYMBOLS)


def test_default_params_match_reference(native):
    """OptimizerParams defaults, include/parorb/optimizer.hpp:22-46."""
    p = native.default_params()
    assert p.algorithm == native.ALGORITHMS["opt_par_mod"]
    assert (p.rho1, p.delta, p.eta) == (1e-4, 0.1, 0.85)
    assert (p.n_diag, p.n_org, p.max_inner, p.max_backtracks) == (100, 1, 10000, 20)
    assert (p.tau_min, p.tau_max, p.grad_tol) == (1e-10, 1e3, 1e-6)
    assert (p.mean_abs_tol, p.energy_tol) == (5e-9, 1e-13)
    assert p.verify_orthonormality == 1 and p.hartree == 1 and p.xc == 1
    assert p.poisson_solver == native.POISSON["dst"]


def test_abi_version_and_sizing(native):
    L = native.lib()
    assert L.po_abi_version() == 3
    g = native.GridDesc((C.c_int64 * 3)(192, 192, 192), (C.c_double * 3)(60.0, 60.0, 60.0))
    one = L.po_solver_bytes(C.byref(g), 512, 1)
    eight = L.po_solver_bytes(C.byref(g), 512, 8)
    assert one > 180 * 2 ** 30 > eight > 0  # C4 does not fit one B200, fits 8


def test_null_handles_are_rejected(native):
    L = native.lib()
    assert L.po_synchronize(None) == native.PO_EINVAL
    assert L.po_destroy(None) == native.PO_OK
    assert L.po_last_error(None) == b"null engine"
    assert L.po_thread_group_create(0, C.byref(C.c_void_p())) == native.PO_EINVAL


@pytest.mark.parametrize("bad", [(0, 8, 8), (8, -1, 8)])
def test_create_validates_grid_without_gpu_work(native, bad):
    """grid.cpp:14-34 argument checks happen before any device call."""
    with pytest.raises(native.InvalidArgument):
        native.Engine(bad, (1.0, 1.0, 1.0), 2)


def test_result_struct_layout_matches_header(native):
    """po_result (include/parorb_gpu.h) as ctypes sees it: the SolveResult
    fields appended in ABI 2 sit after message[200]."""
    R = native.Result
    names = [f[0] for f in R._fields_]
    assert names[-4:] == ["checkpoints", "n_checkpoints", "drift_iterations", "n_drift"]
    assert R.checkpoints.offset > R.message.offset


@pytest.mark.parametrize("N,ng,off,cnt", [(3, 1001, 0, 1001), (3, 1001, 17, 300), (4, 999, 998, 1),
                                          (5, 7, 0, 3), (2, 10, 3, 7)])
def test_rank_slab_normals_are_the_reference_draw(port, native, N, ng, off, cnt):
    """rng.cu rng_normals_slab (host, no GPU): a rank's slab of the reference's
    Rng(seed) orbital-major draw (rng.hpp:13-41, tests/problems.hpp:59-68) is
    bit-identical to the full draw sliced, for odd row lengths (the Box-Muller
    spare crosses orbital rows) and slabs at either end."""
    lib = C.CDLL(native.LIB_PATH)
    f = getattr(lib, "_ZN2po16rng_normals_slabEmilllPd")
    f.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
    import numpy as np
    ref = port.random_normals(42, N * ng).reshape(N, ng)[:, off:off + cnt]
    out = np.empty((N, cnt))
    f(42, N, ng, off, cnt, out.ctypes.data)
    assert np.array_equal(out, ref)
