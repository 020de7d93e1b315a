"""ctypes wrapper over the C restatement (oracle/port/parorb_port.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
bench's CPU-baseline legs — never by the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libparorb_port.so")
_lib = None

ALGORITHMS = {"optm_qr": 0, "opt_par": 1, "opt_par_mod": 2}
OUTCOMES = {0: "converged", 1: "max_iterations", 2: "stagnation", 3: "numerical_failure"}


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_int64 * 3), ("ext", C.c_double * 3),
                ("h", C.c_double * 3), ("w", C.c_double), ("ng", C.c_int64)]


class Atom(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("charge", C.c_double), ("softening", C.c_double)]


class Params(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("bb_variant", C.c_int), ("bb_trace_abs", C.c_int),
                ("convergence_mode", C.c_int), ("rho1", C.c_double), ("delta", C.c_double),
                ("eta", C.c_double), ("n_diag", C.c_int), ("n_org", C.c_int),
                ("max_inner", C.c_int), ("max_backtracks", C.c_int), ("tau_min", C.c_double),
                ("tau_max", C.c_double), ("grad_tol", C.c_double), ("mean_abs_tol", C.c_double),
                ("energy_tol", C.c_double), ("verify_orthonormality", C.c_int)]


class Record(C.Structure):
    _fields_ = [("level", C.c_int), ("iter", C.c_int), ("energy", C.c_double),
                ("grad_norm", C.c_double), ("tau", C.c_double), ("backtracks", C.c_int),
                ("did_orth", C.c_int), ("did_diag", C.c_int), ("offdiag_max", C.c_double)]


class State(C.Structure):
    _fields_ = [("rho", C.POINTER(C.c_double)), ("v_h", C.POINTER(C.c_double)),
                ("v_xc", C.POINTER(C.c_double)), ("v_local", C.POINTER(C.c_double)),
                ("cg_iters", C.c_int)]


class Result(C.Structure):
    _fields_ = [("cap", C.c_int), ("records", C.POINTER(Record)), ("accepted", C.POINTER(C.c_double)),
                ("sigma_eigs", C.POINTER(C.c_double)), ("w_out", C.POINTER(C.c_double)),
                ("n_records", C.c_int), ("n_accepted", C.c_int), ("outcome", C.c_int),
                ("cg_iters_total", C.c_int), ("e_kinetic", C.c_double), ("e_external", C.c_double),
                ("e_hartree", C.c_double), ("e_xc", C.c_double), ("e_total", C.c_double),
                ("final_grad_norm", C.c_double), ("message", C.c_char * 200)]


def build() -> str:
    """Compile the C restatement (no /root/reference needed)."""
    subprocess.run(["make", "-s", "-C", _HERE, "port"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.pp_pairwise_dot.restype = C.c_double
        _lib.pp_pairwise_dot.argtypes = [C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib.pp_pairwise_sum.restype = C.c_double
        _lib.pp_pairwise_sum.argtypes = [C.c_int64, C.POINTER(C.c_double)]
        _lib.pp_xc_energy_density.argtypes = [C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib.pp_xc_potential.argtypes = [C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib.pp_rng_normals.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
    return _lib


def pairwise_dot(a: np.ndarray, b: np.ndarray) -> float:
    """numeric.hpp:30-34 stable_dot."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return lib().pp_pairwise_dot(a.size, _dp(a), _dp(b))


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def make_grid(n, extent) -> Grid:
    g = Grid()
    nn = (C.c_int64 * 3)(*[int(x) for x in n])
    ee = (C.c_double * 3)(*[float(x) for x in extent])
    rc = lib().pp_grid_init(C.byref(g), len(n), nn, ee)
    if rc:
        raise ValueError("invalid grid")
    return g


def external_potential(spec) -> np.ndarray:
    g = make_grid(spec.n, spec.extent)
    atoms = (Atom * max(1, len(spec.atoms)))()
    for i, a in enumerate(spec.atoms):
        atoms[i].pos[:] = a[:3]
        atoms[i].charge = a[3]
        atoms[i].softening = a[4]
    v = np.zeros(g.ng)
    lib().pp_external_potential(C.byref(g), atoms, len(spec.atoms), _dp(v))
    return v


def random_normals(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().pp_rng_normals(C.c_uint64(seed), C.c_int64(count), _dp(out))
    return out


def orthonormalize(spec, block: np.ndarray, measure: bool = True):
    g = make_grid(spec.n, spec.extent)
    n = block.shape[0]
    block = np.ascontiguousarray(block, dtype=np.float64)
    out = np.empty_like(block)
    pre = np.empty((n, n))
    dev = C.c_double(0)
    fb = C.c_int(0)
    rc = lib().pp_orthonormalize(C.byref(g), n, _dp(block), int(measure), _dp(out), _dp(pre),
                                 C.byref(dev), C.byref(fb))
    if rc:
        raise RuntimeError(f"orthonormalize failed rc={rc}")
    return out, pre, dev.value, bool(fb.value)


def random_orthonormal(spec, seed: int | None = None) -> np.ndarray:
    """tests/problems.hpp:59-68 restated: Rng(seed) normals orbital-major, then Orth."""
    seed = spec.start_seed if seed is None else seed
    u = random_normals(seed, spec.n_orbitals * spec.num_points).reshape(spec.n_orbitals, -1)
    return orthonormalize(spec, u)[0]


def laplacian(spec, f: np.ndarray) -> np.ndarray:
    g = make_grid(spec.n, spec.extent)
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.empty_like(f)
    lib().pp_laplacian(C.byref(g), _dp(f), _dp(out))
    return out


def build_hamiltonian(spec, u: np.ndarray, v_ext: np.ndarray | None = None):
    g = make_grid(spec.n, spec.extent)
    if v_ext is None:
        v_ext = external_potential(spec)
    u = np.ascontiguousarray(u)
    bufs = {k: np.zeros(g.ng) for k in ("rho", "v_h", "v_xc", "v_local")}
    st = State(_dp(bufs["rho"]), _dp(bufs["v_h"]), _dp(bufs["v_xc"]), _dp(bufs["v_local"]), 0)
    rc = lib().pp_build_hamiltonian(C.byref(g), u.shape[0], _dp(u), _dp(v_ext), int(spec.hartree),
                                    int(spec.xc), C.c_double(spec.occupation), C.byref(st))
    if rc:
        raise RuntimeError(f"build_hamiltonian rc={rc}")
    bufs["cg_iters"] = st.cg_iters
    bufs["v_ext"] = v_ext
    bufs["_state"] = st
    return bufs


def apply_hamiltonian(spec, v_local: np.ndarray, u: np.ndarray) -> np.ndarray:
    g = make_grid(spec.n, spec.extent)
    u = np.ascontiguousarray(u)
    hu = np.empty_like(u)
    lib().pp_apply_hamiltonian(C.byref(g), _dp(v_local), u.shape[0], _dp(u), _dp(hu))
    return hu


def total_energy(spec, u: np.ndarray, state: dict):
    g = make_grid(spec.n, spec.extent)
    n = u.shape[0]
    out = np.zeros(5)
    kin = np.zeros(n)
    ext = np.zeros(n)
    lib().pp_total_energy(C.byref(g), n, _dp(np.ascontiguousarray(u)), _dp(state["v_ext"]),
                          C.byref(state["_state"]), int(spec.hartree), int(spec.xc),
                          C.c_double(spec.occupation), _dp(out), _dp(kin), _dp(ext))
    return dict(zip(("kinetic", "external", "hartree", "xc", "total"), out)), kin, ext


def gram(spec, a: np.ndarray, b: np.ndarray, same: bool = False) -> np.ndarray:
    g = make_grid(spec.n, spec.extent)
    n = a.shape[0]
    out = np.empty((n, n))
    lib().pp_gram(C.byref(g), n, _dp(np.ascontiguousarray(a)), _dp(np.ascontiguousarray(b)),
                  int(same), _dp(out))
    return out


def subspace_rotate(sigma: np.ndarray):
    n = sigma.shape[0]
    gam = np.empty(n)
    p = np.empty((n, n))
    rc = lib().pp_subspace_rotate(n, _dp(np.ascontiguousarray(sigma)), _dp(gam), _dp(p))
    if rc:
        raise ValueError("subspace_rotate: Sigma asymmetry exceeds tolerance")
    return gam, p


def default_params(**over) -> Params:
    p = Params()
    lib().pp_default_params(C.byref(p))
    conv = {"grad_norm": 0, "mean_abs": 1, "energy_change": 2}
    bbv = {"bb1": 0, "bb2": 1, "alternate": 2}
    for k, v in over.items():
        if k == "algorithm":
            v = ALGORITHMS[v]
        elif k == "convergence_mode":
            v = conv[v]
        elif k == "bb_variant":
            v = bbv[v]
        elif k == "bb_trace_abs":
            v = 1 if v == "abs_trace" else 0
        elif k == "verify_orthonormality":
            v = int(v)
        setattr(p, k, v)
    return p


def solve(spec, u0: np.ndarray | None = None, v_ext: np.ndarray | None = None,
          trace_eigs: bool = True, **param_over):
    """pp_solve = run_single_level (optimizer.cpp:599-613) for spec.algorithm."""
    g = make_grid(spec.n, spec.extent)
    if u0 is None:
        u0 = random_orthonormal(spec)
    if v_ext is None:
        v_ext = external_potential(spec)
    kw = dict(spec.optimizer_params())
    kw.update(param_over)
    kw["algorithm"] = spec.algorithm
    p = default_params(**kw)
    n = spec.n_orbitals
    cap = p.max_inner + 1
    recs = (Record * cap)()
    acc = np.zeros(cap * 9)
    eigs = np.full(cap * n, np.nan)
    w_out = np.empty_like(u0)
    r = Result()
    r.cap = cap
    r.records = recs
    r.accepted = _dp(acc)
    r.sigma_eigs = _dp(eigs) if trace_eigs else C.POINTER(C.c_double)()
    r.w_out = _dp(w_out)
    rc = lib().pp_solve(C.byref(g), n, _dp(v_ext), int(spec.hartree), int(spec.xc),
                        C.c_double(spec.occupation), C.byref(p), _dp(np.ascontiguousarray(u0)),
                        C.byref(r))
    if rc:
        raise RuntimeError(f"pp_solve rc={rc}: {r.message.decode()}")
    records = [dict(level=x.level, iter=x.iter, energy=x.energy, grad_norm=x.grad_norm, tau=x.tau,
                    backtracks=x.backtracks, did_orth=x.did_orth, did_diag=x.did_diag,
                    offdiag_max=x.offdiag_max) for x in recs[: r.n_records]]
    return dict(records=records,
                accepted=acc[: 9 * r.n_accepted].reshape(-1, 9),
                sigma_eigs=eigs[: n * r.n_records].reshape(-1, n),
                w=w_out,
                outcome=OUTCOMES[r.outcome],
                message=r.message.decode(),
                energy=dict(kinetic=r.e_kinetic, external=r.e_external, hartree=r.e_hartree,
                            xc=r.e_xc, total=r.e_total),
                final_grad_norm=r.final_grad_norm,
                cg_iters_total=r.cg_iters_total)


def format_log_row(r: dict) -> str:
    """driver.cpp:136-142 with wall_ms zeroed."""
    return "%d,%d,%s,%s,%s,%d,%d,%d,%s,0.000" % (
        r["level"], r["iter"], _g17(r["energy"]), _g17(r["grad_norm"]), _g17(r["tau"]),
        r["backtracks"], r["did_orth"], r["did_diag"], _g17(r["offdiag_max"]))


def _g17(x: float) -> str:
    return "%.17g" % x
