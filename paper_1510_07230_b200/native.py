"""ctypes binding of the C ABI (include/parorb_gpu.h) and a thin Python mirror
of the reference operator / solver API (energy.hpp, manifold.hpp,
optimizer.hpp). Every call goes to the sm_100a kernels in libparorb_b200.so;
there is no CPU fallback — a missing library or GPU raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libparorb_b200.so")
_lib = None

PO_OK, PO_EINVAL, PO_EDEGENERATE, PO_ESOLVER, PO_ESTAGNATION, PO_ECUDA, PO_ENCCL, PO_ENOMEM = range(8)
PO_VEXT, PO_RHO, PO_VH, PO_VXC, PO_VLOCAL = range(5)
PO_COMM_NONE, PO_COMM_NCCL, PO_COMM_THREADS = range(3)
ALGORITHMS = {"optm_qr": 0, "opt_par": 1, "opt_par_mod": 2}
OUTCOMES = {0: "converged", 1: "max_iterations", 2: "stagnation", 3: "numerical_failure"}
CONVERGENCE = {"grad_norm": 0, "mean_abs": 1, "energy_change": 2}
BB = {"bb1": 0, "bb2": 1, "alternate": 2}
POISSON = {"cg": 0, "cg_warm": 1, "dst": 2}


class InvalidArgument(ValueError):
    """errors.hpp:13 InvalidArgument."""


class DegenerateSetError(RuntimeError):
    """errors.hpp:19 DegenerateSetError."""


class SolverError(RuntimeError):
    """errors.hpp:36 SolverError."""


class StagnationError(RuntimeError):
    """errors.hpp:25 StagnationError."""


class DeviceError(RuntimeError):
    """CUDA / NCCL / allocation failure (no reference counterpart)."""


_ERRORS = {PO_EINVAL: InvalidArgument, PO_EDEGENERATE: DegenerateSetError, PO_ESOLVER: SolverError,
           PO_ESTAGNATION: StagnationError}


class GridDesc(C.Structure):
    _fields_ = [("n", C.c_int64 * 3), ("extent", C.c_double * 3)]


class DistDesc(C.Structure):
    _fields_ = [("rank", C.c_int), ("size", C.c_int), ("kind", C.c_int), ("handle", C.c_void_p),
                ("device", C.c_int)]


class Params(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("bb_variant", C.c_int), ("bb_trace_abs", C.c_int),
                ("convergence_mode", C.c_int), ("rho1", C.c_double), ("delta", C.c_double),
                ("eta", C.c_double), ("n_diag", C.c_int), ("n_org", C.c_int), ("max_inner", C.c_int),
                ("max_backtracks", C.c_int), ("tau_min", C.c_double), ("tau_max", C.c_double),
                ("grad_tol", C.c_double), ("mean_abs_tol", C.c_double), ("energy_tol", C.c_double),
                ("verify_orthonormality", C.c_int), ("hartree", C.c_int), ("xc", C.c_int),
                ("trace_sigma_eigs", C.c_int), ("poisson_solver", C.c_int), ("outer_levels", C.c_int),
                ("seed", C.c_uint64)]


class Record(C.Structure):
    _fields_ = [("level", C.c_int), ("iter", C.c_int), ("energy", C.c_double),
                ("grad_norm", C.c_double), ("tau", C.c_double), ("backtracks", C.c_int),
                ("did_orth", C.c_int), ("did_diag", C.c_int), ("offdiag_max", C.c_double),
                ("wall_ms", C.c_double)]


class Result(C.Structure):
    _fields_ = [("cap", C.c_int), ("records", C.POINTER(Record)), ("accepted", C.POINTER(C.c_double)),
                ("sigma_eigs", C.POINTER(C.c_double)), ("n_records", C.c_int), ("n_accepted", C.c_int),
                ("outcome", C.c_int), ("cg_iters_total", C.c_int64), ("e_kinetic", C.c_double),
                ("e_external", C.c_double), ("e_hartree", C.c_double), ("e_xc", C.c_double),
                ("e_total", C.c_double), ("final_grad_norm", C.c_double), ("wall_seconds", C.c_double),
                ("par_seconds", C.c_double), ("sync_seconds", C.c_double), ("message", C.c_char * 200),
                ("checkpoints", C.POINTER(C.c_double)), ("n_checkpoints", C.c_int),
                ("drift_iterations", C.POINTER(C.c_int)), ("n_drift", C.c_int)]


def _new_result(cap: int, n: int, trace_eigs: bool = False):
    """A po_result with every output array allocated (kept alive in the dict)."""
    keep = {"recs": (Record * cap)(), "acc": np.zeros(cap * 9), "ckpt": np.zeros(cap * 5),
            "drift": np.zeros(cap, dtype=np.int32),
            "eigs": np.full(cap * n, np.nan) if trace_eigs else np.zeros(1)}
    r = Result()
    r.cap = cap
    r.records = keep["recs"]
    r.accepted = keep["acc"].ctypes.data_as(C.POINTER(C.c_double))
    r.sigma_eigs = (keep["eigs"].ctypes.data_as(C.POINTER(C.c_double)) if trace_eigs
                    else C.POINTER(C.c_double)())
    r.checkpoints = keep["ckpt"].ctypes.data_as(C.POINTER(C.c_double))
    r.drift_iterations = keep["drift"].ctypes.data_as(C.POINTER(C.c_int))
    return r, keep


_SIGS = {
    "po_abi_version": ([], C.c_int),
    "po_create": ([C.POINTER(GridDesc), C.c_int, C.c_double, C.POINTER(DistDesc), C.POINTER(C.c_void_p)], C.c_int),
    "po_destroy": ([C.c_void_p], C.c_int),
    "po_last_error": ([C.c_void_p], C.c_char_p),
    "po_local_slab": ([C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "po_solver_bytes": ([C.POINTER(GridDesc), C.c_int, C.c_int], C.c_int64),
    "po_slab_plan": ([C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                      C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "po_stream": ([C.c_void_p], C.c_void_p),
    "po_synchronize": ([C.c_void_p], C.c_int),
    "po_thread_group_create": ([C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "po_thread_group_destroy": ([C.c_void_p], C.c_int),
    "po_alloc_block": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "po_free_block": ([C.c_void_p, C.c_int], C.c_int),
    "po_upload_block": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "po_download_block": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "po_copy_block": ([C.c_void_p, C.c_int, C.c_int], C.c_int),
    "po_set_field": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "po_get_field": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "po_external_potential": ([C.c_void_p, C.c_void_p, C.c_int], C.c_int),
    "po_gaussian_potential": ([C.c_void_p, C.c_void_p, C.c_int], C.c_int),
    "po_random_block": ([C.c_void_p, C.c_int, C.c_uint64], C.c_int),
    "po_fill_normal": ([C.c_void_p, C.c_int, C.c_uint64], C.c_int),
    "po_build_hamiltonian": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                              C.POINTER(C.c_double), C.POINTER(C.c_int)], C.c_int),
    "po_apply_hamiltonian": ([C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "po_total_energy": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p], C.c_int),
    "po_laplacian": ([C.c_void_p, C.c_int, C.c_int], C.c_int),
    "po_gram": ([C.c_void_p, C.c_int, C.c_int, C.c_void_p], C.c_int),
    "po_gram_lincomb": ([C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_void_p], C.c_int),
    "po_mix": ([C.c_void_p, C.c_int, C.c_void_p, C.c_int], C.c_int),
    "po_orthonormalize": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_double),
                           C.POINTER(C.c_int)], C.c_int),
    "po_diagonal_residuals": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "po_stiefel_gradient": ([C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "po_stiefel_gradient_d": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "po_subspace_rotate": ([C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "po_linear_combination": ([C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int], C.c_int),
    "po_direction_sums": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "po_bb_products": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                        C.c_void_p], C.c_int),
    "po_default_params": ([C.POINTER(Params)], None),
    "po_solve": ([C.c_void_p, C.POINTER(Params), C.c_int, C.POINTER(Result)], C.c_int),
    "po_solve_host": ([C.c_void_p, C.POINTER(Params), C.c_void_p, C.c_void_p, C.POINTER(Result)], C.c_int),
    "po_solver_create": ([C.c_void_p, C.POINTER(Params), C.c_int, C.POINTER(Result), C.POINTER(C.c_void_p)], C.c_int),
    "po_solver_step": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "po_solver_current": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "po_solver_finish": ([C.c_void_p], C.c_int),
    "po_solver_destroy": ([C.c_void_p], C.c_int),
    "po_launch_count": ([], C.c_longlong),
    "po_enqueue": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int], C.c_int),
    "po_set_matrix": ([C.c_void_p, C.c_void_p], C.c_int),
    "po_nccl_unique_id": ([C.c_void_p], C.c_int),
    "po_set_poisson_solver": ([C.c_void_p, C.c_int], C.c_int),
    "po_initialize_orbitals": ([C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_int], C.c_int),
    "po_refine_grid": ([C.POINTER(GridDesc), C.POINTER(GridDesc)], C.c_int),
    "po_prolongate": ([C.c_void_p, C.c_int, C.c_void_p, C.c_int], C.c_int),
    "po_solve_levels": ([C.POINTER(GridDesc), C.c_int, C.c_double, C.c_void_p, C.c_int, C.POINTER(Params),
                         C.POINTER(Result), C.POINTER(C.c_void_p), C.POINTER(C.c_int)], C.c_int),
    "po_format_log_row": ([C.POINTER(Record), C.c_char_p, C.c_int], C.c_int),
    "po_write_log": ([C.c_char_p, C.POINTER(Record), C.c_int, C.c_int], C.c_int),
    "po_write_reduction": ([C.c_char_p, C.POINTER(Record), C.c_int, C.c_double], C.c_int),
}

OPS = dict(hamiltonian=0, gram_sym=1, gram=2, mix=3, mix_upper=4, density_xc=5, poisson=6, cholesky=7,
           laplacian=8, gram_trial=9, rotation=10, directions=11, rotation_fused=12, rotation_implicit=13, gram_sigma_bb=14, gram_density=15)

EXPORTED_SYMBOLS = tuple(_SIGS)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _PKG, "-j8"], check=True)
    return LIB_PATH


def lib():
    """Load libparorb_b200.so (raises if it is missing — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `make -C {_PKG}` (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise InvalidArgument("arrays must be C-contiguous float64")
    return a.ctypes.data_as(C.c_void_p)


class Engine:
    """One rank's device-resident state (po_engine)."""

    def __init__(self, n, extent, n_orbitals: int, occupation: float = 1.0, rank: int = 0,
                 size: int = 1, comm_kind: int = PO_COMM_NONE, comm_handle=None, device: int = -1):
        L = lib()
        self._lib = L
        g = GridDesc((C.c_int64 * 3)(*[int(x) for x in n]), (C.c_double * 3)(*[float(x) for x in extent]))
        self._keep = comm_handle
        if isinstance(comm_handle, (bytes, bytearray)):
            self._hbuf = C.create_string_buffer(bytes(comm_handle), len(comm_handle))
            handle = C.cast(self._hbuf, C.c_void_p)
        else:
            handle = comm_handle
        d = DistDesc(rank, size, comm_kind, handle, device)
        h = C.c_void_p()
        rc = L.po_create(C.byref(g), int(n_orbitals), float(occupation), C.byref(d), C.byref(h))
        self.h = h
        if rc != PO_OK:
            msg = L.po_last_error(h).decode() if h else "po_create failed"
            L.po_destroy(h)
            self.h = None
            raise _err(rc, msg)
        self.n = tuple(int(x) for x in n)
        self.extent = tuple(float(x) for x in extent)
        self.N = int(n_orbitals)
        self.occupation = float(occupation)
        z0, nz, ngl = C.c_int64(), C.c_int64(), C.c_int64()
        L.po_local_slab(h, C.byref(z0), C.byref(nz), C.byref(ngl))
        self.z0, self.nz, self.ngl = z0.value, nz.value, ngl.value

    def close(self):
        if self.h:
            self._lib.po_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        if rc != PO_OK:
            raise _err(rc, self._lib.po_last_error(self.h).decode())

    @property
    def stream(self) -> int:
        return self._lib.po_stream(self.h) or 0

    def synchronize(self):
        self._chk(self._lib.po_synchronize(self.h))

    # ---- blocks
    def alloc(self) -> int:
        b = C.c_int()
        self._chk(self._lib.po_alloc_block(self.h, C.byref(b)))
        return b.value

    def free(self, b: int):
        self._chk(self._lib.po_free_block(self.h, b))

    def upload(self, b: int, host: np.ndarray):
        host = np.ascontiguousarray(host, dtype=np.float64)
        if host.size != self.N * self.ngl:
            raise InvalidArgument("block shape mismatch")
        self._chk(self._lib.po_upload_block(self.h, b, _dp(host)))

    def download(self, b: int, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.N, self.ngl))
        self._chk(self._lib.po_download_block(self.h, b, _dp(out)))
        return out

    def block_from(self, host: np.ndarray) -> int:
        b = self.alloc()
        self.upload(b, host)
        return b

    def copy(self, dst: int, src: int):
        self._chk(self._lib.po_copy_block(self.h, dst, src))

    def random_block(self, b: int, seed: int):
        self._chk(self._lib.po_random_block(self.h, b, C.c_uint64(seed)))

    def fill_normal(self, b: int, seed: int):
        """po_fill_normal: device counter-hash N(0,1) fill (measurement blocks)."""
        self._chk(self._lib.po_fill_normal(self.h, b, C.c_uint64(seed)))

    # ---- fields
    def set_field(self, f: int, host: np.ndarray):
        self._chk(self._lib.po_set_field(self.h, f, _dp(np.ascontiguousarray(host, dtype=np.float64))))

    def get_field(self, f: int) -> np.ndarray:
        out = np.empty(self.ngl)
        self._chk(self._lib.po_get_field(self.h, f, _dp(out)))
        return out

    def external_potential(self, atoms):
        a = np.ascontiguousarray(np.asarray(atoms, dtype=np.float64).reshape(-1, 5))
        self._chk(self._lib.po_external_potential(self.h, _dp(a) if a.size else None, a.shape[0]))

    def gaussian_potential(self, wells):
        a = np.ascontiguousarray(np.asarray(wells, dtype=np.float64).reshape(-1, 5))
        self._chk(self._lib.po_gaussian_potential(self.h, _dp(a), a.shape[0]))

    # ---- operators
    def build_hamiltonian(self, u: int, hartree=True, xc=True):
        eh, exc, it = C.c_double(), C.c_double(), C.c_int()
        self._chk(self._lib.po_build_hamiltonian(self.h, u, int(hartree), int(xc), C.byref(eh),
                                                 C.byref(exc), C.byref(it)))
        return eh.value, exc.value, it.value

    def apply_hamiltonian(self, u: int, out: int = -1):
        s, k, e = np.empty(self.N), np.empty(self.N), np.empty(self.N)
        self._chk(self._lib.po_apply_hamiltonian(self.h, u, out, _dp(s), _dp(k), _dp(e)))
        return s, k, e

    def total_energy(self, u: int, hartree=True, xc=True) -> dict:
        out = np.empty(5)
        self._chk(self._lib.po_total_energy(self.h, u, int(hartree), int(xc), _dp(out)))
        return dict(zip(("kinetic", "external", "hartree", "xc", "total"), out.tolist()))

    def laplacian(self, u: int, out: int):
        self._chk(self._lib.po_laplacian(self.h, u, out))

    def gram(self, a: int, b: int) -> np.ndarray:
        g = np.empty((self.N, self.N))
        self._chk(self._lib.po_gram(self.h, a, b, _dp(g)))
        return g

    def gram_lincomb(self, a: int, s: float, b: int) -> np.ndarray:
        g = np.empty((self.N, self.N))
        self._chk(self._lib.po_gram_lincomb(self.h, a, float(s), b, _dp(g)))
        return g

    def mix(self, inp: int, m: np.ndarray, out: int):
        self._chk(self._lib.po_mix(self.h, inp, _dp(np.ascontiguousarray(m, dtype=np.float64)), out))

    def orthonormalize(self, inp: int, out: int, measure: bool = True):
        pre = np.empty((self.N, self.N))
        dev, fb = C.c_double(), C.c_int()
        self._chk(self._lib.po_orthonormalize(self.h, inp, out, int(measure), _dp(pre), C.byref(dev),
                                              C.byref(fb)))
        return pre, dev.value, bool(fb.value)

    def diagonal_residuals(self, u: int, hu: int, z: int):
        s, zz = np.empty(self.N), np.empty(self.N)
        self._chk(self._lib.po_diagonal_residuals(self.h, u, hu, z, _dp(s), _dp(zz)))
        return s, zz

    def stiefel_gradient(self, u: int, hu: int, d: int = -1):
        """manifold.cpp:181-202: (Sigma, <D_i, D_i>); with d >= 0 the block D = HU - U Sigma
        is written there too (po_stiefel_gradient_d)."""
        sig, dd = np.empty((self.N, self.N)), np.empty(self.N)
        self._chk(self._lib.po_stiefel_gradient_d(self.h, u, hu, d, _dp(sig), _dp(dd)))
        return sig, dd

    def subspace_rotate(self, w: int, sigma: np.ndarray):
        gam, p = np.empty(self.N), np.empty((self.N, self.N))
        self._chk(self._lib.po_subspace_rotate(self.h, w, _dp(np.ascontiguousarray(sigma)), _dp(gam), _dp(p)))
        return gam, p

    def linear_combination(self, a: int, s: float, b: int, out: int):
        self._chk(self._lib.po_linear_combination(self.h, a, float(s), b, out))

    def bb_products(self, w: int, wp: int, z: int, zp: int):
        ss, sy, yy = np.empty(self.N), np.empty(self.N), np.empty(self.N)
        self._chk(self._lib.po_bb_products(self.h, w, wp, z, zp, _dp(ss), _dp(sy), _dp(yy)))
        return ss, sy, yy

    def direction_sums(self, u: int, hu: int, u_prev: int = -1, hu_prev: int = -1, sigma_prev=None):
        """po_direction_sums: sigma_ii, Sigma, ||z_i||^2 and (with a history) the BB products of
        the implicit directions z = HU - sigma U (optimizer.cpp:265-320, 386-397)."""
        n = self.N
        sd, sf = np.empty(n), np.empty((n, n))
        zz, ss, sy, yy = np.empty(n), np.empty(n), np.empty(n), np.empty(n)
        spv = None if sigma_prev is None else _dp(np.ascontiguousarray(sigma_prev, dtype=np.float64))
        self._chk(self._lib.po_direction_sums(self.h, u, hu, u_prev, hu_prev, spv, _dp(sd), _dp(sf),
                                              _dp(zz), _dp(ss), _dp(sy), _dp(yy)))
        out = dict(sigma_diag=sd, sigma=sf, zz=zz)
        if u_prev >= 0:
            out.update(ss=ss, sy=sy, yy=yy)
        return out

    # ---- measurement helpers (pure launches on self.stream, no sync)
    def enqueue(self, op: str, a: int = -1, b: int = -1, out: int = -1):
        self._chk(self._lib.po_enqueue(self.h, OPS[op], a, b, out))

    def set_poisson_solver(self, mode: str):
        self._chk(self._lib.po_set_poisson_solver(self.h, POISSON[mode]))

    def set_matrix(self, m: np.ndarray):
        self._chk(self._lib.po_set_matrix(self.h, _dp(np.ascontiguousarray(m, dtype=np.float64))))

    # ---- solver
    @staticmethod
    def make_params(algorithm="opt_par_mod", hartree=True, xc=True, trace_eigs=False, poisson="dst",
                    **over) -> Params:
        p = default_params()
        p.algorithm = ALGORITHMS[algorithm]
        p.hartree, p.xc = int(hartree), int(xc)
        p.trace_sigma_eigs = int(trace_eigs)
        p.poisson_solver = POISSON[poisson]
        for k, v in over.items():
            if k == "convergence_mode":
                v = CONVERGENCE[v]
            elif k == "bb_variant":
                v = BB[v]
            elif k == "bb_trace_abs":
                v = 1 if v == "abs_trace" else 0
            elif k == "verify_orthonormality":
                v = int(v)
            setattr(p, k, v)
        return p

    def solve(self, w: int, algorithm="opt_par_mod", hartree=True, xc=True, trace_eigs=False,
              poisson="dst", **over) -> "SolveResult":
        p = self.make_params(algorithm, hartree, xc, trace_eigs, poisson, **over)
        cap = p.max_inner + 1
        r, keep = _new_result(cap, self.N, trace_eigs)
        rc = self._lib.po_solve(self.h, C.byref(p), w, C.byref(r))
        if rc != PO_OK:
            raise _err(rc, self._lib.po_last_error(self.h).decode() or r.message.decode())
        return _solve_result(r, keep, cap, self.N, trace_eigs)

    def solve_host(self, w_in: np.ndarray, w_out: np.ndarray, algorithm="opt_par_mod", hartree=True,
                   xc=True, poisson="dst", **over) -> "SolveResult":
        """po_solve_host: host orbitals in, final orbitals out (pinned buffers are fastest)."""
        p = self.make_params(algorithm, hartree, xc, False, poisson, **over)
        cap = p.max_inner + 1
        r, keep = _new_result(cap, self.N)
        if w_in.size != self.N * self.ngl or w_out.size != self.N * self.ngl:
            raise InvalidArgument("block shape mismatch")
        rc = self._lib.po_solve_host(self.h, C.byref(p), _dp(w_in), _dp(w_out), C.byref(r))
        if rc != PO_OK:
            raise _err(rc, self._lib.po_last_error(self.h).decode() or r.message.decode())
        return _solve_result(r, keep, cap, self.N, False)

    # ---- outer refinement (optimizer.cpp:638-669, grid.cpp:137-212)
    def initialize_orbitals(self, atoms, seed: int, w: int):
        a = np.ascontiguousarray(np.asarray(atoms, dtype=np.float64).reshape(-1, 5))
        self._chk(self._lib.po_initialize_orbitals(self.h, _dp(a) if len(a) else None, len(a),
                                                   C.c_uint64(seed), w))

    def prolongate(self, cblock: int, fine: "Engine", fblock: int):
        rc = self._lib.po_prolongate(self.h, cblock, fine.h, fblock)
        if rc != PO_OK:
            raise _err(rc, self._lib.po_last_error(fine.h).decode())


class Stepper:
    """po_solver_* iterator: one InnerLoop iteration per step() (bench / callers that
    interleave work). Holds the engine's result struct alive."""

    def __init__(self, e: Engine, w: int, params: Params):
        self.e = e
        self.p = params
        cap = params.max_inner + 1
        self.r, self._keep = _new_result(cap, e.N, bool(params.trace_sigma_eigs))
        self._recs = self._keep["recs"]
        self.h = C.c_void_p()
        rc = e._lib.po_solver_create(e.h, C.byref(self.p), w, C.byref(self.r), C.byref(self.h))
        if rc != PO_OK:
            raise _err(rc, e._lib.po_last_error(e.h).decode())

    def step(self) -> bool:
        more = C.c_int()
        self.e._chk(self.e._lib.po_solver_step(self.h, C.byref(more)))
        return bool(more.value)

    def current(self) -> int:
        b = C.c_int()
        self.e._chk(self.e._lib.po_solver_current(self.h, C.byref(b)))
        return b.value

    def finish(self):
        self.e._chk(self.e._lib.po_solver_finish(self.h))

    def records(self):
        n = min(self.r.n_records, self.r.cap)
        return [dict(iter=x.iter, energy=x.energy, grad_norm=x.grad_norm, tau=x.tau, backtracks=x.backtracks,
                     did_orth=x.did_orth, wall_ms=x.wall_ms) for x in self._recs[:n]]

    def sigma_eigs(self) -> np.ndarray:
        """eig(<(HW)^T W>) per record (params.trace_sigma_eigs)."""
        n = min(self.r.n_records, self.r.cap)
        return self._keep["eigs"][: n * self.e.N].reshape(-1, self.e.N)

    def result(self) -> "SolveResult":
        return _solve_result(self.r, self._keep, self.r.cap, self.e.N, bool(self.p.trace_sigma_eigs))

    def close(self):
        if self.h:
            self.e._lib.po_solver_destroy(self.h)
            self.h = None


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = lib().po_nccl_unique_id(buf)
    if rc != PO_OK:
        raise DeviceError("ncclGetUniqueId failed")
    return buf.raw


def slab_plan(n0: int, size: int, rank: int):
    """po_slab_plan: the engine's own axis-0 partition (host only) -> (z0, nz, lo_peer, hi_peer)."""
    z0, nz, lo, hi = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
    rc = lib().po_slab_plan(int(n0), int(size), int(rank), C.byref(z0), C.byref(nz), C.byref(lo), C.byref(hi))
    if rc != PO_OK:
        raise InvalidArgument("slab_plan: invalid partition")
    return z0.value, nz.value, lo.value, hi.value


def thread_group(size: int) -> int:
    """po_thread_group for in-process ranks (PO_COMM_THREADS); returns the handle."""
    h = C.c_void_p()
    rc = lib().po_thread_group_create(int(size), C.byref(h))
    if rc != PO_OK:
        raise InvalidArgument("thread group")
    return h.value


def thread_group_destroy(h: int):
    lib().po_thread_group_destroy(C.c_void_p(h))


def launch_count() -> int:
    return int(lib().po_launch_count())


@dataclass
class SolveResult:
    """SolveResult, optimizer.hpp:98-112 (orbitals stay on the device)."""
    records: list
    accepted: np.ndarray
    sigma_eigs: np.ndarray | None
    outcome: str
    message: str
    energy: dict
    final_grad_norm: float
    cg_iters_total: int
    wall_seconds: float
    par_seconds: float = 0.0
    sync_seconds: float = 0.0
    checkpoints: list = field(default_factory=list)  # OrthCheckpoint rows (optimizer.hpp:87-93)
    drift_iterations: list = field(default_factory=list)
    extra: dict = field(default_factory=dict)


def _solve_result(r, keep, cap, N, trace_eigs) -> SolveResult:
    recs, acc, eigs = keep["recs"], keep["acc"], keep["eigs"]
    nrec = min(r.n_records, cap)
    ck = keep["ckpt"][: 5 * min(r.n_checkpoints, cap)].reshape(-1, 5)
    checkpoints = [dict(level=int(c[0]), iter=int(c[1]), offdiag_max=float(c[2]),
                        diag_deviation_max=float(c[3]), orth_deviation=float(c[4])) for c in ck]
    drift = [int(x) for x in keep["drift"][: min(r.n_drift, cap)]]
    records = [dict(level=x.level, iter=x.iter, energy=x.energy, grad_norm=x.grad_norm, tau=x.tau,
                    backtracks=x.backtracks, did_orth=x.did_orth, did_diag=x.did_diag,
                    offdiag_max=x.offdiag_max, wall_ms=x.wall_ms) for x in recs[:nrec]]
    return SolveResult(
        records=records, accepted=acc[: 9 * min(r.n_accepted, cap)].reshape(-1, 9),
        sigma_eigs=eigs[: N * nrec].reshape(-1, N) if trace_eigs else None,
        outcome=OUTCOMES[r.outcome], message=r.message.decode(),
        energy=dict(kinetic=r.e_kinetic, external=r.e_external, hartree=r.e_hartree, xc=r.e_xc,
                    total=r.e_total),
        final_grad_norm=r.final_grad_norm, cg_iters_total=r.cg_iters_total,
        wall_seconds=r.wall_seconds, par_seconds=r.par_seconds, sync_seconds=r.sync_seconds,
        checkpoints=checkpoints, drift_iterations=drift)


def refine_grid(n, extent):
    """grid.cpp:137-149 refine_uniform."""
    g = GridDesc((C.c_int64 * 3)(*[int(x) for x in n]), (C.c_double * 3)(*[float(x) for x in extent]))
    f = GridDesc()
    rc = lib().po_refine_grid(C.byref(g), C.byref(f))
    if rc != PO_OK:
        raise _err(rc, "refine_uniform: invalid grid")
    return tuple(f.n), tuple(f.extent)


def solve_levels(spec, outer_levels: int, seed: int, algorithm="opt_par_mod", poisson="dst",
                 **over):
    """optimizer.cpp:638-669 solve on the GPU: returns (SolveResult, final Engine, block)."""
    L = lib()
    p = Engine.make_params(algorithm, spec.hartree, spec.xc, False, poisson, **over)
    p.outer_levels, p.seed = int(outer_levels), int(seed)
    cap = outer_levels * p.max_inner + 1
    r, keep = _new_result(cap, spec.n_orbitals)
    g = GridDesc((C.c_int64 * 3)(*[int(x) for x in spec.n]),
                 (C.c_double * 3)(*[float(x) for x in spec.extent]))
    atoms = np.ascontiguousarray(np.asarray(spec.atoms, dtype=np.float64).reshape(-1, 5))
    h, blk = C.c_void_p(), C.c_int()
    rc = L.po_solve_levels(C.byref(g), spec.n_orbitals, float(spec.occupation),
                           _dp(atoms) if len(atoms) else None, len(atoms), C.byref(p), C.byref(r),
                           C.byref(h), C.byref(blk))
    if rc != PO_OK:
        msg = L.po_last_error(h).decode() if h else r.message.decode()
        if h:
            L.po_destroy(h)
        raise _err(rc, msg or r.message.decode())
    n = list(spec.n)
    for _ in range(outer_levels - 1):
        n = [2 * x + 1 for x in n]
    e = Engine.__new__(Engine)
    e._lib, e.h, e._keep = L, h, None
    e.n, e.extent, e.N, e.occupation = tuple(n), tuple(spec.extent), spec.n_orbitals, spec.occupation
    z0, nz, ngl = C.c_int64(), C.c_int64(), C.c_int64()
    L.po_local_slab(h, C.byref(z0), C.byref(nz), C.byref(ngl))
    e.z0, e.nz, e.ngl = z0.value, nz.value, ngl.value
    return _solve_result(r, keep, cap, spec.n_orbitals, False), e, blk.value


def _records_array(records):
    arr = (Record * len(records))()
    for k, x in enumerate(records):
        arr[k] = Record(x["level"], x["iter"], x["energy"], x["grad_norm"], x["tau"], x["backtracks"],
                        x["did_orth"], x["did_diag"], x["offdiag_max"], x["wall_ms"])
    return arr


def format_log_row(rec: dict) -> str:
    """driver.cpp:136-142 through the C ABI."""
    arr = _records_array([rec])
    buf = C.create_string_buffer(320)
    n = lib().po_format_log_row(arr, buf, 320)
    if n < 0:
        raise InvalidArgument("format_log_row: buffer too small")
    return buf.value.decode()


def write_log(path: str, records: list, log_every: int = 1):
    arr = _records_array(records)
    rc = lib().po_write_log(path.encode(), arr, len(records), int(log_every))
    if rc != PO_OK:
        raise _err(rc, f"cannot write {path}")


def write_reduction(path: str, records: list, e_min: float):
    arr = _records_array(records)
    rc = lib().po_write_reduction(path.encode(), arr, len(records), float(e_min))
    if rc != PO_OK:
        raise _err(rc, f"cannot write {path}")


def default_params() -> Params:
    p = Params()
    lib().po_default_params(C.byref(p))
    return p


def _err(rc: int, msg: str) -> Exception:
    cls = _ERRORS.get(rc, DeviceError)
    return cls(f"[{rc}] {msg}")


def engine_for(spec, rank: int = 0, size: int = 1, comm_kind: int = PO_COMM_NONE, comm_handle=None,
               device: int = -1) -> Engine:
    """Engine with the spec's grid, orbital count, occupation and V_ext."""
    e = Engine(spec.n, spec.extent, spec.n_orbitals, spec.occupation, rank, size, comm_kind, comm_handle,
               device)
    if spec.wells:
        e.gaussian_potential(spec.wells)
    else:
        e.external_potential(spec.atoms)
    return e


def random_orthonormal(e: Engine, seed: int) -> int:
    """tests/problems.hpp:59-68 on the device: Rng(seed) normals (the reference's exact
    bits), then Orth (Cholesky-QR on the device). Returns a block handle."""
    raw = e.alloc()
    e.random_block(raw, seed)
    w = e.alloc()
    e.orthonormalize(raw, w, True)
    e.free(raw)
    return w


def format_log_row(r: dict) -> str:
    """driver.cpp:136-142 with wall_ms zeroed."""
    g = lambda x: "%.17g" % x  # noqa: E731
    return "%d,%d,%s,%s,%s,%d,%d,%d,%s,0.000" % (r["level"], r["iter"], g(r["energy"]), g(r["grad_norm"]),
                                               g(r["tau"]), r["backtracks"], r["did_orth"], r["did_diag"],
                                               g(r["offdiag_max"]))
