"""Parity at the FULL BASELINE shapes against the UNMODIFIED reference.

The reference cannot hand over GB-sized blocks, so its side of these checks is
committed as size-independent fingerprints written by oracle/ref_harness/
trace_ref.cpp (oracle/make_golden.py --big):

* eig(Sigma) at EVERY accepted iterate of the 50-iteration C1 / C2 runs
  (C*_eigs.npz, from the C restatement whose log rows are byte-identical to
  the reference's trajectory);
* C2 and C3 prefixes (prefix_C*.json/.npz): truncated re-runs of
  opt_par_mod_inner with max_inner = 1..3 at 96^3 / N = 33 and 128^3 / N = 128
  — records, checkpoints, eig(Sigma) after every iteration, and a Rademacher
  sketch S = sqrt(w) W X of every iterate, from which ||P_gpu - P_ref||_F is
  estimated (tests/helpers.py sketch_projector_distance);
* every hot-path operator at the C3 shape (N = 128) and at the C4 grid
  (192^3, L = 60, the C4 nuclei) with N = 64 (opsr_*.json/.npz): fields at
  sampled points + norms, blocks as sampled rows + sketches, every N x N matrix.

Gates: energies and eigenvalues within 1e-6 Ha (north star), ||dP||_F <= 1e-6,
operators to the tolerances stated per check."""
import json
import os

import numpy as np
import pytest

from paper_1510_07230_b200 import configs
from helpers import sample_points, sketch_block, sketch_projector_distance

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-6


def _spec(d):
    d = dict(d)
    for k in ("n", "extent"):
        d[k] = tuple(d[k])
    d["atoms"] = [tuple(a) for a in d["atoms"]]
    return configs.ProblemSpec(**d)


def _checkpoints(csv):
    rows = csv.strip().split("\n")[1:]
    return [dict(level=int(f[0]), iter=int(f[1]), offdiag_max=float(f[2]), diag_deviation_max=float(f[3]),
                 orth_deviation=float(f[4])) for f in (r.split(",") for r in rows)]


def _check_checkpoints(got, ref):
    assert len(got) == len(ref)
    for a, b in zip(got, ref):
        assert (a["level"], a["iter"]) == (b["level"], b["iter"])
        assert abs(a["offdiag_max"] - b["offdiag_max"]) < 1e-8
        assert abs(a["diag_deviation_max"] - b["diag_deviation_max"]) < 1e-8
        assert (a["orth_deviation"] < 0) == (b["orth_deviation"] < 0)
        assert a["orth_deviation"] <= 1e-10  # acceptance.cpp:152-160 criterion 4


@pytest.mark.parametrize("cname", ["C1", "C2"])
def test_eigenvalues_every_iteration(port, native, cname):
    """eig(<(HW)^T W>) at all 50 accepted iterates within 1e-6 Ha."""
    ref = np.load(os.path.join(GOLDEN, f"{cname}_eigs.npz"))["eig"]
    gold = json.load(open(os.path.join(GOLDEN, f"{cname}_records.json")))
    spec = configs.by_name(cname)
    e = native.engine_for(spec)
    w = e.block_from(port.random_orthonormal(spec))
    got = e.solve(w, algorithm="opt_par_mod", trace_eigs=True, **spec.optimizer_params())
    assert got.sigma_eigs.shape == ref.shape == (spec.max_inner, spec.n_orbitals)
    assert np.max(np.abs(got.sigma_eigs - ref)) < TOL
    # the SolveResult fields the reference's acceptance suite reads
    assert len(got.checkpoints) == spec.max_inner
    assert max(c["orth_deviation"] for c in got.checkpoints) <= 1e-10
    assert got.drift_iterations == gold["summary"]["drift_iterations"]
    e.close()


def _prefix(native, name, start_from_port=None):
    gold = json.load(open(os.path.join(GOLDEN, f"prefix_{name}.json")))
    arr = np.load(os.path.join(GOLDEN, f"prefix_{name}.npz"))
    spec = _spec(gold["spec"])
    k_max = gold["iterations"]
    sk = gold["sketch"]
    e = native.engine_for(spec)
    if start_from_port is not None:
        w0 = e.block_from(start_from_port(spec))
    else:  # Rng(42) normals bit-identical on the host, orthonormalised on the device
        w0 = native.random_orthonormal(e, spec.start_seed)
    params = e.make_params("opt_par_mod", spec.hartree, spec.xc, True, "dst",
                           **{**spec.optimizer_params(), "max_inner": k_max})
    st = native.Stepper(e, w0, params)
    wq = float(np.prod(spec.spacing))
    dists = []
    for k in range(k_max):
        assert st.step() or k == k_max - 1
        cur = st.current()
        wk = e.download(cur)
        s_gpu = sketch_block(wk, wq, sk["m"], sk["seed"])
        del wk
        g_gpu = e.gram(cur, cur)
        dists.append(sketch_projector_distance(s_gpu, g_gpu, arr["sketch"][k], arr["gram"][k]))
    eig = st.sigma_eigs()
    res = st.result()
    recs = st.records()
    st.close()
    e.close()
    return gold, arr, eig, res, recs, dists


@pytest.mark.parametrize("name", ["C2", "C3", "C4g64"])
def test_prefix_full_shape(native, port, name):
    """C2 (96^3, N = 33; 3 iterations) and C3 (128^3, N = 128; as many as the
    fixture holds: 8): the first outer iterations against truncated re-runs
    of the unmodified reference — energy and backtracks per iteration, eig(Sigma) after every iteration (1e-6 Ha), the
    subspace projector of every iterate (sketched ||dP||_F <= 1e-6) and the
    orthogonalization checkpoints. C4g64: the same for two iterations at the C4
    grid (192^3, L = 60, the C4 nuclei) with N = 64 orbitals."""
    if not os.path.exists(os.path.join(GOLDEN, f"prefix_{name}.json")):
        pytest.skip(f"prefix_{name} fixture not generated (oracle/make_golden.py --big)")
    gold, arr, eig, res, recs, dists = _prefix(
        native, name, start_from_port=port.random_orthonormal if name == "C2" else None)
    ref_recs = gold["records"]
    assert len(recs) == len(ref_recs) == gold["iterations"]
    for a, b in zip(recs, ref_recs):
        assert a["iter"] == b["iter"] and a["backtracks"] == b["backtracks"]
        assert abs(a["energy"] - float(b["energy"])) < TOL, (a, b)
        # the Stiefel gradient norm of the record (at N > 64 from the Grams when provably
        # accurate): within 1e-8 relative of the reference's direct sum
        gref = float(b["grad_norm"])
        assert abs(a["grad_norm"] - gref) <= 1e-8 * max(1.0, gref), (a["grad_norm"], gref)
    assert eig.shape == arr["eig"].shape
    assert np.max(np.abs(eig - arr["eig"])) < TOL
    assert max(dists) < TOL, dists
    _check_checkpoints(res.checkpoints, _checkpoints(gold["checkpoints_csv"]))


def _ops_case(name):
    meta = json.load(open(os.path.join(GOLDEN, f"opsr_{name}.json")))
    return meta, np.load(os.path.join(GOLDEN, f"opsr_{name}.npz")), _spec(meta["spec"])


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name", ["C3", "C4g64"])
def test_operators_full_shape(native, name):
    """Every hot-path operator of one iteration at the C3 shape and at the C4 grid
    (192^3) vs the unmodified reference's ops on the same Rng(42) start:
    V_ext, rho, v_H (DST solve vs the reference's CG, both to ||r|| <= 1e-10 ||b||),
    v_xc, v_local, H.u (+ sigma_ii, kinetic, external per orbital), Gram, Sigma,
    the gradient D and ||D_i||^2, z, one line-search trial Orth(W - 0.3 Z)
    (pre-Gram, projector, energy) and eig(Sigma)."""
    meta, ref, spec = _ops_case(name)
    sk = meta["sketch"]
    wq = float(np.prod(spec.spacing))
    pts = sample_points(spec.num_points, sk["samples"])
    e = native.engine_for(spec)
    w = native.random_orthonormal(e, spec.start_seed)

    def block_checks(blk, key, tol):
        host = e.download(blk)
        assert _rel(host[:, pts], ref[key + "_rows"]) < tol, key
        s = sketch_block(host, wq, sk["m"], sk["seed"])
        del host
        assert _rel(s, ref[key + "_sketch"]) < tol, key
        return s

    def field_checks(fid, key, tol):
        f = e.get_field(fid)
        assert _rel(f[pts], ref[key + "_samples"]) < tol, key
        n_ref = ref[key + "_norms"]
        assert abs(float(np.sum(f)) - n_ref[0]) <= tol * max(abs(n_ref[0]), np.sqrt(n_ref[1]) * 1e3), key
        assert abs(float(np.dot(f, f)) - n_ref[1]) <= tol * n_ref[1], key

    block_checks(w, "u0", 1e-12)
    field_checks(native.PO_VEXT, "v_ext", 1e-13)
    e.build_hamiltonian(w)
    field_checks(native.PO_RHO, "rho", 1e-12)
    field_checks(native.PO_VH, "v_h", 1e-8)
    field_checks(native.PO_VXC, "v_xc", 1e-12)
    field_checks(native.PO_VLOCAL, "v_local", 1e-8)
    en = e.total_energy(w)
    for k in ("kinetic", "external", "hartree", "xc", "total"):
        assert abs(en[k] - meta["energy"][k]) < 1e-7, (k, en[k], meta["energy"][k])
    hw = e.alloc()
    sig_d, kin, ext = e.apply_hamiltonian(w, hw)
    block_checks(hw, "hw", 1e-8)
    assert _rel(kin, ref["kin"]) < 1e-11 and _rel(ext, ref["ext"]) < 1e-11
    assert _rel(sig_d, ref["sigma_diag"]) < 1e-8
    assert np.max(np.abs(e.gram(w, w) - ref["gram_ww"])) < 1e-13
    d = e.alloc()
    sigma, dd = e.stiefel_gradient(w, hw, d)
    assert np.max(np.abs(sigma - ref["sigma"])) < 1e-8
    assert _rel(dd, ref["d_norm2"]) < 1e-7
    block_checks(d, "d", 1e-7)
    z = e.alloc()
    sd, zz = e.diagonal_residuals(w, hw, z)
    assert _rel(sd, ref["sigma_diag"]) < 1e-8
    block_checks(z, "z", 1e-7)
    gam = np.linalg.eigvalsh(0.5 * (sigma + sigma.T))
    assert np.max(np.abs(gam - ref["sigma_eig"])) < TOL
    # one line-search trial (manifold.cpp:136-169)
    trial, wt = e.alloc(), e.alloc()
    e.linear_combination(w, -meta["trial_tau"], z, trial)
    pre, dev, fb = e.orthonormalize(trial, wt, True)
    assert not fb and dev <= 1e-12
    assert np.max(np.abs(pre - ref["orth_pre_gram"])) < 1e-8
    host = e.download(wt)
    s = sketch_block(host, wq, sk["m"], sk["seed"])
    del host
    assert sketch_projector_distance(s, e.gram(wt, wt), ref["orth_w_sketch"], ref["orth_gram"]) < TOL
    e.build_hamiltonian(wt)
    te = e.total_energy(wt)
    assert abs(te["total"] - meta["trial_energy"]["total"]) < 1e-7
    e.close()
