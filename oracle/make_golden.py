"""Generate tests/golden/* from the UNMODIFIED reference (oracle/_ref/trace_ref).

TEST INFRASTRUCTURE ONLY. Needs /root/reference (this container); the GPU box
only reads the committed fixtures. Re-run: `python oracle/make_golden.py`
(C1/C2 full trajectories take ~1.5 / ~6 min on 8 threads; pass --quick to skip).

Fixtures:
  ops_<case>.npz          one evaluation of every hot-path operator on a seeded
                          orthonormal start (trace_ref ops): v_ext, rho, v_H,
                          v_xc, v_local, HU, kinetic/external terms, Gram,
                          Sigma, Z, sigma_ii, a line-search trial's Orth(W - tau Z)
                          and its energy, eig(Sigma)
  solve_<case>.json/.npz  IterationRecord log rows (driver.cpp:136-142, wall_ms
                          zeroed), accepted steps, final energy breakdown, final
                          eig(Sigma), final orbitals (small cases only)
  C1_records.json, C2_records.json
                          the BASELINE configs[0..1] trajectories (50 iterations,
                          opt_par_mod n_org = 1, Rng(42) i.i.d. start)
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_1510_07230_b200 import configs  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
TRACE = os.path.join(HERE, "_ref", "trace_ref")

BOX_ATOMS = [(4.6, 5.2, 6.4, 4.0, 1.0), (7.3, 6.8, 5.1, 4.0, 1.0), (5.9, 7.6, 7.2, 4.0, 1.0),
             (6.6, 4.4, 5.8, 4.0, 1.0)]


def cases():
    """Small parity cases (reference test problems and scaled-down C1)."""
    out = {}
    s = configs.small_molecule(14, 4, L=8.0, max_inner=15)
    s.algorithm = "opt_par"
    out["mol14_opt_par"] = s
    s = configs.small_molecule(14, 4, L=8.0, max_inner=16)
    s.algorithm = "opt_par_mod"
    s.params = {"n_org": 2, "n_diag": 5}
    out["mol14_opt_par_mod"] = s
    s = configs.small_molecule(12, 3, L=8.0, max_inner=12)
    s.algorithm = "optm_qr"
    out["mol12_optm_qr"] = s
    s = configs.ProblemSpec("box12", (12, 12, 12), (12.0, 12.0, 12.0), BOX_ATOMS, 4, hartree=False,
                            xc=False, max_inner=400, algorithm="opt_par")
    out["box12_linear"] = s  # tests/problems.hpp:43-57 at 12^3, grad-norm convergence
    s = configs.ProblemSpec("skew", (12, 10, 14), (7.0, 6.0, 9.0),
                            [(3.0, 2.5, 4.0, 3.0, 1.0), (4.5, 3.2, 5.5, 1.0, 0.7)], 5, max_inner=10,
                            algorithm="opt_par")
    out["skew_opt_par"] = s
    return out


def run(cmd, spec_dict, outdir):
    with open(os.path.join(outdir, "spec.json"), "w") as f:
        json.dump(spec_dict, f)
    subprocess.run([TRACE, cmd, os.path.join(outdir, "spec.json"), outdir], check=True)


def load_bin(path, shape=None):
    a = np.fromfile(path, dtype=np.float64)
    return a.reshape(shape) if shape else a


def read_records(path):
    rows = open(path).read().strip().split("\n")[1:]
    out = []
    for r in rows:
        f = r.split(",")
        out.append({"level": int(f[0]), "iter": int(f[1]), "energy": f[2], "grad_norm": f[3], "tau": f[4],
                    "backtracks": int(f[5]), "did_orth": int(f[6]), "did_diag": int(f[7]),
                    "offdiag_max": f[8], "row": ",".join(f[:9]) + ",0.000"})
    return out


def gen_ops(name, spec):
    with tempfile.TemporaryDirectory() as d:
        run("ops", spec.trace_ref_spec(), d)
        n, ng = spec.n_orbitals, spec.num_points
        arr = {k: load_bin(os.path.join(d, k + ".bin")) for k in
               ("v_ext", "rho", "v_h", "v_xc", "v_local", "eps_xc", "kin", "ext", "sigma_diag", "sigma_eig")}
        for k in ("u0", "hw", "z", "orth_w"):
            arr[k] = load_bin(os.path.join(d, k + ".bin"), (n, ng))
        for k in ("gram_ww", "sigma", "orth_pre_gram"):
            arr[k] = load_bin(os.path.join(d, k + ".bin"), (n, n))
        meta = json.load(open(os.path.join(d, "ops.json")))
    np.savez_compressed(os.path.join(GOLDEN, f"ops_{name}.npz"), **arr)
    with open(os.path.join(GOLDEN, f"ops_{name}.json"), "w") as f:
        json.dump({"spec": json.loads(spec.to_json()), **meta}, f, indent=1)


def gen_solve(name, spec, keep_w=True, threads=1, src_dir=None):
    def collect(d):
        summ = json.load(open(os.path.join(d, "summary.json")))
        recs = read_records(os.path.join(d, "records.csv"))
        eig = load_bin(os.path.join(d, "final_eig.bin"))
        acc = open(os.path.join(d, "accepted.csv")).read()
        out = {"spec": json.loads(spec.to_json()), "records": recs, "summary": summ,
               "final_eig": [repr(float(x)) for x in eig], "accepted_csv": acc}
        with open(os.path.join(GOLDEN, f"{name}.json"), "w") as f:
            json.dump(out, f, indent=1)
        if keep_w:
            w = load_bin(os.path.join(d, "final_w.bin"), (spec.n_orbitals, spec.num_points))
            np.savez_compressed(os.path.join(GOLDEN, f"{name}_w.npz"), w=w)

    if src_dir:
        collect(src_dir)
        return
    with tempfile.TemporaryDirectory() as d:
        run("solve", spec.trace_ref_spec(threads=threads), d)
        collect(d)


def gen_levels(name, spec, outer_levels, seed):
    """optimizer.cpp:638-669 solve (initialize_orbitals + refinement levels)."""
    d_spec = spec.trace_ref_spec(start={"kind": "initialize", "seed": seed})
    d_spec["params"]["outer_levels"] = outer_levels
    d_spec["params"]["seed"] = seed
    with tempfile.TemporaryDirectory() as d:
        run("levels", d_spec, d)
        summ = json.load(open(os.path.join(d, "summary.json")))
        recs = read_records(os.path.join(d, "records.csv"))
        w = load_bin(os.path.join(d, "final_w.bin"), (spec.n_orbitals, summ["final_points"]))
    with open(os.path.join(GOLDEN, f"{name}.json"), "w") as f:
        json.dump({"spec": json.loads(spec.to_json()), "outer_levels": outer_levels, "seed": seed,
                   "records": recs, "summary": summ}, f, indent=1)
    np.savez_compressed(os.path.join(GOLDEN, f"{name}_w.npz"), w=w)


def gen_prolong(name, spec, start):
    """initialize_orbitals (start kind "initialize") or a random start, and its
    refine_uniform + prolongate (grid.cpp:137-212)."""
    with tempfile.TemporaryDirectory() as d:
        run("prolong", spec.trace_ref_spec(start=start), d)
        n = spec.n_orbitals
        fine = [2 * x + 1 for x in spec.n]
        u0 = load_bin(os.path.join(d, "u0.bin"), (n, spec.num_points))
        pr = load_bin(os.path.join(d, "prolong.bin"), (n, fine[0] * fine[1] * fine[2]))
    np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), u0=u0, prolong=pr)
    with open(os.path.join(GOLDEN, f"{name}.json"), "w") as f:
        json.dump({"spec": json.loads(spec.to_json()), "start": start}, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="skip the C1/C2 trajectories")
    ap.add_argument("--from-dir", default="/tmp/golden_runs", help="reuse finished C1/C2 trace_ref runs")
    args = ap.parse_args()
    if not os.path.exists(TRACE):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    os.makedirs(GOLDEN, exist_ok=True)
    gen_ops("mol12", configs.small_molecule(12, 3, L=8.0))
    gen_ops("skew", cases()["skew_opt_par"])
    for name, spec in cases().items():
        gen_solve(f"solve_{name}", spec)
    mol8 = configs.small_molecule(8, 3, L=6.0, max_inner=6)
    gen_levels("levels_mol8", mol8, 2, 5)
    gen_prolong("prolong_init_mol8", mol8, {"kind": "initialize", "seed": 5})
    skew = configs.ProblemSpec("skewp", (6, 5, 7), (4.0, 3.5, 5.0), [(2.0, 1.5, 2.5, 1.0, 1.0)], 2)
    gen_prolong("prolong_skew", skew, {"kind": "random_orthonormal", "seed": 9})
    if not args.quick:
        for cname, fn in (("C1", configs.config1), ("C2", configs.config2)):
            spec = fn()
            src = os.path.join(args.from_dir, cname)
            reuse = os.path.exists(os.path.join(src, "summary.json"))
            gen_solve(f"{cname}_records", spec, keep_w=False, threads=8, src_dir=src if reuse else None)
    print("golden fixtures written to", GOLDEN)


if __name__ == "__main__":
    main()
