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
  prefix_<C>.json/.npz    `--big`: truncated re-runs of the unmodified reference
                          (max_inner = 1..K) at the FULL config shape: records,
                          checkpoints and summary of the K run, and after every
                          iteration k eig(Sigma), the Gram and a Rademacher
                          sketch of W_k (trace_ref.cpp Sketch) — the projector
                          gate without committing GB-sized blocks
  opsr_<C>.json/.npz      `--big`: trace_ref ops at a full config grid with the
                          reduced outputs (fields at sampled points + norms,
                          blocks as sampled rows + sketches, all N x N matrices)
  orth_fallback.json/.npz orthonormalize_with_gram of an ill-conditioned full-rank
                          set: the symmetric-eigen fallback (manifold.cpp:118-132)
  C1_eigs.npz, C2_eigs.npz  `--big C1eig,C2eig`: eig(Sigma) at every accepted
                          iterate of the 50-iteration trajectories, from the C
                          restatement after checking its log rows are
                          byte-identical to the reference's
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
        ck = open(os.path.join(d, "checkpoints.csv")).read()
        out = {"spec": json.loads(spec.to_json()), "records": recs, "summary": summ,
               "final_eig": [repr(float(x)) for x in eig], "accepted_csv": acc,
               "checkpoints_csv": ck}
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


SKETCH = {"m": 64, "seed": 7, "samples": 512}


def gen_ops_reduced(name, spec, threads=8):
    """trace_ref ops with reduced outputs at a full config grid."""
    d_spec = spec.trace_ref_spec(threads=threads)
    d_spec["sketch"] = SKETCH
    n, k = spec.n_orbitals, SKETCH["samples"]
    with tempfile.TemporaryDirectory(dir="/tmp") as d:
        run("ops", d_spec, d)
        arr = {}
        for f in ("v_ext", "rho", "v_h", "v_xc", "v_local", "eps_xc"):
            arr[f + "_samples"] = load_bin(os.path.join(d, f + "_samples.bin"))
            arr[f + "_norms"] = load_bin(os.path.join(d, f + "_norms.bin"))
        for b in ("u0", "hw", "z", "d", "orth_w"):
            arr[b + "_rows"] = load_bin(os.path.join(d, b + "_rows.bin"), (n, k))
            arr[b + "_sketch"] = load_bin(os.path.join(d, b + "_sketch.bin"), (n, SKETCH["m"]))
        for v in ("kin", "ext", "sigma_diag", "sigma_eig", "d_norm2"):
            arr[v] = load_bin(os.path.join(d, v + ".bin"))
        for mtx in ("gram_ww", "sigma", "orth_pre_gram", "orth_gram"):
            arr[mtx] = load_bin(os.path.join(d, mtx + ".bin"), (n, n))
        meta = json.load(open(os.path.join(d, "ops.json")))
    np.savez_compressed(os.path.join(GOLDEN, f"opsr_{name}.npz"), **arr)
    with open(os.path.join(GOLDEN, f"opsr_{name}.json"), "w") as f:
        json.dump({"spec": json.loads(spec.to_json()), "sketch": SKETCH, **meta}, f, indent=1)


def gen_prefix(name, spec, iters, threads=8, extend=False):
    """Truncated re-runs (max_inner = 1..iters) of the unmodified reference: the
    k-th run's final W is the reference's iterate after k iterations (finalize,
    optimizer.cpp:581-597, does not change W). extend: keep the committed runs
    k = 1..K0 of prefix_<name>.npz and only add k = K0 + 1..iters (the reference
    is deterministic; C3 costs ~4 min per iteration on 8 cores)."""
    n = spec.n_orbitals
    eigs, sketches, grams, last = [], [], [], None
    k0 = 1
    if extend:
        old = np.load(os.path.join(GOLDEN, f"prefix_{name}.npz"))
        eigs, sketches, grams = list(old["eig"]), list(old["sketch"]), list(old["gram"])
        k0 = len(eigs) + 1
    for k in range(k0, iters + 1):
        d_spec = spec.trace_ref_spec(threads=threads)
        d_spec["params"]["max_inner"] = k
        d_spec["sketch"] = SKETCH
        d_spec["write_final_w"] = False
        with tempfile.TemporaryDirectory(dir="/tmp") as d:
            run("solve", d_spec, d)
            eigs.append(load_bin(os.path.join(d, "final_eig.bin")))
            sketches.append(load_bin(os.path.join(d, "final_sketch.bin"), (n, SKETCH["m"])))
            grams.append(load_bin(os.path.join(d, "final_gram.bin"), (n, n)))
            if k == iters:
                last = {"records": read_records(os.path.join(d, "records.csv")),
                        "summary": json.load(open(os.path.join(d, "summary.json"))),
                        "checkpoints_csv": open(os.path.join(d, "checkpoints.csv")).read(),
                        "accepted_csv": open(os.path.join(d, "accepted.csv")).read()}
        print(f"{name}: k={k} done", flush=True)
    np.savez_compressed(os.path.join(GOLDEN, f"prefix_{name}.npz"), eig=np.array(eigs),
                        sketch=np.array(sketches), gram=np.array(grams))
    with open(os.path.join(GOLDEN, f"prefix_{name}.json"), "w") as f:
        json.dump({"spec": json.loads(spec.to_json()), "iterations": iters, "sketch": SKETCH, **last},
                  f, indent=1)


def c4_grid_spec(n_orbitals=64):
    """BASELINE config 4's grid and nuclei (192^3, L = 60) with a reduced orbital
    count: the per-operator parity point at the C4 shape."""
    s = configs.config4()
    s.name = f"C4g{n_orbitals}"
    s.n_orbitals = n_orbitals
    return s


def gen_port_eigs(cname):
    """eig(Sigma) at EVERY accepted iterate of a 50-iteration BASELINE trajectory
    from the C restatement (oracle/port), whose log rows are first checked to be
    byte-identical to the unmodified reference's golden trajectory."""
    sys.path.insert(0, HERE)
    import port  # noqa: E402  (test infrastructure)

    spec = configs.by_name(cname)
    gold = json.load(open(os.path.join(GOLDEN, f"{cname}_records.json")))
    r = port.solve(spec, trace_eigs=True)
    rows = [port.format_log_row(x) for x in r["records"]]
    ref_rows = [x["row"] for x in gold["records"]]
    same = rows == ref_rows
    print(f"{cname}: port rows byte-identical to the reference: {same}", flush=True)
    if not same:
        raise SystemExit(f"{cname}: port trajectory differs from the reference golden")
    np.savez_compressed(os.path.join(GOLDEN, f"{cname}_eigs.npz"), eig=r["sigma_eigs"])


def main_big(which):
    for c in ("C1", "C2"):
        if f"{c}eig" in which:
            gen_port_eigs(c)
    if "C2p" in which:
        gen_prefix("C2", configs.config2(), 3)
    if "C3ops" in which:
        gen_ops_reduced("C3", configs.config3())
    if "C3p" in which:
        gen_prefix("C3", configs.config3(), 3)
    for w in which:  # C3p<K>, K > 3: more iterations on top of the committed ones
        if w.startswith("C3p") and w[3:].isdigit():
            gen_prefix("C3", configs.config3(), int(w[3:]), threads=int(os.environ.get("GOLDEN_THREADS", "8")),
                       extend=True)
    if "C4ops" in which:
        gen_ops_reduced("C4g64", c4_grid_spec(64))
    if "C4p" in which:  # two solver iterations at the C4 grid (192^3, the C4 nuclei, N = 64)
        gen_prefix("C4g64", c4_grid_spec(64), 2, threads=int(os.environ.get("GOLDEN_THREADS", "8")))


def gen_orth_fallback(name="orth_fallback", eps=1e-5):
    """orthonormalize_with_gram on a full-rank but ill-conditioned set (the
    Cholesky pass is rejected: p_min^2 < 1e-10 p_max^2, manifold.cpp:97-114; the
    rank check passes: lambda_min / lambda_max ~ 2.5e-11 > 1e-12), so the
    reference takes symmetric_fallback (manifold.cpp:118-132)."""
    sys.path.insert(0, HERE)
    import port  # noqa: E402  (test infrastructure: the seeded normals)

    spec = configs.small_molecule(12, 4, L=8.0)
    ng = spec.num_points
    u = port.random_normals(11, 4 * ng).reshape(4, ng)
    u[3] = u[2] + eps * u[3]
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "u.bin")
        u.tofile(path)
        run("orth", spec.trace_ref_spec(start={"kind": "file", "path": path}), d)
        w = load_bin(os.path.join(d, "orth_w.bin"), (4, ng))
        pre = load_bin(os.path.join(d, "pre_gram.bin"), (4, 4))
        meta = json.load(open(os.path.join(d, "orth.json")))
    np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), u=u, w=w, pre_gram=pre)
    with open(os.path.join(GOLDEN, f"{name}.json"), "w") as f:
        json.dump({"spec": json.loads(spec.to_json()), "eps": eps, "seed": 11, **meta}, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="skip the C1/C2 trajectories")
    ap.add_argument("--from-dir", default="/tmp/golden_runs", help="reuse finished C1/C2 trace_ref runs")
    ap.add_argument("--big", default="", help="comma list of C1eig,C2eig,C2p,C3ops,C3p,C3p<K>,C4ops,C4p (long runs; C3p<K> extends the committed C3 prefix to K iterations)")
    args = ap.parse_args()
    if args.big:
        return main_big(args.big.split(","))
    if not os.path.exists(TRACE):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    os.makedirs(GOLDEN, exist_ok=True)
    gen_ops("mol12", configs.small_molecule(12, 3, L=8.0))
    gen_ops("skew", cases()["skew_opt_par"])
    gen_ops_reduced("mol12", configs.small_molecule(12, 3, L=8.0), threads=1)  # pins the sketch
    for name, spec in cases().items():
        gen_solve(f"solve_{name}", spec)
    mol8 = configs.small_molecule(8, 3, L=6.0, max_inner=6)
    gen_levels("levels_mol8", mol8, 2, 5)
    gen_prolong("prolong_init_mol8", mol8, {"kind": "initialize", "seed": 5})
    skew = configs.ProblemSpec("skewp", (6, 5, 7), (4.0, 3.5, 5.0), [(2.0, 1.5, 2.5, 1.0, 1.0)], 2)
    gen_prolong("prolong_skew", skew, {"kind": "random_orthonormal", "seed": 9})
    gen_orth_fallback()
    if not args.quick:
        for cname, fn in (("C1", configs.config1), ("C2", configs.config2)):
            spec = fn()
            src = os.path.join(args.from_dir, cname)
            reuse = os.path.exists(os.path.join(src, "summary.json"))
            gen_solve(f"{cname}_records", spec, keep_w=False, threads=8, src_dir=src if reuse else None)
    print("golden fixtures written to", GOLDEN)


if __name__ == "__main__":
    main()
