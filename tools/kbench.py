"""Per-kernel device times (CUDA events on the engine stream, warm L2 between
reps is NOT flushed: inputs of C2 are 233 MB per block, larger than L2) for the
ops of one outer iteration at a BASELINE config. Measurement helper."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1510_07230_b200 import configs, native  # noqa: E402


def timeit(e, fn, reps=20):
    try:
        return _timeit(e, fn, reps)
    except Exception as ex:  # op unavailable at this N
        print("  (skipped:", str(ex)[:60], ")")
        return float("nan")


def _timeit(e, fn, reps=20):
    st = torch.cuda.ExternalStream(e.stream)
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


spec = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "C2")
e = native.engine_for(spec)
w = native.random_orthonormal(e, spec.start_seed)
z, out = e.alloc(), e.alloc()
e.random_block(z, 7)
e.build_hamiltonian(w)
hw = e.alloc()
e.apply_hamiltonian(w, hw)
N, ngl = spec.n_orbitals, e.ngl
if os.environ.get("KB_PROBE"):
    os.environ["PO_GRAM_PROBE"] = "1"  # stream the Gram rings without math from here on
blk = 8.0 * N * ngl
res = {}
res["hamiltonian"] = timeit(e, lambda: e.enqueue("hamiltonian", a=w, out=out))
res["gram_sym(G2)"] = timeit(e, lambda: e.enqueue("gram_sym", a=w))
res["gram_trial(G0)"] = timeit(e, lambda: e.enqueue("gram_trial", a=w, b=z))
res["gram_nonsym(Sigma)"] = timeit(e, lambda: e.enqueue("gram", a=hw, b=w))
res["gram_sym+density"] = timeit(e, lambda: e.enqueue("gram_density", a=w))
res["gram_sigma+bb"] = timeit(e, lambda: e.enqueue("gram_sigma_bb", a=hw, b=w))
e.enqueue("gram_sym", a=w)
e.enqueue("cholesky")
res["cholesky"] = timeit(e, lambda: e.enqueue("cholesky"))
res["rotation"] = timeit(e, lambda: e.enqueue("rotation", a=w, b=z, out=out))
res["mix_upper"] = timeit(e, lambda: e.enqueue("mix_upper", a=w, out=out))
res["mix_full"] = timeit(e, lambda: e.enqueue("mix", a=w, out=out))
res["rotation_fused"] = timeit(e, lambda: e.enqueue("rotation_fused", a=w, b=z, out=out))
e.enqueue("gram", a=hw, b=w)
res["rotation_implicit"] = timeit(e, lambda: e.enqueue("rotation_implicit", a=w, b=hw, out=out))
e.enqueue("gram", a=hw, b=w)
res["directions"] = timeit(e, lambda: e.enqueue("directions", a=w, b=hw, out=out))
res["density_xc"] = timeit(e, lambda: e.enqueue("density_xc", a=w))
res["poisson"] = timeit(e, lambda: e.enqueue("poisson"), reps=10)
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6547.2
_fp = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
fp64 = _fp.get("dmma_issue_tflops") or _fp["fp64_tflops"]  # the measured DMMA issue rate
ng = spec.num_points
tri, full = N * (N + 1) * ng, 2 * N * N * ng
flops = {"gram_sym(G2)": tri, "gram_trial(G0)": tri, "gram_nonsym(Sigma)": full, "gram_sigma+bb": full, "gram_sym+density": tri,
         "rotation": tri,
         "mix_upper": tri, "mix_full": full, "rotation_fused": 2 * tri, "rotation_implicit": tri,
         "directions": full}
bytes_ = {"hamiltonian": 2 * blk, "gram_sym(G2)": blk, "gram_trial(G0)": 2 * blk,
          "gram_nonsym(Sigma)": 2 * blk, "gram_sigma+bb": 4 * blk, "gram_sym+density": blk, "rotation": 3 * blk, "rotation_fused": 3 * blk, "directions": 4 * blk,
          "rotation_implicit": 3 * blk,
          "density_xc": blk, "mix_upper": 2 * blk, "mix_full": 2 * blk}
for k, v in res.items():
    frac = f"{bytes_[k] / v / 1e3 / hbm:.2f} of HBM" if k in bytes_ else ""
    tf = f"  {flops[k] / v / 1e6:6.2f} TF/s = {flops[k] / v / 1e6 / fp64:.2f} of FP64" if k in flops else ""
    print(f"{k:22s} {v:8.1f} us  {frac}{tf}")
e.close()
