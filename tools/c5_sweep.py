"""BASELINE configs[4] (C5) kernel microbenchmark sweep on one B200.

Grids 64^3/128^3/192^3/256^3 x N in {64, 256, 1024, 2048}; every block is
FILLED on the device with i.i.d. N(0,1) values (po_fill_normal: a counter hash,
not the reference's Rng bits — the C5 spec allows a device generator) and each
row records filled: true. Local potential: a smooth seeded field of 32
Gaussians (width 2 bohr, A ~ U(-5, 0)). Timed separately with CUDA events on
the engine stream (median of reps): batched H.u, density (+ LDA xc fused),
Gram U^T U (symmetric), and the U L^-T rotation with L from the Cholesky of
that block's Gram. Every row is also verified on the same data (verified: true):
the rotated block is orthonormal to 1e-9 and <(Hu)^T u> is symmetric to 1e-10
relative. Points that do not fit one GPU are reported as such (never skipped
silently). Writes gpurun_out/c5_sweep.json.

Rooflines: H.u / density against the measured HBM peak (MEASURED_PEAKS.json);
Gram (N(N+1) N_g flops) and rotation (N(N+1) N_g flops, triangular) against the
measured FP64 DMMA issue rate (profiles/fp64_peak.json; cuBLAS DGEMM reaches
~95% of it) and against HBM.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1510_07230_b200 import configs, native  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
_fp = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
FP64 = _fp.get("dmma_issue_tflops") or _fp["fp64_tflops"]
free = torch.cuda.mem_get_info()[0]


def timeit(e, fn, reps=5):
    st = torch.cuda.ExternalStream(e.stream)
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


rows = []
sizes = [int(x) for x in os.environ.get("C5_SIZES", "64,128,192,256").split(",")]
norbs = [int(x) for x in os.environ.get("C5_N", "64,256,1024,2048").split(",")]
for n in sizes:
    for N in norbs:
        spec = configs.config5(n, N)
        ng = spec.num_points
        block = 8.0 * N * ng
        need = 2 * block + 64 * ng * 8 + 16 * N * N * 8 + (1 << 30)
        row = {"grid": n, "N": N, "block_GB": block / 1e9}
        if need > 0.92 * free:
            row["status"] = f"does not fit one B200 ({need / 1e9:.0f} GB needed, {free / 1e9:.0f} GB free)"
            rows.append(row)
            print(json.dumps(row), flush=True)
            continue
        e = native.engine_for(spec)
        u = e.alloc()
        e.fill_normal(u, 42)  # every point, every row (filled: true)
        out = e.alloc()
        e.build_hamiltonian(u, hartree=False, xc=True)  # v_local = V(r) + v_xc
        bytes_h = 16.0 * N * e.ngl + 8.0 * e.ngl
        t_h = timeit(e, lambda: e.enqueue("hamiltonian", a=u, out=out))
        t_d = timeit(e, lambda: e.enqueue("density_xc", a=u))
        bytes_d = 8.0 * N * e.ngl + 24.0 * e.ngl
        t_g = timeit(e, lambda: e.enqueue("gram_sym", a=u))
        fl_g = float(N) * (N + 1) * ng
        # L^{-T} from the Cholesky of this block's Gram (the rotation of manifold.cpp:97-114)
        e.enqueue("gram_sym", a=u)
        e.enqueue("cholesky", a=u)
        t_r = timeit(e, lambda: e.enqueue("mix_upper", a=u, out=out))
        fl_r = float(N) * (N + 1) * ng
        # size-independent checks on the same filled blocks (no CPU reference fits here):
        #  * the rotation of the block by the L^-T of its own Gram is orthonormal
        #    (Gram + Cholesky + triangular rotation together, manifold.cpp:97-114, 150-157);
        #  * H is symmetric on the block: <(Hu)^T u> equals its transpose
        #    (H u + the non-symmetric Gram, manifold.cpp:181-187's own check)
        g2 = e.gram(out, out)
        orth_dev = float(np.abs(g2 - np.eye(N)).max())
        e.enqueue("hamiltonian", a=u, out=out)
        sg = e.gram(out, u)
        asym = float(np.abs(sg - sg.T).max() / max(1.0, np.abs(sg).max()))
        row.update({
            "filled": True,
            "verified": bool(orth_dev < 1e-9 and asym < 1e-10),
            "rotation_orthonormality_dev": orth_dev, "hamiltonian_gram_rel_asymmetry": asym,
            "hamiltonian_us": 1e3 * t_h, "hamiltonian_GBs": bytes_h / t_h / 1e6,
            "hamiltonian_frac_hbm": bytes_h / t_h / 1e6 / HBM,
            "density_xc_us": 1e3 * t_d, "density_frac_hbm": bytes_d / t_d / 1e6 / HBM,
            "gram_us": 1e3 * t_g, "gram_TFs": fl_g / t_g / 1e9, "gram_frac_fp64": fl_g / t_g / 1e9 / FP64,
            "gram_frac_hbm": block / t_g / 1e6 / HBM,
            "rotation_us": 1e3 * t_r, "rotation_TFs": fl_r / t_r / 1e9,
            "rotation_frac_fp64": fl_r / t_r / 1e9 / FP64, "rotation_frac_hbm": 2 * block / t_r / 1e6 / HBM,
        })
        rows.append(row)
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()}), flush=True)
        e.close()
        torch.cuda.empty_cache()

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "c5_sweep.json"), "w") as f:
    json.dump({"hbm_gbs": HBM, "fp64_tflops": FP64, "rows": rows}, f, indent=1)
