"""Cost of the replicated Hartree solve (DST-I + the CG residual check, and
the reference's cold CG for comparison) at the BASELINE grids, CUDA events on
the engine stream: what a slab-decomposed run pays per trial on every rank
(DESIGN §6). Measurement helper."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1510_07230_b200 import configs, native  # noqa: E402


def timeit(e, fn, reps):
    st = torch.cuda.ExternalStream(e.stream)
    fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / reps


for name in ("C2", "C3", "C4"):
    spec = configs.by_name(name)
    spec.n_orbitals = 8  # the solve only sees the density
    e = native.engine_for(spec)
    w = native.random_orthonormal(e, spec.start_seed)
    e.enqueue("density_xc", a=w)
    out = []
    for mode, reps in (("dst", 10), ("cg", 2)):
        e.set_poisson_solver(mode)
        out.append(f"{mode} {timeit(e, lambda: e.enqueue('poisson'), reps):.3f} ms")
    print(f"{name} {spec.n[0]}^3: " + ", ".join(out), flush=True)
    e.close()
