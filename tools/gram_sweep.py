"""Warm device time of the large-N Gram variants at a BASELINE shape (CUDA
events on the engine stream): symmetric one-source (G_HH, verification G2),
symmetric two-source (a trial's G0 of W - tau Z) and the non-symmetric Sigma.
Measurement helper."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1510_07230_b200 import configs, native  # noqa: E402


def timeit(e, fn, reps=20):
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


spec = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "C3")
e = native.engine_for(spec)
w, z = e.alloc(), e.alloc()
e.random_block(w, 3)
e.random_block(z, 7)
fp64 = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["fp64_tflops"]
N, ng = spec.n_orbitals, spec.num_points
for name, fn, fl in (("sym", lambda: e.enqueue("gram_sym", a=w), N * (N + 1) * ng),
                     ("sym2", lambda: e.enqueue("gram_trial", a=w, b=z), N * (N + 1) * ng),
                     ("nonsym", lambda: e.enqueue("gram", a=w, b=z), 2 * N * N * ng)):
    us = timeit(e, fn)
    print(f"{name:8s} {us:8.1f} us  {fl / us / 1e6 / fp64:.2f} of FP64")
e.close()
