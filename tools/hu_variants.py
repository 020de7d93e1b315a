"""Needs the measurement build: make -C paper_1510_07230_b200 -B VARIANTS=1.
Time the batched H u design variants (C2 block) with CUDA events."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1510_07230_b200 import configs, native

spec = configs.config2()
e = native.engine_for(spec)
w = native.random_orthonormal(e, 42)
out = e.alloc()
e.build_hamiltonian(w)
st = torch.cuda.ExternalStream(e.stream)
bytes_ = 16.0 * spec.n_orbitals * e.ngl + 8.0 * e.ngl
for v in [8] + list(range(9, 24)):
    for _ in range(3):
        e._chk(e._lib.po_enqueue(e.h, 100 + v, w, -1, out))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20):
        e._chk(e._lib.po_enqueue(e.h, 100 + v, w, -1, out))
    b.record(st)
    b.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"variant {v}: {ms*1e3:7.1f} us  {bytes_/ms/1e6:7.0f} GB/s  {bytes_/ms/1e6/6547.2:.3f} of peak")
# correctness of the TMA variant vs variant 0 (same partials layout differs; compare outputs)
import numpy as np
o0, o8 = e.alloc(), e.alloc()
e._chk(e._lib.po_enqueue(e.h, 100, w, -1, o0)); e._chk(e._lib.po_enqueue(e.h, 108, w, -1, o8))
a0, a8 = e.download(o0), e.download(o8)
print("variant 8 max |diff| vs 0:", float(np.abs(a0 - a8).max()), "scale", float(np.abs(a0).max()))
