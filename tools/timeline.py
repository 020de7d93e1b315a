"""GPU timeline of K outer iterations (torch.profiler / CUPTI kernel records):
per-kernel device time, GPU-busy fraction and the largest idle gaps.
Measurement helper: python tools/timeline.py [C2] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1510_07230_b200 import configs, native  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec = configs.by_name(name)
e = native.engine_for(spec)
w0 = native.random_orthonormal(e, spec.start_seed)
params = e.make_params("opt_par_mod", True, True, False, "dst", max_inner=K + 8, n_org=1, n_diag=100)
st = native.Stepper(e, w0, params)
for _ in range(3):
    st.step()
e.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(K):
        st.step()
    e.synchronize()
evs = [ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(ev.time_range.start, ev.time_range.end, ev.name) for ev in evs])
if not ks:
    print("no kernel records")
    sys.exit(0)
t0, t1 = ks[0][0], max(k[1] for k in ks)
busy, gaps, last = 0.0, [], ks[0][0]
for s, en, nm in ks:
    if s > last:
        gaps.append((s - last, nm))
    busy += en - s
    last = max(last, en)
span = t1 - t0
print(f"{K} steps: span {span / K:.1f} us/step, kernels busy {busy / K:.1f} us/step "
      f"({100 * busy / span:.1f}%), idle {(span - busy) / K:.1f} us/step, launches {len(ks) / K:.1f}/step")
gaps.sort(reverse=True)
print("largest gaps (us, next kernel):")
for g, nm in gaps[:12]:
    print(f"  {g:7.1f}  {nm[:70]}")
agg = {}
for s, en, nm in ks:
    key = nm.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:60]
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += en - s
print("per-kernel device time per step:")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"  {t / K:8.1f} us  x{c / K:4.1f}  {k}")
