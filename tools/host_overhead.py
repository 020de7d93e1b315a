"""Host-side cost of one outer iteration: the C2 control flow on a tiny grid
(GPU work negligible), wall time per step. Measurement helper."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1510_07230_b200 import configs, native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
spec = configs.small_molecule(n, 33, L=10.0)
e = native.engine_for(spec)
w0 = native.random_orthonormal(e, 42)
params = e.make_params("opt_par_mod", True, True, False, "dst", max_inner=80, n_org=1, n_diag=100)
st = native.Stepper(e, w0, params)
for _ in range(5):
    st.step()
e.synchronize()
t0 = time.perf_counter()
k = 0
for _ in range(40):
    if not st.step():
        break
    k += 1
e.synchronize()
dt = (time.perf_counter() - t0) / max(k, 1)
recs = st.records()[-k:]
print(f"grid {n}^3 N=33: {dt * 1e6:.0f} us per outer iteration (host + launch latency), "
      f"{native.launch_count()} launches total, backtracks {sum(r['backtracks'] for r in recs)}")
