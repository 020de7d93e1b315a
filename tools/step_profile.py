"""Kernel launch list of K outer iterations of the bench workload (C2 by default).

Run under ncu with --profile-from-start off: only the K timed iterations are
inside the cudaProfilerStart/Stop range, so the per-kernel totals divided by K
are the per-iteration breakdown (cold-cache, serialised — shares, not absolutes).
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/step_launches.csv python tools/step_profile.py --steps 5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--poisson", default="dst")
    a = ap.parse_args()
    import torch

    from paper_1510_07230_b200 import configs, native
    spec = configs.by_name(a.config)
    e = native.engine_for(spec)
    w0 = native.random_orthonormal(e, spec.start_seed)
    params = e.make_params("opt_par_mod", True, True, False, a.poisson,
                           max_inner=a.warmup + a.steps + 2, n_org=1, n_diag=100)
    st = native.Stepper(e, w0, params)
    for _ in range(a.warmup):
        st.step()
    e.synchronize()
    l0 = native.launch_count()
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        st.step()
    e.synchronize()
    torch.cuda.profiler.stop()
    recs = st.records()[-a.steps:]
    print(f"steps {a.steps} launches {native.launch_count() - l0} "
          f"backtracks {sum(r['backtracks'] for r in recs)} "
          f"wall_ms {[round(r['wall_ms'], 3) for r in recs]}")
    st.close()
    e.close()


if __name__ == "__main__":
    main()
