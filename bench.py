#!/usr/bin/env python
"""Benchmark of the B200-native hot path (one JSON line on rank 0).

A "step" is ONE outer iteration of the reference's orbital-update +
orthonormalise loop (InnerLoop iteration with n_org = 1, optimizer.cpp:358-576)
on BASELINE configs[1] (C2: 96^3 grid, 20 seeded nuclei, N = 33 orbitals,
fp64): directions + BB step + backtracked trial(s) (Gram -> Cholesky -> U L^-T
-> density/xc -> Poisson CG -> v_local -> fused H u / energy) + acceptance.

metric: orbital.gridpoint H.u updates/s = N * N_g * steps / time; each outer
iteration applies H to every orbital at every grid point once (the accepted
trial's fused H u), so s per outer iteration = N * N_g / value.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (oracle/_ref,
the unmodified reference built here; else the C restatement) on the same
config on the host cores. Under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1510_07230_b200 import configs  # noqa: E402

METRIC = "orbital·gridpoint H·u updates/s"
UNIT = "updates/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML every
    ~2 ms (the C2 timed region is tens of ms), nvidia-smi as a fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, [reasons])
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
        except Exception:
            self._nv = None

    def _sample_nvml(self):
        nv = self._nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        reasons = [name for name, attr in self.REASONS if bits & getattr(nv, attr, 0)]
        self.samples.append((float(sm), float(mx), reasons))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if out:
            f = [x.strip() for x in out.split(",")]
            reasons = [self.REASONS[k][0] for k in range(4) if len(f) > 3 + k and f[3 + k].lower() == "active"]
            try:
                self.samples.append((float(f[0]), float(f[1]), reasons))
            except ValueError:
                pass

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nv else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.002 if self._nv else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.samples:  # region shorter than one sample: take one right after
            try:
                self._sample_nvml() if self._nv else self._sample_smi()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"]}
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples]
        reasons = sorted({r for s in self.samples for r in s[2]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nv else "nvidia-smi"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


# ------------------------------------------------------------ CPU reference

def ref_binary():
    p = os.path.join(ROOT, "oracle", "_ref", "trace_ref")
    return p if os.path.exists(p) else None


def run_reference_iterations(spec, iterations: int, threads: int):
    """Unmodified reference (oracle/_ref/trace_ref -> opt_par_mod_inner) on the
    config; returns per-iteration wall ms of InnerLoop (IterationRecord.wall_ms,
    optimizer.cpp:574) and whether the real reference was used."""
    spec = configs.ProblemSpec(**{**spec.__dict__})
    spec.max_inner = iterations
    binary = ref_binary()
    if binary:
        with tempfile.TemporaryDirectory() as d:
            with open(os.path.join(d, "spec.json"), "w") as f:
                json.dump(spec.trace_ref_spec(threads=threads), f)
            subprocess.run([binary, "solve", os.path.join(d, "spec.json"), d], check=True,
                           capture_output=True)
            rows = open(os.path.join(d, "records.csv")).read().strip().split("\n")[1:]
            return [float(r.split(",")[-1]) for r in rows], "reference", threads
    # C restatement (single-threaded port) when the reference binary is absent
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import port  # noqa: E402  (test/baseline infrastructure only)

    u0 = port.random_orthonormal(spec)
    times = []
    t = time.perf_counter()
    r = port.solve(spec, u0=u0, trace_eigs=False, max_inner=iterations)
    total = time.perf_counter() - t
    n = max(1, len(r["records"]))
    times = [1e3 * total / n] * n
    return times, "port", 1


def cpu_baseline(spec, threads):
    ms, kind, cores = run_reference_iterations(spec, 1, threads)
    per = ms[0] / 1e3
    return {"value": spec.n_orbitals * spec.num_points / per, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"1 outer iteration of {spec.name} ({spec.n[0]}^3, N={spec.n_orbitals}) via "
                      f"{'unmodified reference opt_par_mod_inner' if kind == 'reference' else 'C restatement'}"
                      f", {per:.2f} s/iteration"}


def reference_arm(args, spec):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    warm = min(args.warmup, 1)
    k = min(args.steps, 15)
    ms, kind, cores = run_reference_iterations(spec, warm + k, threads)
    timed = ms[warm:warm + k]
    sec = float(np.sum(timed)) / 1e3
    value = spec.n_orbitals * spec.num_points * len(timed) / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(timed), "warmup": warm, "ms_per_step": 1e3 * sec / len(timed),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config)",
            "config": {"workload": f"{spec.name}: {spec.n[0]}^3 grid, N={spec.n_orbitals}, "
                                   "opt_par_mod n_org=1, one outer iteration per step",
                       "threads": threads},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"{len(timed)} outer iterations of {spec.name} after {warm} warm-up "
                                       f"(IterationRecord.wall_ms), Executor({threads})"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- ours

def time_kernel(torch, native, e, op, reps, a=-1, b=-1, out=-1):
    """Average device time (ms) of one launch, CUDA events on the engine stream."""
    stream = torch.cuda.ExternalStream(e.stream)
    for _ in range(2):
        e.enqueue(op, a, b, out)
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(reps):
        e.enqueue(op, a, b, out)
    s1.record(stream)
    s1.synchronize()
    return s0.elapsed_time(s1) / reps


def ours(args, spec):
    import torch
    import torch.distributed as dist

    from paper_1510_07230_b200 import native

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
        uid = [native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        e = native.engine_for(spec, rank, world, native.PO_COMM_NCCL, uid[0], device=local)
    else:
        e = native.engine_for(spec, device=local)

    def barrier():
        if world > 1:
            dist.barrier()

    N, ng = spec.n_orbitals, spec.num_points
    w0 = native.random_orthonormal(e, spec.start_seed)
    total_steps = args.warmup + args.steps
    params = e.make_params("opt_par_mod", True, True, False, args.poisson,
                           max_inner=2 * total_steps + 4, n_org=1, n_diag=100)
    st = native.Stepper(e, w0, params)
    stream = torch.cuda.ExternalStream(e.stream)
    for _ in range(args.warmup):
        st.step()
    e.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = native.launch_count()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        done = 0
        for _ in range(args.steps):
            if not st.step():
                break
            done += 1
        ev1.record(stream)
        ev1.synchronize()
    launches = native.launch_count() - l0
    e.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    recs = st.records()
    steps = max(done, 1)
    step_wall = [r["wall_ms"] for r in recs[-steps:]] if recs else []
    value = N * ng * steps / (ms / 1e3)

    # ---- e2e (headline): the reference-facing call on HOST buffers. A user of
    # the drop-in replaces InnerLoop::run(W) with po_solve on a host block: the
    # timed region uploads W from pinned memory, runs K outer iterations (each
    # reads its energy record back to the host), and downloads the final W.
    host = torch.empty(N * e.ngl, dtype=torch.float64, pin_memory=True).numpy().reshape(N, e.ngl)
    e.download(st.current(), host)
    e2e_steps = max(1, args.steps)
    # untimed warm-up call: the engine keeps solver scratch across calls (as a
    # long-lived drop-in engine does), so the timed call allocates nothing
    e.solve_host(host, host, "opt_par_mod", True, True, args.poisson, max_inner=1, n_org=1, n_diag=100)
    e.download(st.current(), host)
    e.synchronize()
    barrier()
    t0 = time.perf_counter()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    # po_solve_host: upload, K iterations, finalize with the download overlapped
    res = e.solve_host(host, host, "opt_par_mod", True, True, args.poisson, max_inner=e2e_steps,
                       n_org=1, n_diag=100)
    ev3.record(stream)
    ev3.synchronize()
    e2e_ms = ev2.elapsed_time(ev3)
    wall_e2e = time.perf_counter() - t0
    e2e_iters = max(1, len(res.records))
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = N * ng * e2e_iters / (e2e_ms / 1e3)
    # secondary: the whole block round-trips through host memory EVERY iteration
    rt_steps = max(1, min(args.steps, 10))
    e.download(st.current(), host)  # the stepper's own iterate (host held the solve's result)
    e.synchronize()
    ev4, ev5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev4.record(stream)
    for _ in range(rt_steps):
        e.upload(st.current(), host)
        st.step()
        e.download(st.current(), host)
    ev5.record(stream)
    ev5.synchronize()
    rt_ms = ev4.elapsed_time(ev5)
    if world > 1:
        t = torch.tensor([rt_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rt_ms = float(t.item())
    rt_value = N * ng * rt_steps / (rt_ms / 1e3)
    block_bytes = N * e.ngl * 8

    # ---- roofline of the dominant kernels (CUDA events on the launching stream)
    peaks, peak_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    cur = st.current()
    scratch = e.alloc()
    e.build_hamiltonian(cur)  # default state for the stencil's v_local
    h_ms = time_kernel(torch, native, e, "hamiltonian", 20, a=cur, out=scratch)
    h_bytes = 16.0 * N * e.ngl + 8.0 * e.ngl  # read u + write Hu per orbital.point, + v_local
    g_ms = time_kernel(torch, native, e, "gram_sym", 20, a=cur)
    # the step's other dominant kernels, same clock (measurement ops through po_enqueue)
    fp64 = None
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            fp64 = float(json.load(f)["fp64_tflops"])
    except Exception:
        pass
    step_kernels = []

    def add_kernel(name, ms, nbytes, flops=None):
        ent = {"kernel": name, "launch_ms": ms, "algorithmic_bytes": nbytes,
               "hbm_frac": nbytes / (ms / 1e3) / 1e9 / hbm}
        if flops is not None and fp64:
            ent["algorithmic_flops"] = flops
            ent["fp64_frac"] = flops / (ms / 1e3) / 1e12 / fp64
        step_kernels.append(ent)

    blk = float(N) * e.ngl * 8
    add_kernel("hamiltonian4_kernel (H u)", h_ms, h_bytes)
    hw_b, z_b = e.alloc(), e.alloc()
    e.enqueue("hamiltonian", a=cur, out=hw_b)
    sg_ms = time_kernel(torch, native, e, "gram", 10, a=hw_b, b=cur)  # Sigma = w (HW)^T W
    add_kernel("Sigma Gram (HW)^T W", sg_ms, 2 * blk, 2.0 * N * N * ng)
    add_kernel("symmetric Gram W^T W", g_ms, blk, float(N) * (N + 1) * ng)
    if N <= 48:  # the small-N fused passes of the C2 step
        e.enqueue("gram", a=hw_b, b=cur)
        d_ms = time_kernel(torch, native, e, "directions", 10, a=cur, b=hw_b, out=z_b)
        # implicit z (the iteration's form): reads W, HW, W_prev, HW_prev, writes nothing
        add_kernel("directions_tma_kernel (||z||^2, ||D||^2, BB)", d_ms, 4 * blk, 2.0 * N * N * ng)
        e.enqueue("gram_sym", a=cur)
        e.enqueue("cholesky")
        r_ms = time_kernel(torch, native, e, "rotation_fused", 10, a=cur, b=hw_b, out=scratch)
        add_kernel("rotate_fused_kernel (rotation + G2 + density)", r_ms, 3 * blk,
                   2.0 * N * (N + 1) * ng)
    else:
        e.enqueue("gram_sym", a=cur)
        e.enqueue("cholesky")
        r_ms = time_kernel(torch, native, e, "rotation", 10, a=cur, b=hw_b, out=scratch)
        add_kernel("triangular rotation (W - tau Z) L^-T", r_ms, 3 * blk, float(N) * (N + 1) * ng)
    e.free(hw_b)
    e.free(z_b)
    e.enqueue("density_xc", a=cur)
    e.set_poisson_solver(args.poisson)
    p_ms = time_kernel(torch, native, e, "poisson", 5)
    st.close()
    traffic = None
    if spec.name == "C2":  # dram read+write per launch from the committed ncu --set full capture
        try:
            with open(os.path.join(ROOT, "profiles", "traffic_C2.json")) as f:
                traffic = json.load(f)["hamiltonian_traffic_bytes_per_launch"]
        except Exception:
            traffic = None
    roofline = {"kernel": "hamiltonian4_kernel (batched H u + fused sigma/kinetic/external)",
                "bound": "hbm", "achieved": h_bytes / (h_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": h_bytes / (h_ms / 1e3) / 1e9 / hbm, "traffic": traffic,
                "traffic_source": "profiles/traffic_C2.json (ncu dram__bytes_read+write, 1 launch)",
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                "algorithmic_bytes_per_launch": h_bytes, "launch_ms": h_ms}
    iter_ms = ms / steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": iter_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config, i.i.d. N(0,1) start from parorb::Rng(42))",
            "config": {"workload": f"{spec.name}: {spec.n[0]}^3 grid, N={N}, L={spec.extent[0]} bohr, "
                                   "opt_par_mod n_org=1 (= opt_par), one outer iteration per step",
                       "parallelism": f"slab{world}" if world > 1 else "single",
                       "l2": f"inputs larger than L2 (orbital block {block_bytes / 1e6:.0f} MB per copy)"},
            "s_per_outer_iteration": iter_ms / 1e3,
            "backtracks_in_timed_steps": int(sum(r["backtracks"] for r in recs[-steps:])),
            "step_wall_ms": {"min": min(step_wall), "median": float(np.median(step_wall)),
                             "max": max(step_wall)} if step_wall else None,
            "kernel_ms": {"hamiltonian": h_ms, "gram_sym": g_ms, "poisson_cg_solve": p_ms},
            "roofline": roofline,
            "step_kernels": step_kernels,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": block_bytes / e2e_iters,
                    "d2h_bytes_per_step": block_bytes / e2e_iters + 2 * (9 * N + 64) * 8,
                    "steps": e2e_iters, "wall_s": wall_e2e,
                    "how": "po_solve_host on pinned host buffers: H2D of W, K outer iterations (decision "
                           "scalars read back each), D2H of the final W overlapped with the finalize "
                           "pass, CUDA events around all of it",
                    "roundtrip_every_step": {"value": rt_value, "unit": UNIT, "steps": rt_steps,
                                             "h2d_bytes_per_step": block_bytes,
                                             "d2h_bytes_per_step": block_bytes}},
            "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(spec, os.cpu_count() or 1)
        except Exception as ex:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    e.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--poisson", default="dst", choices=["dst", "cg", "cg_warm"])
    args = ap.parse_args()
    spec = configs.by_name(args.config)
    if args.impl == "reference":
        return reference_arm(args, spec)
    return ours(args, spec)


if __name__ == "__main__":
    sys.exit(main())
