#!/usr/bin/env python
"""Benchmark of the B200-native hot path (one JSON line on rank 0).

A "step" is ONE outer iteration of the reference's orbital-update +
orthonormalise loop (InnerLoop iteration with n_org = 1, optimizer.cpp:358-576):
directions + BB step + backtracked trial(s) (Gram -> Cholesky -> U L^-T ->
density/xc -> Poisson -> v_local -> fused H u / energy) + acceptance.

Workload: BASELINE configs[2] (C3: 128^3 grid, 60 seeded nuclei, N = 128,
fp64) — the largest configuration that fits one GPU (C4 needs 8); --config
C1 / C2 select the smaller ones.

metric: orbital.gridpoint H.u updates/s = N * N_g * steps / time; each outer
iteration applies H to every orbital at every grid point once (the accepted
trial's fused H u), so s per outer iteration = N * N_g / value.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one rank per GPU). --impl reference times the reference's own CPU
implementation (oracle/_ref, the unmodified reference built here; else the C
restatement) on the same config on the host cores. Under torchrun only rank 0
runs it.
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


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(spec, world: int) -> dict:
    """The config both arms report (identical strings: the driver compares them)."""
    blk = 8.0 * spec.n_orbitals * spec.num_points
    return {"workload": f"{spec.name}: {spec.n[0]}^3 grid, N={spec.n_orbitals}, L={spec.extent[0]} bohr, "
                        "opt_par_mod n_org=1 (= opt_par), one outer iteration per step",
            "parallelism": f"slab{world}" if world > 1 else "single",
            "l2": (f"inputs larger than L2 (orbital block {blk / 1e6:.0f} MB per copy, L2 126 MB): no flush needed"
                   if blk > 126e6 else
                   f"orbital block {blk / 1e6:.0f} MB fits L2; no flush (each iteration writes several new blocks)")}


# reference-arm sample per config: timed outer iterations after one warm-up
# iteration (the unmodified reference takes ~1.5 s / ~7 s / ~230 s per outer
# iteration at C1 / C2 / C3 on 8-16 host cores; its Gram is serial), sized so
# the whole --impl reference run stays well inside the driver's 30 min
REF_STEPS = {"C1": 15, "C2": 15, "C3": 3}


class CpuBaseline:
    """cpu_baseline of the GPU arm (rank 0, N = 1): one outer iteration of the
    unmodified reference on the same config with all host threads, run after
    the GPU measurements."""

    def __init__(self, spec):
        self.spec = spec
        self.threads = os.cpu_count() or 1
        self.result = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        try:
            ms, kind, cores = run_reference_iterations(self.spec, 1, self.threads)
            per = ms[0] / 1e3
            spec = self.spec
            self.result = {
                "value": spec.n_orbitals * spec.num_points / per, "unit": UNIT, "cores": cores, "kind": kind,
                "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                "sample": f"1 outer iteration (iteration 0, IterationRecord.wall_ms) of {spec.name} "
                          f"({spec.n[0]}^3, N={spec.n_orbitals}) via "
                          f"{'the unmodified reference opt_par_mod_inner' if kind == 'reference' else 'the C restatement'}"
                          f", Executor({cores}), {per:.2f} s/iteration"}
        except Exception as ex:  # reported, never fatal
            self.result = {"value": None, "error": str(ex)[:200]}

    def get(self):
        self._t.join()
        return self.result


def reference_arm(args, spec):
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    warm = 1
    k = max(1, min(args.steps, REF_STEPS.get(spec.name, 15)))
    ms, kind, cores = run_reference_iterations(spec, warm + k, threads)
    timed = ms[warm:warm + k]
    sec = float(np.sum(timed)) / 1e3
    value = spec.n_orbitals * spec.num_points * len(timed) / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(timed), "warmup": warm, "ms_per_step": 1e3 * sec / len(timed),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config, i.i.d. N(0,1) start from parorb::Rng(42))",
            "config": workload_config(spec, world),
            "iterations_timed": list(range(warm, warm + len(timed))),
            "requested": {"steps": args.steps, "warmup": args.warmup,
                          "note": f"the reference is sampled: {len(timed)} outer iterations after {warm} "
                                  f"warm-up ({REF_STEPS.get(spec.name, 15)} max for {spec.name}); the GPU arm "
                                  "reports the same iteration indices under reference_indices"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                             "sample": f"outer iterations {warm}..{warm + len(timed) - 1} of {spec.name} "
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


def load_json(*parts):
    try:
        with open(os.path.join(ROOT, *parts)) as f:
            return json.load(f)
    except Exception:
        return None


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

    def max_over_ranks(ms):
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    N, ng = spec.n_orbitals, spec.num_points
    w0 = native.random_orthonormal(e, spec.start_seed)
    total_steps = args.warmup + args.steps
    params = e.make_params("opt_par_mod", True, True, False, args.poisson,
                           max_inner=2 * total_steps + 4, n_org=1, n_diag=100)
    stream = torch.cuda.ExternalStream(e.stream)

    # ---- the same outer-iteration indices the reference arm samples (1 .. k)
    k_ref = max(1, min(args.steps, REF_STEPS.get(spec.name, 15)))
    st = native.Stepper(e, w0, params)
    st.step()  # iteration 0 (the reference arm's warm-up)
    e.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(k_ref):
        st.step()
    ev1.record(stream)
    ev1.synchronize()
    ref_idx_ms = max_over_ranks(ev0.elapsed_time(ev1)) / k_ref
    st.close()

    # ---- the timed region: K outer iterations after W warm-up iterations
    st = native.Stepper(e, w0, params)
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
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    recs = st.records()
    steps = max(done, 1)
    step_wall = [r["wall_ms"] for r in recs[-steps:]] if recs else []
    value = N * ng * steps / (ms / 1e3)

    # ---- e2e (headline): the reference-facing call on HOST buffers. A user of
    # the drop-in replaces InnerLoop::run(W) with po_solve_host on the block it
    # holds in pageable std::vector memory (integration/parorb_gpu_adapter.hpp):
    # the timed region uploads W (pinned chunk pipeline, staging.cu), runs K
    # outer iterations (each reads its decision scalars back) and downloads the
    # final W (overlapped with the finalize pass).
    e2e_steps = max(1, args.steps)
    block_bytes = N * e.ngl * 8

    def e2e_run(host):
        e.download(st.current(), host)
        # untimed warm-up call: a long-lived engine keeps its scratch blocks
        e.solve_host(host, host, "opt_par_mod", True, True, args.poisson, max_inner=1, n_org=1, n_diag=100)
        e.download(st.current(), host)
        e.synchronize()
        barrier()
        t0 = time.perf_counter()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        res = e.solve_host(host, host, "opt_par_mod", True, True, args.poisson, max_inner=e2e_steps,
                           n_org=1, n_diag=100)
        b.record(stream)
        b.synchronize()
        wall = time.perf_counter() - t0
        iters = max(1, len(res.records))
        return N * ng * iters / (max_over_ranks(a.elapsed_time(b)) / 1e3), iters, wall

    pageable = np.empty((N, e.ngl))
    e2e_value, e2e_iters, wall_e2e = e2e_run(pageable)
    del pageable
    pinned = torch.empty(N * e.ngl, dtype=torch.float64, pin_memory=True).numpy().reshape(N, e.ngl)
    e2e_pinned, _, _ = e2e_run(pinned)
    # secondary: the whole block round-trips through host memory EVERY iteration
    rt_steps = max(1, min(args.steps, 10))
    e.download(st.current(), pinned)
    e.synchronize()
    ev4, ev5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev4.record(stream)
    for _ in range(rt_steps):
        e.upload(st.current(), pinned)
        st.step()
        e.download(st.current(), pinned)
    ev5.record(stream)
    ev5.synchronize()
    rt_value = N * ng * rt_steps / (max_over_ranks(ev4.elapsed_time(ev5)) / 1e3)
    del pinned

    # ---- per-kernel rooflines (CUDA events on the launching stream)
    peaks, peak_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    fp = load_json("profiles", "fp64_peak.json") or {}
    fp64 = fp.get("dmma_issue_tflops") or fp.get("fp64_tflops")
    fp64_src = ("profiles/fp64_peak.json dmma_issue_tflops (measured DMMA issue-rate probe, "
                "tools/dmma_probe.cu; cuBLAS DGEMM reaches %.1f)" % fp.get("fp64_tflops", float("nan"))
                if fp.get("dmma_issue_tflops") else "profiles/fp64_peak.json fp64_tflops (cuBLAS DGEMM)")
    cur = st.current()
    scratch = e.alloc()
    e.build_hamiltonian(cur)  # default state for the stencil's v_local
    blk = float(N) * e.ngl * 8
    step_kernels = []

    def add_kernel(name, ms_, nbytes, flops=None, per_iter=1):
        ent = {"kernel": name, "launch_ms": ms_, "launches_per_iteration": per_iter,
               "algorithmic_bytes": nbytes, "hbm_frac": nbytes / (ms_ / 1e3) / 1e9 / hbm}
        if flops is not None and fp64:
            ent["algorithmic_flops"] = flops
            ent["fp64_frac"] = flops / (ms_ / 1e3) / 1e12 / fp64
        ent["share_of_step"] = per_iter * ms_ / (ms / steps)
        step_kernels.append(ent)
        return ent

    h_ms = time_kernel(torch, native, e, "hamiltonian", 20, a=cur, out=scratch)
    h = add_kernel("hamiltonian4_kernel (H u + sigma/kinetic/external)", h_ms, 2 * blk + 8.0 * e.ngl)
    hw_b, z_b = e.alloc(), e.alloc()
    e.enqueue("hamiltonian", a=cur, out=hw_b)
    sg_ms = time_kernel(torch, native, e, "gram", 10, a=hw_b, b=cur)  # Sigma = w (HW)^T W
    g_ms = time_kernel(torch, native, e, "gram_sym", 20, a=cur)
    if N <= 48:  # the small-N fused passes of the C1/C2 step
        add_kernel("gram_tma_kernel dual (Sigma + G_HH)", sg_ms, 2 * blk, 2.0 * N * N * ng)
        e.enqueue("gram", a=hw_b, b=cur)
        d_ms = time_kernel(torch, native, e, "directions", 10, a=cur, b=hw_b, out=z_b)
        add_kernel("directions_tma_kernel (||z||^2, ||D||^2, BB)", d_ms, 4 * blk, 2.0 * N * N * ng)
        e.enqueue("gram_sym", a=cur)
        e.enqueue("cholesky")
        r_ms = time_kernel(torch, native, e, "rotation_fused", 10, a=cur, b=hw_b, out=scratch)
        dom = add_kernel("rotate_fused_kernel (rotation + G2 + density)", r_ms, 3 * blk, 2.0 * N * (N + 1) * ng)
        dom_bound = "hbm"
    else:  # the large-N tiles of the C3 step
        sig_bytes = 2 * blk
        if N <= 128:
            # the iteration's Sigma Gram also carries the directions' elementwise half
            # (||z||^2, BB products; W_prev / HW_prev streamed beside HW / W): 4 blocks
            sg_ms = time_kernel(torch, native, e, "gram_sigma_bb", 10, a=hw_b, b=cur)
            sig_bytes = 4 * blk
            sig = add_kernel("gram_big_kernel<128, BB> Sigma = w (HW)^T W + ||z||^2 / BB sums (implicit z)",
                             sg_ms, sig_bytes, 2.0 * N * N * ng)
        else:
            sig = add_kernel("gram_big_kernel<128> Sigma = w (HW)^T W", sg_ms, 2 * blk, 2.0 * N * N * ng)
        add_kernel("gram_big_kernel<128> symmetric (G_HH; verification G2 + the trial's density)", g_ms, blk,
                   float(N) * (N + 1) * ng, per_iter=2)
        if N > 128:  # (the separate elementwise pass is HBM-bound; ||D||^2 comes from the Grams)
            e.enqueue("gram", a=hw_b, b=cur)
            d_ms = time_kernel(torch, native, e, "directions", 10, a=cur, b=hw_b, out=z_b)
            add_kernel("dir_big_kernel (direct D norms, implicit z, ||z||^2, BB; fallback pass)", d_ms, 4 * blk,
                       2.0 * N * N * ng, per_iter=0)
        e.enqueue("gram_sym", a=cur)
        e.enqueue("cholesky")
        r_ms = time_kernel(torch, native, e, "rotation_implicit", 10, a=cur, b=hw_b, out=scratch)
        add_kernel("mix_tri_kernel (W - tau z) L^-T, implicit z", r_ms, 3 * blk, float(N) * (N + 1) * ng)
        # (no density pass: 64 < N <= 128 trials get rho from the verification Gram)
        # gram_big_kernel over its three launches of the iteration (Sigma, G_HH, the
        # verification G2): the kernel with the largest share of the step
        tot_ms = sg_ms + 2 * g_ms
        dom = {"kernel": "gram_big_kernel<128> (Sigma [+ directions' sums] + G_HH + G2, per-launch average)",
               "launch_ms": tot_ms / 3, "algorithmic_flops": (2.0 * N * N + 2.0 * N * (N + 1)) * ng / 3,
               "algorithmic_bytes": (sig_bytes + 2 * blk) / 3,
               "share_of_step": sig["share_of_step"] + step_kernels[2]["share_of_step"]}
        dom["fp64_frac"] = dom["algorithmic_flops"] / (dom["launch_ms"] / 1e3) / 1e12 / fp64 if fp64 else None
        dom_bound = "tensor"
    e.free(hw_b)
    e.free(z_b)
    e.enqueue("density_xc", a=cur)
    e.set_poisson_solver(args.poisson)
    p_ms = time_kernel(torch, native, e, "poisson", 5)
    st.close()
    traffic = load_json("profiles", f"traffic_{spec.name}.json") or {}
    dom_traffic = traffic.get("dominant_kernel_traffic_bytes_per_launch")
    if dom_bound == "tensor":
        roofline = {"kernel": dom["kernel"], "bound": "tensor",
                    "achieved": dom["algorithmic_flops"] / (dom["launch_ms"] / 1e3) / 1e12, "peak": fp64,
                    "unit": "TFLOP/s", "frac": dom["fp64_frac"], "traffic": dom_traffic,
                    "peak_source": fp64_src, "algorithmic_flops_per_launch": dom["algorithmic_flops"],
                    "algorithmic_bytes_per_launch": dom["algorithmic_bytes"], "launch_ms": dom["launch_ms"],
                    "share_of_step": dom["share_of_step"]}
    else:
        roofline = {"kernel": dom["kernel"], "bound": "hbm",
                    "achieved": dom["algorithmic_bytes"] / (dom["launch_ms"] / 1e3) / 1e9, "peak": hbm,
                    "unit": "GB/s", "frac": dom["hbm_frac"], "traffic": dom_traffic,
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                    "algorithmic_bytes_per_launch": dom["algorithmic_bytes"], "launch_ms": dom["launch_ms"]}
    roofline["traffic_source"] = (f"profiles/traffic_{spec.name}.json (ncu dram__bytes_read+write, one launch)"
                                  if dom_traffic else "no ncu capture for this config")
    iter_ms = ms / steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": iter_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config, i.i.d. N(0,1) start from parorb::Rng(42))",
            "config": workload_config(spec, world),
            "s_per_outer_iteration": iter_ms / 1e3,
            "backtracks_in_timed_steps": int(sum(r["backtracks"] for r in recs[-steps:])),
            "step_wall_ms": {"min": min(step_wall), "median": float(np.median(step_wall)),
                             "max": max(step_wall)} if step_wall else None,
            "reference_indices": {"iterations": list(range(1, 1 + k_ref)), "ms_per_step": ref_idx_ms,
                                  "value": N * ng / (ref_idx_ms / 1e3),
                                  "note": "the outer iterations the reference arm times (after its one "
                                          "warm-up iteration), timed the same way on the GPU"},
            "kernel_ms": {"hamiltonian": h_ms, "gram_sym": g_ms, "gram_sigma": sg_ms, "poisson": p_ms},
            "roofline": roofline,
            "step_kernels": step_kernels,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": block_bytes / e2e_iters,
                    "d2h_bytes_per_step": block_bytes / e2e_iters + 2 * (9 * N + 64) * 8,
                    "steps": e2e_iters, "wall_s": wall_e2e, "host_buffers": "pageable (numpy)",
                    "how": "po_solve_host on pageable host buffers as the C++ drop-in passes them "
                           "(std::vector): H2D of W through the pinned chunk pipeline, K outer "
                           "iterations (decision scalars read back each), D2H of the final W "
                           "overlapped with the finalize pass, CUDA events around all of it",
                    "pinned_host_buffers": {"value": e2e_pinned, "unit": UNIT},
                    "roundtrip_every_step": {"value": rt_value, "unit": UNIT, "steps": rt_steps,
                                             "h2d_bytes_per_step": block_bytes,
                                             "d2h_bytes_per_step": block_bytes}},
            "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # after every GPU measurement, so the host load never overlaps a timed region
        line["cpu_baseline"] = CpuBaseline(spec).get()
    if rank == 0:
        print(json.dumps(line), flush=True)
    e.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--poisson", default="dst", choices=["dst", "cg", "cg_warm"])
    args = ap.parse_args()
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run (the driver's own form)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(free_port()), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if world is not None and int(world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    spec = configs.by_name(args.config)
    if args.impl == "reference":
        return reference_arm(args, spec)
    return ours(args, spec)


if __name__ == "__main__":
    sys.exit(main())
