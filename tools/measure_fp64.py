"""Measure the B200 FP64 (tensor) peak that MEASURED_PEAKS.json lacks
(BASELINE.md §2): cuBLAS DGEMM 8192^3 via torch.matmul(float64), CUDA events,
best of 10 (burst) and back-to-back for 4 s (sustained), 2 N^3 flops each; and
the DMMA issue-rate ceiling from tools/dmma_probe.cu (mma.sync.m8n8k4.f64
chains on every SM, the best configuration) — the attainable tensor-pipe rate
our kernels are measured against (cuBLAS stays a few % below it).
Writes profiles/fp64_peak.json."""
import json
import os
import subprocess
import time

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = 2 * n ** 3 / (best / 1e3) / 1e12
# sustained
t_end = time.time() + 4.0
count = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() < t_end:
    torch.matmul(a, b, out=c)
    count += 1
    if count % 8 == 0:
        torch.cuda.synchronize()
e1.record()
e1.synchronize()
sustained = 2 * n ** 3 * count / (e0.elapsed_time(e1) / 1e3) / 1e12
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                      "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
probe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dmma_probe")
if not os.path.exists(probe):
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", probe + ".cu", "-o", probe],
                   check=True)
txt = subprocess.run([probe], capture_output=True, text=True, check=True).stdout
dmma = max(float(ln.split(":")[1].split()[0]) for ln in txt.splitlines()
           if ln.startswith("DMMA") and "failed" not in ln)
out = {"dmma_issue_tflops": dmma, "dmma_probe": txt.strip().splitlines(), "fp64_tflops": burst, "fp64_tflops_sustained": sustained, "how": "cublasDgemm 8192^3 via torch.matmul "
       "float64, CUDA events, best of 10 (burst) / back-to-back 4 s (sustained), 2N^3 flops",
       "gpu": torch.cuda.get_device_name(), "clocks_after": clk}
os.makedirs("profiles", exist_ok=True)
with open("profiles/fp64_peak.json", "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
