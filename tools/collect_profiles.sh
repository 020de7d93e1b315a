#!/bin/bash
# Round profile collection on one B200 (run under gpurun). Every number that
# lands in profiles/ comes from a command here that first ran without ncu.
# Writes gpurun_out/prof/; the .ncu-rep files stay on the box (64 MiB limit):
# their raw / details / source pages come back as CSV.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 300 python tools/measure_fp64.py > $OUT/fp64.log 2>&1; cp profiles/fp64_peak.json $OUT/ 2>/dev/null
for C in C3 C2; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  echo "bench $C rc=$?"
  timeout 300 python tools/kbench.py $C > $OUT/kbench_$C.txt 2>&1
  timeout 300 python tools/step_profile.py --config $C --steps 5 > $OUT/step_$C.log 2>&1
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/step_launches_$C.csv python tools/step_profile.py --config $C --steps 5 > /dev/null 2>&1
  echo "ncu launches $C rc=$?"
done
timeout 300 python tools/timeline.py C3 8 > $OUT/timeline_C3.txt 2>&1
timeout 300 python tools/gram_sweep.py C3 > $OUT/gram_sweep_C3.txt 2>&1
# Poisson (DST-I + CG check) cost at the C4 grid: the replicated solve of a slab run
timeout 300 python tools/poisson_cost.py > $OUT/poisson_cost.txt 2>&1
# one full capture of the dominant kernels of each step (dram traffic, FP64 pipe, stalls)
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:"gram_big_kernel|mix_tri_kernel|hamiltonian4_kernel|cholesky_inv_gs_kernel|dst_" -c 12 \
    -o /tmp/c3_full python tools/step_profile.py --config C3 --steps 1 --warmup 3 > /dev/null 2>&1
echo "ncu full C3 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:"hamiltonian4_kernel|directions_tma_kernel|rotate_fused_kernel|gram_tma_kernel" -c 8 \
    -o /tmp/c2_full python tools/step_profile.py --config C2 --steps 1 --warmup 3 > /dev/null 2>&1
echo "ncu full C2 rc=$?"
for C in c3 c2; do
  ncu -i /tmp/${C}_full.ncu-rep --page raw --csv > $OUT/${C}_full_raw.csv 2>/dev/null
  ncu -i /tmp/${C}_full.ncu-rep --page details --csv > $OUT/${C}_full_details.csv 2>/dev/null
done
timeout 1500 python tools/c5_sweep.py > $OUT/c5.log 2>&1 && cp gpurun_out/c5_sweep.json $OUT/
echo "c5 rc=$?"
