#!/bin/bash
# Round profile collection on one B200 (run under gpurun). Every number that
# lands in profiles/ comes from a command here that first ran without ncu.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 20 --warmup 3 > $OUT/bench_C2.json 2> $OUT/bench_C2.err
echo "bench rc=$?"
python tools/kbench.py C2 > $OUT/kbench_C2.txt 2>&1
python tools/kbench.py C3 > $OUT/kbench_C3.txt 2>&1
python tools/c5_sweep.py > $OUT/c5.log 2>&1 && cp gpurun_out/c5_sweep.json $OUT/
python tools/step_profile.py --steps 5 > $OUT/step_C2.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/step_launches_C2.csv python tools/step_profile.py --steps 5 > /dev/null 2>&1
echo "ncu launches rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/bench_launches_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "ncu bench rc=$?"
# one full capture of each dominant kernel of the C2 iteration (dram traffic per launch)
ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:"hamiltonian4_kernel|directions_tma_kernel|rotate_fused_kernel|gram_tma_kernel" -c 8 \
    -o $OUT/c2_full python tools/step_profile.py --steps 1 --warmup 3 > /dev/null 2>&1
echo "ncu full rc=$?"
