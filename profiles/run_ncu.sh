#!/bin/bash
# Profiling recipe used for profiles/ (B200_PROFILING.md): launch list + one --set full capture
# of a steady-state decode_kernel launch.  Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
# 1) every launch of ~5 steady-state steps with its device time (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 11000 -c 250 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --ff 300 --no-cpu-baseline \
    > gpurun_out/ncu_launches_stdout.log 2>&1
# 2) full capture of one decode_kernel launch after the fast-forward (steady-state batch)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 9700 -c 1 \
    -o gpurun_out/prof_decode python bench.py --steps 3 --warmup 3 --ff 300 --no-cpu-baseline \
    > gpurun_out/ncu_full_stdout.log 2>&1 || \
  DBK_BENCH_KV_GB=40 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel \
    -s 9700 -c 1 -o gpurun_out/prof_decode python bench.py --steps 3 --warmup 3 --ff 300 --no-cpu-baseline \
    > gpurun_out/ncu_full_stdout_40g.log 2>&1
ls -la gpurun_out
