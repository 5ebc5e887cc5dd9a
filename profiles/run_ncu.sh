#!/bin/bash
# Profiling recipe used for profiles/ (B200_PROFILING.md): launch list + one --set full capture
# of a steady-state K1 launch (7B) and K2 launch (70B GQA).  Run under gpurun from the repo root.
mkdir -p gpurun_out
# 1) every launch of ~7 steady-state steps with its device time (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 11000 -c 250 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --ff 300 --no-cpu-baseline \
    > gpurun_out/ncu_launches_stdout.log 2>&1
# 2) full capture of one K1 launch after the fast-forward (steady-state batch)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 9700 -c 1 \
    -o gpurun_out/prof_decode python bench.py --steps 3 --warmup 3 --ff 300 --no-cpu-baseline \
    > gpurun_out/ncu_full_stdout.log 2>&1
# 3) full capture of one K2 launch (Llama-3-70B shape, GQA 8)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_kernel -s 16100 -c 1 \
    -o gpurun_out/prof_gqa python bench.py --config llama3-70b-gqa --steps 3 --warmup 3 --ff 200 --no-cpu-baseline \
    > gpurun_out/ncu_gqa_stdout.log 2>&1
ls -la gpurun_out/*.ncu-rep
