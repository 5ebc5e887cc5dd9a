#!/bin/bash
# Per-kernel device time of ONE steady-state full-model step (7B, --model): ncu over the kernels
# inside bench.py's NVTX range (--ncu-step), durations only, clocks not locked.
mkdir -p gpurun_out
timeout 1500 ncu --nvtx --nvtx-include "dbk_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ncu_model_step.csv python bench.py --ncu-step --model --warmup 3 --no-cpu-baseline --ff ${FF:-300} ${EXTRA} \
    > gpurun_out/ncu_model_step.json 2> gpurun_out/ncu_model_step.err
python3 profiles/summarize_launches.py gpurun_out/ncu_model_step.csv > gpurun_out/ncu_model_step_summary.txt
cat gpurun_out/ncu_model_step_summary.txt; tail -2 gpurun_out/ncu_model_step.json | cut -c1-600
