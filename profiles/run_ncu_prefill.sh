#!/bin/bash
# K7 (prefill) ncu capture: one launch of the 7B-shape prefill (8 x 2048 prompts) after warm-up.
set -e
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel --launch-skip 3 -c 1 \
    -o gpurun_out/ncu_prefill -f python experiments/prefill_bench.py --shape 0 --reps 2 --dtypes f16 --out gpurun_out/pb_ncu.json
ncu -i gpurun_out/ncu_prefill.ncu-rep --page raw --csv > gpurun_out/ncu_prefill_raw.csv
ncu -i gpurun_out/ncu_prefill.ncu-rep --page details --csv > gpurun_out/ncu_prefill_details.csv
ncu -i gpurun_out/ncu_prefill.ncu-rep --page source --csv > gpurun_out/ncu_prefill_source.csv 2>/dev/null || true
