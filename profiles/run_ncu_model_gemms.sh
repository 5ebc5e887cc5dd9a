#!/bin/bash
# ncu --set full of the first four GEMM launches (QKV+RoPE/KV, O+residual, gate|up+SiLU,
# down+residual) of one steady-state 7B full-model step (bench.py --ncu-step --model).
mkdir -p gpurun_out
timeout 1500 ncu --nvtx --nvtx-include "dbk_step/" --set full --import-source on -k regex:gemm_tc -c 4 -f \
    -o gpurun_out/model_gemms python bench.py --ncu-step --model --warmup 3 --no-cpu-baseline --ff ${FF:-300} \
    > gpurun_out/ncu_model_gemms.log 2>&1
tail -3 gpurun_out/ncu_model_gemms.log
