#!/bin/bash
# ncu --set full of one no-split GEMM launch (N = 128 x 148, K = 1024, M = 256, cta_group 1):
# the epilogue-dominated case of profiles/r02_gemm_trace.log.
mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on -k regex:gemm_tc -c 1 -f -o gpurun_out/gemm_epi \
    python experiments/gemm_bench.py --shapes "" --custom "18944:1024" --ms 256 --reps 2 > gpurun_out/ncu_gemm_epi.log 2>&1
tail -2 gpurun_out/ncu_gemm_epi.log
