#!/bin/bash
# Model GEMM (gemm_tc.cu) on one B200: parity tests, throughput next to cuBLAS on the projection
# shapes (experiments/gemm_bench.py, CUDA graphs, cold weights), and one ncu --set full capture
# of the 7B O and QKV projections at M = 512.  Outputs under gpurun_out/ (copied to profiles/).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -5 > gpurun_out/gemm_test.log
timeout 400 python experiments/gemm_bench.py --reps 40 --out gpurun_out/gemm_bench.json > gpurun_out/gemm_bench.log 2>&1
timeout 300 ncu --set full --import-source on -k regex:gemm_tc -c 4 -f -o gpurun_out/gemm_full \
    python experiments/gemm_bench.py --shapes 7b_o,7b_qkv --ms 512 --reps 2 > gpurun_out/ncu_gemm.log 2>&1
tail -3 gpurun_out/ncu_gemm.log
