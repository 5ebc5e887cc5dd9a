#!/bin/bash
# Per-CTA phase stamps (%globaltimer) of single GEMM launches: where a launch's time goes.
mkdir -p gpurun_out
timeout 300 python experiments/gemm_bench.py --shapes "${SHAPES:-7b_o,7b_qkv}" --ms ${MS:-64,256,512} --reps 20 --trace --trace-modes "${TMODES:-f16}" \
   --custom "${CUSTOM:-18944:1024;9472:1024}" > gpurun_out/gemm_trace.log 2>&1
cat gpurun_out/gemm_trace.log
