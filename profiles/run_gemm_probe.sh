#!/bin/bash
# L2 -> SM operand bandwidth probe with the model GEMM: shapes with one 128 x BN tile per SM and
# no K split (N = 128 x 148 weight rows), weights L2-resident (K small) or not (K large).
mkdir -p gpurun_out
timeout 300 python experiments/gemm_bench.py --shapes "" --ms 32,64,128,256 --reps 40 \
   --custom "18944:512;18944:1024;18944:2048;18944:4096;9472:1024;37888:1024" > gpurun_out/gemm_probe.log 2>&1
cat gpurun_out/gemm_probe.log | cut -c1-400
