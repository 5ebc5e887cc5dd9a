#!/bin/bash
# ncu --set full of one steady-state K2 launch (70B GQA config) and one K1 launch at chunk 8
# (split-K heavy), with source-level stall sampling.
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_kernel -s 16100 -c 1 \
    -o gpurun_out/prof_gqa python bench.py --config llama3-70b-gqa --steps 3 --warmup 3 --ff 200 --no-cpu-baseline \
    > gpurun_out/ncu_gqa_stdout.log 2>&1
DBK_CHUNK_PAGES=8 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 9700 -c 1 \
    -o gpurun_out/prof_k1_c8 python bench.py --steps 3 --warmup 3 --ff 300 --no-cpu-baseline \
    > gpurun_out/ncu_k1c8_stdout.log 2>&1
ls -la gpurun_out/*.ncu-rep
