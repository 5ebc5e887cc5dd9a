#!/bin/bash
# Full ncu captures (--set full) of the steady-state K1 (7B) and K2 (70B GQA TP1) decode launches of
# the final round-2 build: one engine step in an NVTX range (bench.py --ncu-step), its first decode
# launch profiled; raw pages exported as CSV for profiles/.
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "dbk_step/" -k regex:decode_kernel -c 1 \
    -o gpurun_out/prof_decode_r02 -f python bench.py --ncu-step --warmup 3 --ff 300 --no-cpu-baseline \
    > gpurun_out/ncu_full_stdout.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "dbk_step/" -k regex:decode_gqa_kernel -c 1 \
    -o gpurun_out/prof_gqa_r02 -f python bench.py --config llama3-70b-gqa --ncu-step --warmup 3 --ff 200 --no-cpu-baseline \
    > gpurun_out/ncu_gqa_stdout.log 2>&1
for r in prof_decode_r02 prof_gqa_r02; do
    ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
ls -la gpurun_out | grep prof_
