#!/bin/bash
# Full ncu captures of the steady-state K1 (7B) and K2 (70B GQA) launches for the current build
# (same commands as run_ncu.sh steps 2-3), exported as raw CSV pages for profiles/.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 9700 -c 1 \
    -o gpurun_out/prof_decode -f python bench.py --steps 3 --warmup 3 --ff 300 --no-cpu-baseline \
    > gpurun_out/ncu_full_stdout.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_kernel -s 16100 -c 1 \
    -o gpurun_out/prof_gqa -f python bench.py --config llama3-70b-gqa --steps 3 --warmup 3 --ff 200 --no-cpu-baseline \
    > gpurun_out/ncu_gqa_stdout.log 2>&1
for r in prof_decode prof_gqa; do
    ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
    ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
done
ls -la gpurun_out
