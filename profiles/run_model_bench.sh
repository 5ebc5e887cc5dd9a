#!/bin/bash
# Full-model decode step (NEXT row 3) on one B200: the 7B bench line with --model, plus a launch
# list (ncu gpu__time_duration per kernel) of 3 steps for the per-kernel split.
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline --model ${EXTRA} > gpurun_out/model_bench.json 2> gpurun_out/model_bench.err
tail -1 gpurun_out/model_bench.json | python3 -c "
import json,sys; d=json.loads(sys.stdin.read())
print('tok/s', d['value'], 'ms/step', d['ms_per_step'], 'e2e', (d.get('e2e') or {}).get('value'), 'clocks', d['clocks']['sm_mhz'], d['clocks']['reasons'])
print({k: v for k, v in d['config'].items() if 'model' in k or 'attn' in k or 'gemm' in k})"
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/model_launches.csv \
   python bench.py --no-cpu-baseline --model --no-e2e --ff 50 --steps 3 --warmup 3 > /dev/null 2>&1
python3 profiles/summarize_launches.py gpurun_out/model_launches.csv > gpurun_out/model_launches_summary.txt 2>&1
head -30 gpurun_out/model_launches_summary.txt
fi
