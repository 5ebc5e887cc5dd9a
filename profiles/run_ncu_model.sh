#!/bin/bash
# Launch list of the full decode step (NEXT row 3), 7B shape, static b = 512 from step 0:
# every kernel of ~2 steps with its device time (cold-cache, serialised: compare SHARES).
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 700 --csv \
    --log-file gpurun_out/launches_model.csv python bench.py --model --policy static --b-static 512 \
    --steps 3 --warmup 3 --ff 5 --no-cpu-baseline > gpurun_out/ncu_model_stdout.log 2>&1
