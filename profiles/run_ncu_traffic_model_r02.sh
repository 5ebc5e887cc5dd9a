#!/bin/bash
# DRAM traffic of the model step's decode launches (7B --model), appended to ncu_traffic.json's
# entries by profiles/ncu_traffic.py (run under gpurun; DBK_BUILD = the build's short hash)
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 1500 ncu --nvtx --nvtx-include "dbk_step/" --metrics $M --clock-control none --csv \
    --log-file gpurun_out/ncu_traffic_7b_model.csv python bench.py --ncu-step --warmup 3 --no-cpu-baseline --ff 300 --model \
    > gpurun_out/ncu_traffic_7b_model.json 2> gpurun_out/ncu_traffic_7b_model.err
python profiles/ncu_traffic.py gpurun_out/ncu_traffic_model.json "7b_model:gpurun_out/ncu_traffic_7b_model.csv:gpurun_out/ncu_traffic_7b_model.json"
cat gpurun_out/ncu_traffic_model.json | head -30
