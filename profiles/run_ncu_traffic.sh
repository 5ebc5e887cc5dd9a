#!/bin/bash
# DRAM traffic of the decode kernels of one steady-state engine step per configuration, for
# bench.py's roofline.traffic (profiles/ncu_traffic.json).  Run under gpurun from the repo root.
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
specs=()
cap() {  # $1 name, rest: bench args
  name=$1; shift
  timeout 1200 ncu --nvtx --nvtx-include "dbk_step/" --metrics $M --clock-control none --csv \
      --log-file gpurun_out/ncu_traffic_$name.csv python bench.py --ncu-step --warmup 3 --no-cpu-baseline "$@" \
      > gpurun_out/ncu_traffic_$name.json 2> gpurun_out/ncu_traffic_$name.err
  specs+=("$name:gpurun_out/ncu_traffic_$name.csv:gpurun_out/ncu_traffic_$name.json")
}
cap 7b --ff 300
cap 7b_per_layer --ff 300 --per-layer-launches
cap 70b_tp1 --config llama3-70b-gqa --ff 200
cap 70b_tp4 --config llama3-70b-gqa --ff 200 --tp-shard 4
cap 70b_tp8 --config llama3-70b-gqa --ff 200 --tp-shard 8
cap 13b --config llama2-13b-sla --ff 300
python profiles/ncu_traffic.py gpurun_out/ncu_traffic.json "${specs[@]}"
