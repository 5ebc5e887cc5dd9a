#!/bin/bash
# K2 variants on the 70B GQA config (one box): (warps x stages) trade-off; 2-D vs 5-D TMA
out=gpurun_out/tune_gqa_$(date +%s).txt
run() {
  r=$(timeout 300 python bench.py --config llama3-70b-gqa --no-cpu-baseline --ff 200 --steps 30 2>&1 | tail -1)
  echo "$1 $(echo "$r" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], d["ms_per_step"], r["achieved"], r["frac"], r["ms_per_launch"], r["chunk_pages"], r["read_probe_gbs"], r["frac_of_read_probe"])' 2>&1)" | tee -a $out
}
run "4x3"
DBK_GQA_WS=2x6 run "2x6"
DBK_GQA_WS=8x3 run "8x3"
DBK_GQA_TMA2=1 run "4x3_tma2d"
run "4x3_again"
