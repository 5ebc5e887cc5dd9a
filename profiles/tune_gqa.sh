#!/bin/bash
# K2 variants on the 70B GQA config (one box): 5-D single-box tiles vs 2-D boxes; chunk 32 vs 64
out=gpurun_out/tune_gqa_$(date +%s).txt
run() {
  r=$(timeout 300 python bench.py --config llama3-70b-gqa --no-cpu-baseline --ff 200 --steps 30 2>&1 | tail -1)
  echo "$1 $(echo "$r" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], d["ms_per_step"], r["achieved"], r["frac"], r["ms_per_launch"], r["chunk_pages"], r["read_probe_gbs"], r["frac_of_read_probe"])' 2>&1)" | tee -a $out
}
run "tma5d"
DBK_GQA_TMA2=1 run "tma2d"
DBK_CHUNK_PAGES=64 run "tma5d_chunk64"
DBK_CHUNK_PAGES=16 run "tma5d_chunk16"
run "tma5d_again"
