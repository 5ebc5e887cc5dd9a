#!/bin/bash
# K2 chunk size (pages per task) with multi-layer launches on the 70B per-GPU shards.
out=gpurun_out/tune_chunks_ml_$(date +%s).txt
run() {
  r=$(timeout 400 python bench.py --config llama3-70b-gqa --no-cpu-baseline --no-e2e --ff 200 --steps 30 $2 2>&1 | tail -1)
  echo "$1 $(echo "$r" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], d["ms_per_step"], r["achieved"], r["frac"], r["chunk_pages"], r["frac_of_read_probe"], d["config"]["decode_launches_per_step"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])' 2>&1)" | tee -a $out
}
for tp in ${TPS:-8 4}; do
  for cp in ${CHUNKS:-12 20 32 48 64}; do
    DBK_CHUNK_PAGES=$cp run "tp$tp chunk$cp" "--tp-shard $tp"
  done
done
