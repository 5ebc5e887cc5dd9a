#!/bin/bash
# K2 (warps x stages per CTA) variants on the 70B GQA per-GPU shards (TP1 / TP4 / TP8), one box.
# Prints: variant tp tokens/s ms/step achieved_GB/s frac ms/launch chunk read_probe frac_of_probe clocks
out=gpurun_out/tune_gqa_tp_$(date +%s).txt
run() {  # $1 label, $2 extra bench args
  r=$(timeout 400 python bench.py --config llama3-70b-gqa --no-cpu-baseline --no-e2e --ff 200 --steps 30 $2 2>&1 | tail -1)
  echo "$1 $(echo "$r" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], d["ms_per_step"], r["achieved"], r["frac"], r["ms_per_launch"], r["chunk_pages"], r["read_probe_gbs"], r["frac_of_read_probe"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])' 2>&1)" | tee -a $out
}
for v in ${VARIANTS:-4x3 1x3 2x3}; do
  for tp in ${TPS:-1 4 8}; do
    if [ $tp = 1 ]; then a=""; else a="--tp-shard $tp"; fi
    DBK_GQA_WS=$v run "$v tp$tp" "$a"
  done
done
