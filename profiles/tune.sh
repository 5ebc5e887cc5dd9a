#!/bin/bash
# Tuning sweep (run under gpurun): decode tokens/s and attention GB/s per variant.
out=gpurun_out/tune_$(date +%s).txt
for cfg in llama2-7b llama3-70b-gqa; do
  for cp in default 16 32 64; do
    if [ "$cp" = default ]; then unset DBK_CHUNK_PAGES; else export DBK_CHUNK_PAGES=$cp; fi
    r=$(timeout 300 python bench.py --config $cfg --no-cpu-baseline --ff 300 --steps 30 2>&1 | tail -1)
    echo "$cfg chunk=$cp $(echo "$r" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], d["ms_per_step"], r["achieved"], r["frac"], r["ms_per_launch"], r["chunk_pages"], r["ctas_per_sm"], d["config"]["mean_batch"])' 2>&1)" | tee -a $out
  done
done
unset DBK_CHUNK_PAGES
