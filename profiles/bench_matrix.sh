#!/bin/bash
# Bench lines of the hot-path configurations (one B200): 7B (configs[1]), 13B SLA (configs[2]),
# 70B GQA TP1 and the per-GPU KV-head shards of TP2/4/8 (configs[3]); multi-layer launches
# (default) and per-layer launches.  Summary: name tok/s ms/step GB/s frac frac_probe launches/step clocks
mkdir -p gpurun_out
run() {  # $1 name, rest: bench args
  name=$1; shift
  timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/r02_bench_$name.json 2> gpurun_out/r02_bench_$name.err
  python3 - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r02_bench_{n}.json").read().strip().splitlines()[-1])
    r, c = d["roofline"], d["config"]
    print(n, d["value"], d["ms_per_step"], r["achieved"], r["frac"], r["frac_of_read_probe"], c["decode_launches_per_step"],
          d["clocks"]["sm_mhz"], d["clocks"]["reasons"], (d.get("e2e") or {}).get("value"), flush=True)
except Exception as e:
    print(n, "ERR", e)
PY
}
for spec in ${SPECS:-7b 7b_pl 70b_tp1 70b_tp8 70b_tp8_pl 70b_tp4 70b_tp2 70b_tp8_r7 13b}; do
  case $spec in
    7b) run 7b ;;
    7b_pl) run 7b_per_layer --per-layer-launches ;;
    13b) run 13b_sla --config llama2-13b-sla ;;
    70b_tp1) run 70b_tp1 --config llama3-70b-gqa ;;
    70b_tp2) run 70b_tp2_shard --config llama3-70b-gqa --tp-shard 2 ;;
    70b_tp4) run 70b_tp4_shard --config llama3-70b-gqa --tp-shard 4 ;;
    70b_tp8) run 70b_tp8_shard --config llama3-70b-gqa --tp-shard 8 ;;
    70b_tp8_r7) run 70b_tp8_rank7_shard --config llama3-70b-gqa --tp-shard 8 --tp-rank 7 ;;
    70b_tp8_pl) run 70b_tp8_shard_per_layer --config llama3-70b-gqa --tp-shard 8 --per-layer-launches ;;
    7b_model) run 7b_model --model --steps 20 ;;
    13b_model) run 13b_model --model --config llama2-13b-sla --steps 20 ;;
  esac
done
