# K2 warps x stages variants (DBK_GQA_WS) on the final build, 70B TP1 and TP8 shard
mkdir -p gpurun_out
for ws in default 2x6 8x3 2x3; do for tp in 1 8; do
  extra=""; [ $tp -gt 1 ] && extra="--tp-shard $tp"
  if [ $ws = default ]; then unset DBK_GQA_WS; else export DBK_GQA_WS=$ws; fi
  timeout 600 python bench.py --config llama3-70b-gqa $extra --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tg_${ws}_$tp.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/tg_${ws}_$tp.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$ws tp$tp', d['value'], r['achieved'], r['frac_of_read_probe'], d['clocks']['sm_mhz'])"
done; done
