# K2: a last page holding <= 8 tokens moves only its first 8 K/V rows (8-row TMA boxes)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "gqa" tests/test_gpu_tp_ranks.py 2>&1 | tail -2
for hb in 0 1; do for tp in 1 8; do
  extra=""; [ $tp -gt 1 ] && extra="--tp-shard $tp"
  DBK_GQA_HALF=$hb timeout 900 python bench.py --config llama3-70b-gqa $extra --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/k2p_${hb}_tp$tp.json 2> gpurun_out/k2p_${hb}_tp$tp.err
  python -c "
import json; d=json.loads(open('gpurun_out/k2p_${hb}_tp$tp.json').read().strip().splitlines()[-1]); r=d['roofline']; print('part=$hb tp$tp', d['value'], d['ms_per_step'], r['achieved'], r['frac'], r.get('frac_of_read_probe'), d['clocks']['sm_mhz'])"
done; done
