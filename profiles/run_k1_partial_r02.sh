# K1: the last partly filled page of each request reads only its valid K/V rows (no page padding over HBM)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_e2e.py 2>&1 | tail -2
for i in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/k1p_bench$i.json 2> gpurun_out/k1p_bench$i.err
python -c "
import json; d=json.loads(open('gpurun_out/k1p_bench$i.json').read().strip().splitlines()[-1]); r=d['roofline']; print('bench', d['value'], d['ms_per_step'], r['achieved'], r['frac'], r.get('frac_of_read_probe'), d['clocks']['sm_mhz'])"
done
timeout 1200 ncu --nvtx --nvtx-include "dbk_step/" --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/k1p_ncu_7b.csv python bench.py --ncu-step --warmup 3 --no-cpu-baseline --ff 300 > gpurun_out/k1p_ncu_7b.json 2> gpurun_out/k1p_ncu_7b.err
tail -4 gpurun_out/k1p_ncu_7b.csv
