mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "generator or toy or shapes or bench_config_sampled" tests/test_gpu_e2e.py 2>&1 | tail -2
timeout 600 ncu --nvtx --nvtx-include "dbk_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/synth_ncu.csv python bench.py --ncu-step --warmup 3 --no-cpu-baseline --ff 300 > /dev/null 2>&1
grep gpu__time_duration gpurun_out/synth_ncu.csv | awk -F'","' '{print $7, $NF}' | cut -c1-120
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/synth_bench.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/synth_bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print('bench', d['value'], d['ms_per_step'], r['share_of_step'], r['frac_of_read_probe'], d['clocks']['sm_mhz'])"
