# e2e path: parity tests, then the bench line (attention-only 7B) and the e2e probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_bench_multirank.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['gpu_launches'])"
timeout 600 python experiments/e2e_probe.py 2>&1 | tail -26 | tr -d '\n' | tr -s ' '; echo
