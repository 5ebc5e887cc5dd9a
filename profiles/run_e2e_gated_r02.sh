# end-to-end steps: per-layer readiness flags (in-kernel acquire) instead of stream events between
# the chained decode launches, outputs written zero-copy into the pinned host rows
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_e2e.py tests/test_gpu_bench_multirank.py 2>&1 | tail -2
timeout 300 python experiments/e2e_probe.py > gpurun_out/e2e_probe_gated.json 2>&1; cat gpurun_out/e2e_probe_gated.json | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v['ms_per_step'],3) for k,v in d.items()})"
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_gated_bench.json 2> gpurun_out/e2e_gated_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/e2e_gated_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e'], d['clocks']['sm_mhz'])"
