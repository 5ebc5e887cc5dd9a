# decode page ids from the device block table: decode/engine parity + bench; racecheck/initcheck details on smoke()
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dp_ranks.py tests/test_gpu_tp_ranks.py tests/test_gpu_swap.py tests/test_gpu_e2e.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 900 compute-sanitizer --tool initcheck --print-limit 6 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/initcheck.txt 2>&1; grep -v "Host Frame" gpurun_out/initcheck.txt | head -60 | cut -c1-200
