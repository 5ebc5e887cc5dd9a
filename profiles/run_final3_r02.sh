# last build check of round 2: the whole GPU suite, smoke(), the default bench line (what the driver runs)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_final3.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], d['e2e']['value'], r['achieved'], r['frac'], r['frac_of_read_probe'], r['traffic_source'], d['clocks'], d['gpu_launches'])"
