# final-build check after the late round-2 changes: GPU suite, smoke(), default bench line, model bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
timeout 900 python bench.py --model --steps 20 --warmup 5 > gpurun_out/bench_model_final2.json 2> gpurun_out/bench_model_final2.err
for f in bench_final2 bench_model_final2; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'], d['gpu_launches'])"; done
