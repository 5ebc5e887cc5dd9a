# bench default (7B attention-only) and --model, 20 timed steps each
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.err
timeout 900 python bench.py --model --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_model.json 2> gpurun_out/bench_model.err; tail -c 300 gpurun_out/bench_model.err
python - <<'P'
import json
for f in ("gpurun_out/bench_default.json","gpurun_out/bench_model.json"):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["value"], d["ms_per_step"], d["e2e"], d["clocks"]["sm_mhz"])
P
