# paper experiments on the final build: Table I analog with the full 7B model (own GEMMs), the 13B model bench line,
# and a re-measure of one GEMM point (70B-TP8 gate|up at M = 256)
mkdir -p gpurun_out
timeout 300 python experiments/gemm_bench.py --ms 256 --shapes 70b_tp8_gu --bn-sweep 128,256 --out gpurun_out/gemm_tp8gu.json 2>&1 | tail -1 | cut -c1-300
timeout 900 python bench.py --model --config llama2-13b-sla --no-cpu-baseline > gpurun_out/r02_bench_13b_model.json 2> gpurun_out/r02_bench_13b_model.err
python -c "
import json; d=json.loads(open('gpurun_out/r02_bench_13b_model.json').read().strip().splitlines()[-1]); print('13b model', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'])"
timeout 2400 python experiments/paper_tables.py --table1 --model --out gpurun_out/r02_table1_model.json > gpurun_out/r02_table1_model.log 2>&1; tail -6 gpurun_out/r02_table1_model.log | cut -c1-200
