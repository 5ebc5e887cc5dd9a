# model step: the attention launched behind the QKV GEMM streams every page but each request's last
# one before its grid-dependency wait
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_gpu_model.py tests/test_gpu_pd.py tests/test_gpu_tp_model.py 2>&1 | tail -2
for i in 1 2; do
timeout 900 python bench.py --model --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/mp_bench$i.json 2> gpurun_out/mp_bench$i.err
python -c "
import json; d=json.loads(open('gpurun_out/mp_bench$i.json').read().strip().splitlines()[-1]); r=d['roofline']; print('model', d['value'], d['ms_per_step'], r['achieved'], r['frac_of_read_probe'], r['share_of_step'], d['clocks']['sm_mhz'])"
done
