# GEMM entry-time prefetch (tensormap + first weight boxes into L2) on/off, parity, multirank bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_bench_multirank.py -x -q 2>&1 | tail -3
for pf in 0 1; do
  DBK_GEMM_PREFETCH=$pf timeout 600 python experiments/gemm_bench.py --ms 64,256,512 --shapes 7b_qkv,7b_o,7b_gu,7b_down,70b_tp8_qkv --out gpurun_out/pf$pf.json > /dev/null 2>&1
  DBK_GEMM_PREFETCH=$pf timeout 900 python bench.py --model --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/model_pf$pf.json 2> gpurun_out/model_pf$pf.err
  tail -c 300 gpurun_out/model_pf$pf.json | head -c 0
  python -c "import json;d=json.loads(open('gpurun_out/model_pf$pf.json').read().strip().splitlines()[-1]);print('pf$pf model', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
