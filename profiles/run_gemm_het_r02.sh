# whole-tile GEMMs: the mostly idle last wave re-tiled at half the activation width (default) vs
# never (DBK_GEMM_HET=0); parity, GEMM bench on the model shapes, the 7B / 13B model steps
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x tests/test_gpu_gemm.py tests/test_gpu_model.py 2>&1 | tail -2
for het in 0 1; do
  DBK_GEMM_HET=$het timeout 900 python experiments/gemm_bench.py --ms 256,487,512 --shapes 7b_qkv,7b_gu,7b_lm,13b_qkv,13b_gu,70b_tp8_gu --out gpurun_out/het$het.json > /dev/null 2>&1
  for cfg in llama2-7b llama2-13b-sla; do
    DBK_GEMM_HET=$het timeout 900 python bench.py --model --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/het${het}_$cfg.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/het${het}_$cfg.json').read().strip().splitlines()[-1]); print('het=$het $cfg', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
