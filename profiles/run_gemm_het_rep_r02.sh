mkdir -p gpurun_out
for rep in a b; do for het in 0 1; do
  DBK_GEMM_HET=$het timeout 900 python experiments/gemm_bench.py --ms 256,487,512 --shapes 7b_gu,7b_lm,13b_qkv,13b_gu,70b_tp8_gu --out gpurun_out/het${het}_$rep.json > /dev/null 2>&1
done; done
