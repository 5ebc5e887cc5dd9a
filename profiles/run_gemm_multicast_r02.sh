mkdir -p gpurun_out
export DBK_GEMM_SPLIT=1
echo "== forced NP=2 parity"; DBK_GEMM_NP=2 timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -x -q 2>&1 | tail -5
echo "== bench NP=1"; DBK_GEMM_NP=1 timeout 600 python experiments/gemm_bench.py --ms 256,512 --shapes 7b_qkv,7b_o,7b_gu,7b_down,7b_lm,13b_qkv,13b_gu,13b_down,70b_tp8_gu,70b_tp8_down --out gpurun_out/mc_np1.json 2>&1 | tail -3
echo "== bench NP=2"; DBK_GEMM_NP=2 timeout 600 python experiments/gemm_bench.py --ms 256,512 --shapes 7b_qkv,7b_o,7b_gu,7b_down,7b_lm,13b_qkv,13b_gu,13b_down,70b_tp8_gu,70b_tp8_down --out gpurun_out/mc_np2.json 2>&1 | tail -3
