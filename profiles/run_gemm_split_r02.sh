# GEMM split-K for the whole-tile epilogues (few tiles, M <= 256): parity (GEMM + model + TP model), gemm_bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py tests/test_gpu_tp_model.py -x -q 2>&1 | tail -3
timeout 600 python experiments/gemm_bench.py --ms 64,256,512 --out gpurun_out/gemm_bench_r02.json 2>&1 | tail -40 | cut -c1-130
