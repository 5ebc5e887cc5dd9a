# GEMM split-K (per-K-range fp32 workspace slices, distributed reduction + epilogue): parity, then gemm_bench with and without
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py tests/test_gpu_tp_model.py -x -q 2>&1 | tail -3
timeout 600 python experiments/gemm_bench.py --ms 64,256,512 --out gpurun_out/gemm_bench_split.json 2>&1 | tail -1 | cut -c1-100
DBK_GEMM_SPLIT=0 timeout 600 python experiments/gemm_bench.py --ms 64,256,512 --out gpurun_out/gemm_bench_nosplit.json 2>&1 | tail -1 | cut -c1-100
