# K7: parity (prefill + PD), throughput vs torch SDPA; SYNC=1 adds synccheck on smoke()
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_pd.py -x -q 2>&1 | tail -3
timeout 300 python experiments/prefill_bench.py --out gpurun_out/prefill_bench_r02.json 2>&1 | tail -10 | cut -c1-190
if [ -n "$SYNC" ]; then
timeout 600 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/synccheck_k7.txt 2>&1; echo rc=$? >> gpurun_out/synccheck_k7.txt
tail -3 gpurun_out/synccheck_k7.txt
fi
