# final-build check: the whole GPU suite, smoke(), the default bench line, racecheck on the CTA-pair vs single-CTA GEMM
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'], d['gpu_launches'])"
for cg in cg1 cg2; do echo "racecheck $cg"; timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python -m pytest -x -q "tests/test_gpu_gemm.py::test_gemm_swiglu_epilogue[$cg]" "tests/test_gpu_gemm.py::test_gemm_split_k_few_tiles[$cg-64]" 2>&1 | grep -E "SUMMARY|passed|failed"; done
