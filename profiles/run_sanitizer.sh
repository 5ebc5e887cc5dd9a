#!/bin/bash
# compute-sanitizer on toy-sized runs of every kernel (SURVEY.md §4 tier 2 / §5): smoke()
# (K1, K2, K7, the model step's kernels: norms, tcgen05 GEMMs), the toy engines (device-resident, PD
# fusion, swap preemption).  Run under gpurun from the repo root.
mkdir -p gpurun_out
out=gpurun_out/sanitizer.txt
: > $out
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool: smoke()" >> $out
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -6 >> $out
done
echo "== memcheck: toy engines (parity tests)" >> $out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -x -q \
  tests/test_gpu_parity.py::test_engine_toy_memory_policy_replays_bit_exact \
  tests/test_gpu_pd.py tests/test_gpu_swap.py::test_engine_swap_preemption_replays 2>&1 | tail -8 >> $out
echo "== memcheck: GEMM split-K (workspace, arrival counters) and the model step through it; e2e engine steps" >> $out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -x -q \
  "tests/test_gpu_gemm.py::test_gemm_split_k_few_tiles" tests/test_gpu_model.py::test_model_step_split_k_epilogues \
  tests/test_gpu_e2e.py 2>&1 | tail -8 >> $out
echo "== racecheck: GEMM split-K" >> $out
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -x -q \
  "tests/test_gpu_gemm.py::test_gemm_split_k_few_tiles[cg2-64]" 2>&1 | tail -6 >> $out
cat $out
