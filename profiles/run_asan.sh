#!/bin/bash
# Host sanitizer run: libdbk_asan.so = the host C++ (allocator, request table,
# scheduler, engine, exchange) compiled with -fsanitize=address,undefined (paper_2503_05248_b200/
# build.py --sanitize), and the oracle's C file likewise (DBK_ORACLE_SANITIZE=1).
#   bash profiles/run_asan.sh cpu   # the -m "not gpu" suite (dev box)
#   bash profiles/run_asan.sh gpu   # the toy-sized GPU engine tests (under gpurun; CUDA needs protect_shadow_gap=0)
mode=${1:-cpu}
python paper_2503_05248_b200/build.py --sanitize > /dev/null || exit 1
export LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS=detect_leaks=0:halt_on_error=1:protect_shadow_gap=0:replace_intrin=0
export UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
export DBK_LIB=$PWD/paper_2503_05248_b200/libdbk_asan.so DBK_ORACLE_SANITIZE=1
python - <<'PY'
import os, paper_2503_05248_b200 as dbk  # noqa
maps = open("/proc/self/maps").read()
print("loaded:", "libdbk_asan.so" in maps, "libasan" in maps, "libubsan" in maps)
PY
if [ "$mode" = cpu ]; then
  timeout 1800 python -m pytest -m "not gpu" tests -q -p no:cacheprovider 2>&1 | tail -3
else
  timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "engine or append or chunking or layers" 2>&1 | tail -3
  # (the multi-process GPU tests -- test_gpu_dp_ranks, test_gpu_tp_ranks -- are left out: their spawned
  # children cannot open the device under the ASan runtime, "CUDA-capable device(s) busy or
  # unavailable"; their host logic runs sanitized in the CPU suite's gloo tests)
  timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_gpu_pd.py tests/test_gpu_swap.py tests/test_gpu_e2e.py 2>&1 | tail -3
fi
