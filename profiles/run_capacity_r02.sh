#!/bin/bash
# Capacity (Table II / Fig. 5 analog) with the full 13B model on our own GEMMs:
# static b swept over 128 / 192 / 256 vs Alg. 1 + Alg. 2 (min), without and with PD fusion under
# the survey's reading R25 (chunk = b_t - N^d), D_SLA = tau(b_mem/2) from the Fig. 3 fit, one
# arrival seed, 3 % bisection tolerance.  Output gpurun_out/r02_capacity_model.json.
mkdir -p gpurun_out
timeout ${T:-4200} python experiments/paper_tables.py --model --capacity --cap-config llama2-13b-sla \
    --cap-lo 4 --cap-hi 40 --cap-tol 0.03 --cap-seeds ${SEEDS:-11} --cap-static-bs 128,192,256 \
    --cap-modes ${MODES:-static:nopd,combined:nopd,static:pd,combined:pd} \
    --out gpurun_out/r02_capacity_model.json > gpurun_out/r02_capacity_model.log 2>&1
tail -5 gpurun_out/r02_capacity_model.log
