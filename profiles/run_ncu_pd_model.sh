#!/bin/bash
# Launch list of PD fusion through the full model (7B, static b = 256, whole-trace start):
# GEMM / K7 prefill / K1 decode / small-kernel shares of a fused iteration.
mkdir -p gpurun_out
cat > gpurun_out/pd_model_probe.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import bench
S = bench.setup_engine(cfg_name="llama2-7b", policy="static", b_static=256, time_attention=False,
                       pd_fusion=True, full_model=True, n_req=600)
eng = S["eng"]
bufs = eng.buffers(S["qd"], S["od"])
bench.run_steps(S, 40, bufs, torch.cuda.current_stream())
PY
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1500 --csv \
    --log-file gpurun_out/launches_pd_model.csv python gpurun_out/pd_model_probe.py > gpurun_out/ncu_pd_model_stdout.log 2>&1
