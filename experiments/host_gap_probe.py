"""Where the attention-only step's non-attention time goes: device time of the step (CUDA events
inside the engine, step_ns) vs the timed region's wall on the stream (CUDA events around K steps),
and the host time of one engine call (decision, admission, metadata, launches, the stats sync).

    python experiments/host_gap_probe.py [--steps 50]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--config", default="llama2-7b")
args = ap.parse_args()
S = bench.setup_engine(cfg_name=args.config)
eng = S["eng"]
stream = torch.cuda.current_stream()
bufs = eng.buffers(S["qd"], S["od"])
bench.run_steps(S, 300, bufs, stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
host = []
recs = []
e0.record(stream)
for _ in range(args.steps):
    t = time.perf_counter()
    recs.append(eng.step(bufs, stream))
    host.append(time.perf_counter() - t)
e1.record(stream)
torch.cuda.synchronize()
wall = e0.elapsed_time(e1)
dev = sum(r["step_ns"] for r in recs) / 1e6
att_ms, _, _ = eng.attn_timing(reset=True)
out = {"config": args.config, "steps": len(recs), "stream_wall_ms_per_step": wall / len(recs),
       "device_step_ms_per_step": dev / len(recs), "attention_ms_per_step": att_ms / len(recs),
       "gap_ms_per_step": (wall - dev) / len(recs), "host_call_ms_mean": 1e3 * sum(host) / len(host),
       "host_call_ms_min": 1e3 * min(host), "n_decode_mean": sum(r["n_decode"] for r in recs) / len(recs)}
print(json.dumps(out, indent=1))
