"""Per-step device time series of one engine run (measurement): are slow runs slow in every step
(layout of the pool in this process) or in some steps (interference)?

  python experiments/step_series.py --config llama3-70b-gqa --tp-shard 8 --ff 200 --steps 200
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3-70b-gqa")
    ap.add_argument("--tp-shard", type=int, default=1)
    ap.add_argument("--ff", type=int, default=200)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--per-layer-launches", action="store_true")
    args = ap.parse_args()
    import torch

    import bench
    torch.cuda.set_device(0)
    S = bench.setup_engine(device=0, cfg_name=args.config, tp=args.tp_shard, time_attention=True,
                           per_layer_launches=args.per_layer_launches)
    eng = S["eng"]
    bufs = eng.buffers(S["qd"], S["od"])
    stream = torch.cuda.current_stream()
    for _ in range(args.ff):
        eng.step(bufs, stream)
    gbs, recs = [], []
    for _ in range(args.steps):
        eng.attn_timing(reset=True)
        rec = eng.step(bufs, stream)
        ms, la, by = eng.attn_timing(reset=True)
        gbs.append(by / 1e9 / (ms / 1e3))
        recs.append(dict(t=rec["t"], ms=round(ms, 3), n=rec["n_decode"], adm=rec["n_admitted"], fin=rec["n_finished"],
                         launches=rec["launches"], kernels=la, step_ms=round(rec["step_ns"] / 1e6, 3)))
    g = np.array(gbs)
    for k in np.argsort(g)[:3]:
        print("slow", round(float(g[k]), 0), json.dumps(recs[k]), "prev", json.dumps(recs[k - 1]) if k else None)
    blocks = [round(float(np.median(g[i:i + 20])), 0) for i in range(0, len(g), 20)]
    print(json.dumps({"kv_ptr_mod_2M": S["pool"].kv.data_ptr() % (1 << 21), "gbs_min": round(float(g.min()), 0),
                      "gbs_median": round(float(np.median(g)), 0), "gbs_max": round(float(g.max()), 0),
                      "block_medians": blocks}))


if __name__ == "__main__":
    main()
