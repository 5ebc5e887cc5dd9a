"""Task timeline of the decode kernels (K1 / K2) over one engine step (measurement only).

  DBK_TRACE_TASKS is set here before the pool exists; every warp task then appends a record
  (start, end in %globaltimer ns; SM; launch; task; pages).  Prints, for the traced step, per
  launch: span, the gap to / overlap with the previous launch, the warp-busy fraction
  (sum of task time / (resident warps x span)), and over the whole step the fraction of
  warp-time spent in tasks -- where the attention window is lost (ramp, drain, gaps).

  python experiments/trace_tasks.py --config llama3-70b-gqa --tp-shard 8 [--ff 200] [--json out]
"""
from __future__ import annotations

import argparse
import ctypes
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
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    os.environ["DBK_TRACE_TASKS"] = str(1 << 22)
    import torch

    import bench
    torch.cuda.set_device(0)
    S = bench.setup_engine(device=0, cfg_name=args.config, tp=args.tp_shard, time_attention=True)
    eng, pool, dbk = S["eng"], S["pool"], S["dbk"]
    bufs = eng.buffers(S["qd"], S["od"])
    stream = torch.cuda.current_stream()
    for _ in range(args.ff):
        eng.step(bufs, stream)
    for _ in range(3):
        eng.step(bufs, stream)
    n = ctypes.c_int64()
    dbk._lib.dbk_pool_trace_d2h(pool.h, None, 0, ctypes.byref(n), 1)  # reset
    eng.attn_timing(reset=True)
    rec = eng.step(bufs, stream)
    att_ms, att_launches, att_bytes = eng.attn_timing(reset=True)
    cap = 1 << 22
    buf = np.zeros((cap, 4), np.uint64)
    dbk._lib.dbk_pool_trace_d2h(pool.h, buf.ctypes.data, cap, ctypes.byref(n), 1)
    r = buf[:n.value]
    t0, t1 = r[:, 0].astype(np.int64), r[:, 1].astype(np.int64)
    sm = (r[:, 2] >> np.uint64(32)).astype(np.int64)
    seq = (r[:, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    pages = (r[:, 3] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    base = t0.min()
    t0, t1 = t0 - base, t1 - base
    info = pool.info()
    warps = 148 * 8  # resident warps of the persistent grid (8 per SM in every variant measured)
    launches = sorted(set(seq.tolist()))
    rows = []
    prev_end = None
    for L in launches:
        m = seq == L
        a, b = int(t0[m].min()), int(t1[m].max())
        busy = float((t1[m] - t0[m]).sum())
        # time until 90 % of this launch's warps-with-work have finished their last task
        ends = np.sort(t1[m])
        rows.append(dict(launch=L, start_us=a / 1e3, end_us=b / 1e3, span_us=(b - a) / 1e3,
                         gap_us=None if prev_end is None else (a - prev_end) / 1e3,
                         tasks=int(m.sum()), pages=int(pages[m].sum()),
                         busy_frac=busy / (warps * (b - a)) if b > a else None,
                         tail_us=(b - ends[int(0.9 * len(ends))]) / 1e3))
        prev_end = b
    # concurrency: tasks in flight per SM, sampled at 200 instants of the step
    inst = np.linspace(t0.min(), t1.max(), 200)
    conc = []
    for x in inst:
        live = (t0 <= x) & (t1 > x)
        if live.any():
            conc.append(np.bincount(sm[live], minlength=148).max())
    max_per_sm = int(max(conc)) if conc else 0
    total_span = (t1.max() - t0.min()) / 1e3
    busy_all = float((t1 - t0).sum()) / (warps * (t1.max() - t0.min()))
    out = dict(config=args.config, tp=args.tp_shard, decode_path=info["decode_path"], chunk_pages=info["chunk_pages"],
               step=dict(n_decode=rec["n_decode"], step_ms=rec["step_ns"] / 1e6, attn_ms_events=att_ms,
                         attn_bytes=att_bytes, launches=att_launches),
               trace_span_us=total_span, warp_busy_frac=busy_all, tasks=int(len(r)), max_tasks_per_sm=max_per_sm,
               sms_used=int(len(set(sm.tolist()))),
               pages_per_task_mean=float(pages.mean()), task_us_mean=float((t1 - t0).mean() / 1e3),
               task_us_p90=float(np.percentile(t1 - t0, 90) / 1e3),
               launches=rows)
    spans = [x["span_us"] for x in rows]
    gaps = [x["gap_us"] for x in rows if x["gap_us"] is not None]
    print(json.dumps({k: v for k, v in out.items() if k != "launches"}, indent=1))
    print(f"launch span us: mean {np.mean(spans):.1f} min {np.min(spans):.1f} max {np.max(spans):.1f}; "
          f"start-to-prev-end gap us: mean {np.mean(gaps):.2f} (negative = overlap)")
    print("first launches:")
    for x in rows[:4] + rows[-2:]:
        print(json.dumps(x))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
