#!/usr/bin/env python
"""K7 (chunked-prefill attention, tcgen05) throughput vs the dense tensor-core peak.

  python experiments/prefill_bench.py [--out gpurun_out/prefill_bench.json]

For each shape: n prompts of S tokens whose K/V are in the paged pool (synthetic), one
dbk_prefill_step over chunks [q_start, S) timed with CUDA events (median of reps);
algorithmic flops = 4 d Hq sum_rows (p + 1) (QK^T + PV over the causal triangle).  For
context, torch SDPA (library flash/cuDNN kernels, dense contiguous K/V, no paging) on the
same causal problem when q_start = 0.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _peak_tflops():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        if "bf16_tflops" in m:  # burst figure: the kernel is timed alone
            return float(m["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (cuBLAS burst)"
    except OSError:
        pass
    return 2250.0, "nominal (B200_PROFILING.md fallback)"


def run_shape(dbk, torch, Hq, Hkv, d, n, S, q_start, reps=20, dtype="bf16"):
    P = 16
    pages = -(-S // P)
    cap = n * pages + 4
    pool = dbk.KVPool(1, Hq, Hkv, d, cap, n + 1, pages + 1, dtype)
    ids = np.arange(n, dtype=np.int64) + 1
    for r in ids:
        pool.request_begin(r, S, 1)
    pool.append_tokens(ids, [S] * n, seed=1)
    q_len = S - q_start
    rows = n * q_len
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    q = (torch.randn(rows, Hq, d, device="cuda") * 0.5).to(tdt)
    out = torch.empty(rows, Hq, d, dtype=tdt, device="cuda")
    odt = 1 if dtype == "bf16" else 0
    starts, lens = [q_start] * n, [q_len] * n
    for _ in range(3):
        pool.prefill_step(ids, starts, lens, 0, q, out, out_dtype=odt)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    st = torch.cuda.current_stream()
    for k in range(reps):
        ev[2 * k].record(st)
        pool.prefill_step(ids, starts, lens, 0, q, out, out_dtype=odt, stream=st)
        ev[2 * k + 1].record(st)
    torch.cuda.synchronize()
    ms = float(np.median([ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(reps)]))
    flops = 4.0 * d * Hq * n * sum(p + 1 for p in range(q_start, S))
    res = dict(Hq=Hq, Hkv=Hkv, d=d, n=n, S=S, q_start=q_start, ms=ms, tflops=flops / ms / 1e9)
    pool.close()
    if q_start == 0:
        qq = torch.randn(n, Hq, S, d, device="cuda", dtype=tdt)
        kk = torch.randn(n, Hkv, S, d, device="cuda", dtype=tdt)
        vv = torch.randn(n, Hkv, S, d, device="cuda", dtype=tdt)
        f = torch.nn.functional.scaled_dot_product_attention
        kw = dict(is_causal=True, enable_gqa=Hq != Hkv)
        for _ in range(3):
            f(qq, kk, vv, **kw)
        torch.cuda.synchronize()
        for k in range(reps):
            ev[2 * k].record(st)
            f(qq, kk, vv, **kw)
            ev[2 * k + 1].record(st)
        torch.cuda.synchronize()
        ms2 = float(np.median([ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(reps)]))
        res.update(sdpa_ms=ms2, sdpa_tflops=flops / ms2 / 1e9)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/prefill_bench.json")
    ap.add_argument("--shape", type=int, default=-1, help="run only this shape index")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dtypes", default="f16,bf16", help="KV / q dtypes (the bench configs are fp16)")
    a = ap.parse_args()
    import torch

    import paper_2503_05248_b200 as dbk
    torch.cuda.set_device(0)
    peak, src = _peak_tflops()
    shapes = [  # (Hq, Hkv, d, n, S, q_start)
        (32, 32, 128, 8, 2048, 0),     # Llama-2-7B heads, 8 prompts of 2k
        (32, 32, 128, 4, 4096, 0),
        (32, 32, 128, 16, 1024, 512),  # chunked: second half of 1k prompts
        (64, 8, 128, 8, 2048, 0),      # Llama-3-70B heads (GQA 8)
        (40, 40, 128, 8, 2048, 0),     # Llama-2-13B heads
    ]
    rows = []
    if a.shape >= 0:
        shapes = [shapes[a.shape]]
    for dt in a.dtypes.split(","):
        for s in shapes:
            r = run_shape(dbk, torch, *s, reps=a.reps, dtype=dt)
            r["dtype"] = dt
            r["frac_of_peak"] = r["tflops"] / peak
            rows.append(r)
            print(json.dumps(r), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(dict(peak_tflops=peak, peak_source=src, rows=rows), f, indent=1)


if __name__ == "__main__":
    main()
