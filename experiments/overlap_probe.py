#!/usr/bin/env python
"""Measurement probe for the model step's attention / GEMM overlap (DESIGN.md §10b item 4).

Two micro-batches of 256 decode rows (Llama-2-7B layer shapes): can one micro-batch's paged
attention (HBM-bound, K1) run on part of the SMs while the other micro-batch's projections
(tensor-core bound at M = 256) run on the rest, and how much of the serial time does that save?

  * attention of one micro-batch alone with its grid capped to S SMs (DBK_DECODE_SMS)
  * one micro-batch's GEMM block (O, gate|up + SiLU, down, QKV) alone, capped to 148 - S SMs
  * both at once on two streams (GEMMs issued first so their CTAs hold their SMs)

    python experiments/overlap_probe.py [--splits 148,104,96,88,80] [--out gpurun_out/overlap_probe.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--splits", default="148,112,104,96,88,80,72")
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/overlap_probe.json")
    a = ap.parse_args()
    import paper_2503_05248_b200 as dbk
    torch.cuda.set_device(0)
    H, F, Hq, d = 4096, 11008, 32, 128
    n = a.rows
    rng = np.random.default_rng(5)
    ctx = rng.integers(1, 790, n).astype(np.int32)   # mean ~395: configs[1]'s context mix
    pages = int(sum(-(-ctx // 16))) + 8
    ids = np.arange(n, dtype=np.int64) + 1
    dev_sms = torch.cuda.get_device_properties(0).multi_processor_count

    def make_pool(sms):
        if sms < dev_sms:
            os.environ["DBK_DECODE_SMS"] = str(sms)
        else:
            os.environ.pop("DBK_DECODE_SMS", None)
        p = dbk.KVPool(1, Hq, Hq, d, pages, n + 1, int(ctx.max()) // 16 + 2, "f16")
        for r, c in zip(ids, ctx):
            p.request_begin(int(r), int(c), 1)
        p.append_tokens(ids, ctx, seed=3)
        return p

    def make_gemm(sms):
        if sms < dev_sms:
            os.environ["DBK_GEMM_SMS"] = str(sms)
        else:
            os.environ.pop("DBK_GEMM_SMS", None)
        g = dbk.Gemm(0, 2)
        os.environ.pop("DBK_GEMM_SMS", None)
        return g

    q = (torch.randn(n, Hq, d, device="cuda") * 0.5).half()
    out = torch.empty(n, Hq, d, device="cuda", dtype=torch.float16)
    # weights of one layer, several copies so a block never finds them in L2
    copies = 2
    W = [dict(qkv=torch.randn(3 * H, H, device="cuda").half() * 0.02, o=torch.randn(H, H, device="cuda").half() * 0.02,
              gu=torch.randn(2 * F, H, device="cuda").half() * 0.02, down=torch.randn(H, F, device="cuda").half() * 0.02)
         for _ in range(copies)]
    x = torch.randn(n, H, device="cuda").half()
    xa = torch.randn(n, F, device="cuda").half()
    res = torch.zeros(n, H, device="cuda")
    yq = torch.empty(n, 3 * H, device="cuda", dtype=torch.float16)
    act = torch.empty(n, F, device="cuda", dtype=torch.float16)

    def gemm_block(g, i, s):
        w = W[i % copies]
        g(x, w["o"], res, "acc32", stream=s)
        g(x, w["gu"], act, "silu", stream=s)
        g(xa, w["down"], res, "acc32", stream=s)
        g(x, w["qkv"], yq, "f16", stream=s)

    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]

    def timed(fn, reps):
        fn(0)
        torch.cuda.synchronize()
        ts = []
        for i in range(reps):
            torch.cuda.synchronize()
            ev[0].record()
            fn(i)
            ev[1].record()
            ev[1].synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        return float(np.median(ts))

    kv_bytes = float(np.sum(ctx)) * 2 * Hq * d * 2
    rows = []
    for S in [int(v) for v in a.splits.split(",")]:
        pool = make_pool(S)
        G = dev_sms - S if S < dev_sms else dev_sms
        g = make_gemm(G)
        att = lambda i, s=None: pool.decode_step(ids, 0, q, out, out_dtype=0, stream=s)  # noqa: E731
        t_att = timed(lambda i: att(i), a.reps)
        t_gemm = timed(lambda i: gemm_block(g, i, None), a.reps)
        row = {"attn_sms": S, "gemm_sms": G, "attn_ms": t_att, "attn_tbs": kv_bytes / t_att / 1e9,
               "gemm_block_ms": t_gemm}
        if S < dev_sms:
            def both(i):
                cur = torch.cuda.current_stream()
                s1.wait_stream(cur)
                s2.wait_stream(cur)
                with torch.cuda.stream(s2):
                    gemm_block(g, i, s2)
                with torch.cuda.stream(s1):
                    att(i, s1)
                cur.wait_stream(s1)
                cur.wait_stream(s2)
            row["both_ms"] = timed(both, a.reps)
            row["serial_ms"] = t_att + t_gemm
        rows.append(row)
        print(json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in row.items()}), flush=True)
        pool.close()
        g.close()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"rows_per_microbatch": n, "kv_bytes": kv_bytes, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
