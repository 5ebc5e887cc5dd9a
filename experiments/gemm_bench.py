"""Throughput of the model GEMM (dbk_gemm: tcgen05 stream-K, cta_group 1 and 2) next to the
library GEMM in the same process (torch.matmul -> cuBLAS) on the decode step's projection
shapes (Llama-2-7B / -13B, Llama-3-70B TP shards) at decode batch sizes.

`reps` launches captured in one CUDA graph (so host launch cost is not measured), CUDA events
around a replay; flops = 2 M N K.  The launches rotate over >= 400 MB of weight copies, so the
weights come from HBM as in the model step, where every layer's weights are read once per step.

    python experiments/gemm_bench.py [--ms 64,128,256,512] [--out profiles/rNN_gemm_bench.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_05248_b200 as dbk  # noqa: E402

SHAPES = {  # name: (N, K)
    "7b_qkv": (12288, 4096), "7b_o": (4096, 4096), "7b_gu": (22016, 4096), "7b_down": (4096, 11008),
    "7b_lm": (32000, 4096),
    "13b_qkv": (15360, 5120), "13b_gu": (27648, 5120), "13b_down": (5120, 13824),
    "70b_tp8_qkv": (1280, 8192), "70b_tp8_gu": (7168, 8192), "70b_tp8_down": (8192, 3584),
}


def time_graph(fn, reps, replays=3):
    """Device time per call of `reps` calls captured in one CUDA graph (no host launch cost),
    best of `replays` replays; fn(i) issues call i on the current stream."""
    for i in range(2):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(replays):
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="64,128,256,487,512")
    ap.add_argument("--shapes", default=",".join(SHAPES))
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default=None)
    ap.add_argument("--trace", action="store_true", help="per-CTA phase stamps of one launch")
    ap.add_argument("--modes", default="f16", help="epilogues to time: f16, silu (gate|up shapes)")
    ap.add_argument("--split", action="store_true", help="also time the operand pipeline alone (no MMAs) "
                    "and the MMAs alone (no operand loads)")
    ap.add_argument("--hot", action="store_true", help="one weight copy (L2-resident when it fits)")
    ap.add_argument("--bn-sweep", default="", help="also time cta_group 2 at these forced tile widths, e.g. 128,192,256")
    ap.add_argument("--trace-modes", default="f16")
    ap.add_argument("--custom", default="", help="extra shapes 'N:K;N:K' named cNxK")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    g1, g2 = dbk.Gemm(0, 1), dbk.Gemm(0, 2)
    res = []
    names = a.shapes.split(",") if a.shapes else []
    for c in filter(None, a.custom.split(";")):
        N, K = (int(v) for v in c.split(":"))
        SHAPES[f"c{N}x{K}"] = (N, K)
        names.append(f"c{N}x{K}")
    for name in names:
        N, K = SHAPES[name]
        # enough weight copies that a call never finds its weights in the 126 MB L2 (the model
        # step reads every layer's weights once)
        copies = 1 if a.hot else max(2, -(-400 * 2 ** 20 // (N * K * 2)))
        ws = [(torch.rand(N, K, device="cuda", dtype=torch.float16) - 0.5) / K ** 0.5 for _ in range(copies)]
        w = ws[0]
        for M in [int(m) for m in a.ms.split(",")]:
            x = torch.rand(M, K, device="cuda", dtype=torch.float16) - 0.5
            y = torch.empty(M, N, device="cuda", dtype=torch.float16)
            fl = 2.0 * M * N * K
            row = {"shape": name, "M": M, "N": N, "K": K}
            row["cublas_ms"] = time_graph(lambda i: torch.matmul(x, ws[i % copies].t(), out=y), a.reps)
            ref = torch.matmul(x.float(), w.float().t())
            for tag, g in (("cg1", g1), ("cg2", g2)):
                if N % (128 * g.cta_group):
                    continue
                row[f"{tag}_ms"] = time_graph(
                    lambda i: g(x, ws[i % copies], y, "f16", stream=torch.cuda.current_stream()), a.reps)
                if a.split:
                    for dm, dn in ((1, "loads_only"), (2, "mma_only")):
                        dbk._lib.dbk_gemm_trace(g.h, None, dm)
                        row[f"{tag}_{dn}_ms"] = time_graph(
                            lambda i: g(x, ws[i % copies], y, "f16", stream=torch.cuda.current_stream()), a.reps)
                        dbk._lib.dbk_gemm_trace(g.h, None, 0)
                for bn in [int(v) for v in a.bn_sweep.split(",") if v]:
                    if tag != "cg2":
                        continue
                    dbk._lib.dbk_gemm_force_tile(g.h, bn)
                    row[f"bn{bn}_ms"] = time_graph(
                        lambda i: g(x, ws[i % copies], y, "f16", stream=torch.cuda.current_stream()), a.reps)
                    dbk._lib.dbk_gemm_force_tile(g.h, 0)
                if "silu" in a.modes.split(","):
                    act = torch.empty(M, N // 2, device="cuda", dtype=torch.float16)
                    row[f"{tag}_silu_ms"] = time_graph(
                        lambda i: g(x, ws[i % copies], act, "silu", stream=torch.cuda.current_stream()), a.reps)
                g(x, w, y, "f16")
                torch.cuda.synchronize()
                row[f"{tag}_maxrel"] = float(((y.float() - ref).abs().max() / ref.abs().max()).item())
            for tmode in (a.trace_modes.split(",") if a.trace else []):
                yt = y if tmode == "f16" else torch.zeros(M, N, device="cuda", dtype=torch.float32)
                for tag0, g in (("cg1", g1), ("cg2", g2)):
                    tag = tag0 if tmode == "f16" else f"{tag0}_{tmode}"
                    tb = torch.zeros(148, 8, dtype=torch.int64, device="cuda")
                    dbk._lib.dbk_gemm_trace(g.h, tb.data_ptr(), 0)
                    g(x, ws[1 % copies], yt, tmode)
                    torch.cuda.synchronize()
                    dbk._lib.dbk_gemm_trace(g.h, None, 0)
                    t = tb.cpu().numpy()
                    t = t[t[:, 0] > 0]
                    t0 = t[:, 0].min()
                    rel = (t - t0) / 1e3
                    med = np.median(rel, axis=0)
                    row[f"{tag}_trace_us"] = {"ctas": int(len(t)), "median_stamps": [round(float(v), 2) for v in med[:8]],
                                              "max_stamps": [round(float(v), 2) for v in rel.max(axis=0)[:8]]}
            for k in list(row):
                if k.endswith("_ms"):
                    row[k.replace("_ms", "_tflops")] = fl / (row[k] * 1e-3) / 1e12
            res.append(row)
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in row.items()}),
                  flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"gpu": torch.cuda.get_device_name(0), "reps": a.reps, "rows": res}, f, indent=1)


if __name__ == "__main__":
    main()
