"""Host-observed latency of one statistics exchange at one rank (measurement): libdbk's mailbox
(one exchange kernel writing the gathered records into mapped host memory + the stream sync)
vs libdbk's NCCL path (record H2D, ncclAllGather, D2H, sync).  At one rank neither crosses
NVLink, so this isolates the fixed per-step cost each transport adds to the host loop.

  python experiments/exchange_latency.py [--iters 2000]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2000)
    args = ap.parse_args()
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2503_05248_b200 as dbk
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29611")
    dist.init_process_group("gloo", rank=0, world_size=1)
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    rec = {f: i + 1 for i, f in enumerate(dbk._lib.STATS_FIELDS)}
    out = {}
    mb = dbk.Mailbox(dist, 1, 0, 0)
    comm = dbk.Comm(dist, 1, 0, 0)
    st = dbk.dbk_stats(*[rec[f] for f in dbk._lib.STATS_FIELDS])
    allb = (dbk.dbk_stats * 1)()
    g = dbk.dbk_stats()
    for name, fn in (("mailbox", lambda: mb.exchange(rec, 0, stream)),
                     ("nccl", lambda: dbk._lib.dbk_stats_allgather(comm.h, ctypes.byref(st), allb, ctypes.byref(g), 0,
                                                                   stream.cuda_stream))):
        for _ in range(100):
            fn()
        ts = []
        for _ in range(args.iters):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        ts = np.array(ts) * 1e6
        out[name] = {"us_median": round(float(np.median(ts)), 2), "us_p99": round(float(np.percentile(ts, 99)), 2)}
    print(json.dumps({"exchange_latency_1rank": out, "iters": args.iters}))
    mb.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
