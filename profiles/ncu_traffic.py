#!/usr/bin/env python
"""Reduce the ncu captures of profiles/run_ncu_traffic.sh to profiles/ncu_traffic.json, the file
bench.py reads for roofline.traffic: per configuration, the decode kernels of ONE engine step
(captured inside the NVTX range dbk_step) -- DRAM read + write bytes per launch, their sum over
the step against the step's algorithmic attention bytes (printed by bench.py --ncu-step), and
the cold-cache serialised duration of each launch.

  python profiles/ncu_traffic.py OUT.json NAME:CSV:STEP_JSON [NAME:CSV:STEP_JSON ...]
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict


def kernels(path):
    rows = defaultdict(dict)
    names = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        k = int(r["ID"])
        names[k] = r["Kernel Name"]
        v = r["Metric Value"].replace(",", "")
        try:
            rows[k][r["Metric Name"]] = float(v)
        except ValueError:
            pass
    return [(names[k], rows[k]) for k in sorted(rows)]


def main():
    out = sys.argv[1]
    build = os.environ.get("DBK_BUILD")  # set by the caller: the GPU box's copy has no .git
    try:
        if not build:
            build = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True,
                                   cwd=os.path.dirname(os.path.abspath(__file__))).stdout.strip() or None
    except OSError:
        build = None
    entries = []
    for spec in sys.argv[2:]:
        name, csv_path, step_path = spec.split(":")
        with open(step_path) as f:
            step = [json.loads(ln)["ncu_step"] for ln in f if ln.startswith('{"ncu_step"')][0]
        ks = [(n, m) for n, m in kernels(csv_path) if step["kernel"] + "<" in n]
        if not ks:
            print(f"{name}: no {step['kernel']} launches in {csv_path}", file=sys.stderr)
            continue
        dram = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for _, m in ks]
        dur = [m.get("gpu__time_duration.sum", 0) for _, m in ks]
        alg = step["attn_bytes"]
        entries.append({
            "name": name, "config": step["config"], "tp": step["tp"], "model": step["model"],
            "kernel": step["kernel"], "kernel_name": ks[0][0], "launches": len(ks),
            "per_layer_launches": step["per_layer_launches"], "n_decode": step["n_decode"],
            "chunk_pages": step["chunk_pages"],
            "dram_bytes_per_launch": int(sum(dram) / len(ks)),
            "algorithmic_bytes_per_launch": int(alg / len(ks)),
            "traffic_over_algorithmic": round(sum(dram) / alg, 4) if alg else None,
            "ncu_duration_us_per_launch": round(sum(dur) / len(ks) / 1e3, 2),
            "ncu_dram_tbps": round(sum(dram) / sum(dur) / 1e3, 3) if sum(dur) else None,
            "file": os.path.basename(csv_path), "build": build})
    with open(out, "w") as f:
        json.dump({"how": "profiles/run_ncu_traffic.sh: ncu --nvtx --nvtx-include dbk_step/ --metrics "
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none "
                          "python bench.py --ncu-step ... (one steady-state engine step per configuration)",
                   "entries": entries}, f, indent=1)
    for e in entries:
        print(json.dumps(e))


if __name__ == "__main__":
    main()
