#!/usr/bin/env python
"""B200 analogs of the paper's experiments on the decode hot path.

  python experiments/paper_tables.py [--fig3] [--table1] [--sla] [--out gpurun_out/paper_tables.json]

* --fig3   : static-b sweep on the Llama-2-7B shape (steady state after a fast-forward):
             tau_step(b) and Phi(b) = b / tau_step(b) (Eq. 6), OLS fit tau = a0 + a1 b
             (Fig. 3).  Attention-only step: no weights, so a0 is small.
* --table1 : whole-trace throughput (generated tokens / total device time, all-at-once
             arrivals) for static b in {64, 128, 256} vs the memory-aware rule (Alg. 1),
             the shape of Table I row 3 -- attention-only.
* --sla    : the SLA feedback (Alg. 2 + min with Alg. 1) on the 13B shape with a binding
             D_SLA = tau(b_mem / 2) from the sweep's fit, and the literal 50 ms.
* --pd-model: the PD table with the full model: prompts prefilled through the weights.
* --swap   : preemption by swapping vs recomputation (NEXT row 4) on the 7B shape with a
             40 GB KV cap: static b = 256 over-commits it (recompute / swap to a 16 GB pinned
             host space) vs the memory-aware rule, which keeps the batch under the cap.
Every run goes through the C-ABI engine; numbers are device-timed (CUDA events).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


FULL_MODEL = False  # --model: every run is the whole decode step with synthetic weights (NEXT row 3)


def _run(cfg, policy, b_static=256, sla_ms=None, ff=300, steps=40, full=False, n_req=None):
    import gc

    import torch
    gc.collect()
    torch.cuda.empty_cache()
    S = bench.setup_engine(cfg_name=cfg, policy=policy, b_static=b_static, sla_ms=sla_ms, time_attention=False,
                           n_req=n_req, full_model=FULL_MODEL)
    eng = S["eng"]
    bufs = eng.buffers(S["qd"], S["od"])
    stream = torch.cuda.current_stream()
    t0 = time.time()
    if full:
        recs, ms = bench.run_steps(S, 10 ** 9, bufs, stream)
    else:
        bench.run_steps(S, ff, bufs, stream)
        recs, ms = bench.run_steps(S, steps, bufs, stream)
    out = dict(policy=policy, b_static=b_static if policy == "static" else None, sla_ms=sla_ms,
               steps=len(recs), device_ms=ms, tokens=int(sum(r["n_decode"] for r in recs)),
               mean_batch=float(np.mean([r["n_decode"] for r in recs])),
               mean_step_ms=float(np.mean([r["step_ns"] for r in recs]) / 1e6),
               preemptions=int(sum(r["n_preempted"] for r in recs)), wall_s=time.time() - t0)
    out["tokens_per_s"] = out["tokens"] / (ms / 1e3)
    if not full:
        out["b_trace_tail"] = [r["b_next"] for r in recs[-10:]]
    out["full_model"] = FULL_MODEL
    S["eng"].close()
    if S.get("model") is not None:
        S["model"].close()
    S["pool"].close()
    S.clear()
    return out


def fig3(cfg="llama2-7b", bs=(16, 32, 64, 128, 192, 256, 384, 512)):
    rows = [_run(cfg, "static", b_static=b) for b in bs]
    b = np.array([r["mean_batch"] for r in rows])
    tau = np.array([r["mean_step_ms"] for r in rows])
    a1, a0 = np.polyfit(b, tau, 1)
    return dict(config=cfg, rows=rows, fit=dict(a0_ms=float(a0), a1_ms=float(a1)),
                phi=[float(x) for x in 1000.0 * b / tau])


def table1(cfg="llama2-7b"):
    rows = [_run(cfg, "static", b_static=b, full=True) for b in (64, 128, 256)]
    rows.append(_run(cfg, "memory", full=True))
    return dict(config=cfg, rows=rows)


def sla(fit=None, cfg="llama2-13b-sla"):
    rows = [_run(cfg, "combined", sla_ms=50.0, ff=200, steps=60)]
    if fit is not None:
        rows.append(_run(cfg, "combined", sla_ms=fit, ff=200, steps=60))
    return dict(config=cfg, rows=rows)


def _tbt_p99(recs):
    """p99 time between tokens over all generated tokens (every token of a step waits the
    step's latency; nearest rank)."""
    lat = np.array([r["step_ns"] for r in recs], np.float64) / 1e6
    w = np.array([r["n_decode"] for r in recs], np.int64)
    order = np.argsort(lat)
    cum = np.cumsum(w[order])
    k = int(np.ceil(0.99 * cum[-1]))
    return float(lat[order][np.searchsorted(cum, k)])


def capacity(cfg="llama2-13b-sla", d_sla=None, eps_d=None, window_s=20.0,
             modes=(("static", False), ("combined", False), ("static", True), ("combined", True)),
             b_static=None, lo=10.0, hi=640.0, tol=0.05, max_delay_s=2.0, ctrl_margin_ms=0.0, pd_token_budget=0,
             seeds=(None,), static_bs=None):
    """Table II / Fig. 5 analog: capacity = the largest Poisson rate (qps) at which
    the p99 TBT stays <= D_SLA + eps_D AND the median scheduling delay (arrival -> first
    admission, from dbk_engine_request_times) stays <= 2 s -- Sarathi-Serve's definition, which
    the paper adopts -- found by bisection on the rate, for the static baseline and for
    Alg. 2 + Alg. 1, without and with PD fusion (Table II row 3 "implemented with PD fusion
    scenario").  Each probe sends qps x window_s requests (a fixed arrival window).

    Round 2: the bisection runs once per arrival seed (`seeds`: the trace's length
    seed is fixed, the Poisson arrival stream varies) and reports the capacity per seed plus
    mean / min / max, to a tolerance `tol`; `static_bs` sweeps the static baseline over several b
    under the same SLA so the comparison is against the BEST static b, not one setting.
    ctrl_margin_ms != 0 steers Alg. 2 below the SLA it is judged at -- NOT the paper's Alg. 2
    (P:221-248); rows record it."""
    from synth import configs, trace
    c = configs.CONFIGS[cfg]
    t = c["trace"]
    out = dict(config=cfg, d_sla_ms=d_sla, eps_d_ms=eps_d, window_s=window_s, max_delay_s=max_delay_s,
               ctrl_margin_ms=ctrl_margin_ms, pd_token_budget=pd_token_budget, rows=[])

    def probe(policy, pd, qps, seed=None, bst=None):
        n_req = max(100, int(qps * window_s))
        tr = trace.make_trace(n_req, t["mean_in"], t["mean_out"], t["L_max"], t["seed"], dist=t["dist"],
                              arrival="poisson", rate_qps=qps, arrival_seed=seed)
        import gc

        import torch
        gc.collect()
        torch.cuda.empty_cache()
        S = bench.setup_engine(cfg_name=cfg, policy=policy, b_static=bst or b_static or 256, sla_ms=d_sla - ctrl_margin_ms,
                               eps_d_ms=eps_d, time_attention=False, trace_override=tr, pd_fusion=pd,
                               full_model=FULL_MODEL, pd_token_budget=pd_token_budget if pd else 0)
        eng = S["eng"]
        bufs = eng.buffers(S["qd"], S["od"])
        recs, ms = bench.run_steps(S, 10 ** 9, bufs, torch.cuda.current_stream())
        adm, fin = eng.request_times()
        delay = float(np.median(adm - tr.arrival_ns)) / 1e9
        p99 = _tbt_p99(recs)
        dev_s = sum(r["step_ns"] for r in recs) / 1e9
        res = dict(qps=qps, p99_tbt_ms=p99, median_sched_delay_s=delay,
                   decode_tokens_per_s=sum(r["n_decode"] for r in recs) / dev_s,
                   prefill_tokens_per_s=sum(r.get("n_prefill", 0) for r in recs) / dev_s,
                   mean_b=float(np.mean([r["b_t"] for r in recs])), steps=len(recs))
        res["ok"] = bool(p99 <= d_sla + eps_d and delay <= max_delay_s)
        S["eng"].close()
        if S.get("model") is not None:
            S["model"].close()
        S["pool"].close()
        S.clear()
        return res

    for pol, pd in modes:
        for bst in (static_bs if (pol == "static" and static_bs) else [None]):
            per_seed = []
            for seed in seeds:
                a, b = lo, hi
                best, probes = None, []
                while b - a > tol * a:
                    mid = (a * b) ** 0.5
                    r = probe(pol, pd, mid, seed, bst)
                    probes.append(r)
                    print(json.dumps(dict(policy=pol, pd=pd, b_static=bst, seed=seed, **r)), flush=True)
                    if r["ok"]:
                        a, best = mid, r
                    else:
                        b = mid
                per_seed.append(dict(seed=seed, capacity_qps=a if best else None, at_capacity=best, probes=probes))
            caps = [x["capacity_qps"] for x in per_seed if x["capacity_qps"]]
            out["rows"].append(dict(policy=pol, pd_fusion=pd, b_static=(bst or b_static or 256) if pol == "static" else None,
                                    capacity_qps=float(np.mean(caps)) if caps else None,
                                    capacity_min=min(caps) if caps else None, capacity_max=max(caps) if caps else None,
                                    tol=tol, per_seed=per_seed))
            print(json.dumps({k: v for k, v in out["rows"][-1].items() if k != "per_seed"}), flush=True)
    return out


def pd_table(cfg="llama2-7b", bs=(64, 128, 256), full_model=False, pd_token_budget=0):
    """PD-fusion whole-trace runs (Table I shape, all-at-once arrivals): static b vs the
    memory-aware rule deciding the fused iteration's token budget (R25).  full_model: prompts
    are prefilled through the weights (QKV/O/MLP GEMMs + K7) instead of the KV fill."""
    import gc

    import torch
    rows = []
    for pol, b in [("static", x) for x in bs] + [("memory", None)]:
        gc.collect()
        torch.cuda.empty_cache()
        S = bench.setup_engine(cfg_name=cfg, policy=pol, b_static=b or 256, time_attention=False, pd_fusion=True,
                               full_model=full_model, pd_token_budget=pd_token_budget)
        eng = S["eng"]
        bufs = eng.buffers(S["qd"], S["od"])
        t0 = time.time()
        recs, ms = bench.run_steps(S, 10 ** 9, bufs, torch.cuda.current_stream())
        dev_s = ms / 1e3
        rows.append(dict(policy=pol, b_static=b, full_model=full_model, steps=len(recs), device_s=dev_s,
                         decode_tokens_per_s=sum(r["n_decode"] for r in recs) / dev_s,
                         prefill_tokens_per_s=sum(r["n_prefill"] for r in recs) / dev_s,
                         mean_b=float(np.mean([r["b_t"] for r in recs])),
                         preemptions=int(sum(r["n_preempted"] for r in recs)), wall_s=time.time() - t0))
        print(json.dumps(rows[-1]), flush=True)
        S["eng"].close()
        if S.get("model") is not None:
            S["model"].close()
        S["pool"].close()
        S.clear()
        del eng, bufs  # the engine holds the pool, the pool holds the KV allocation
    return dict(config=cfg, full_model=full_model, pd_token_budget=pd_token_budget, rows=rows)


def surge_table(cfg="surge-7b-dp", lam0=None, bs=(64, 128, 256), policies=("memory", "combined"),
                d_sla=20.0, eps_d=0.8):
    """BASELINE configs[4] analog on one GPU (one DP rank's share, its own 40 GB KV cap): a
    piecewise-Poisson surge -- lambda0 for 60 s, 2.5 lambda0 for 30 s, lambda0 for 60 s,
    lambda0 sized so the steady state holds ~60 % of the cap (Little: N = 0.6 eta / E[ctx],
    lifetime = l_out steps of tau(N) from the Fig. 3 fit) -- through static b vs the dynamic
    rules.  Reports tokens/s, preemptions, peak KV occupancy, p99 TBT and scheduling delay."""
    import gc

    import torch
    from synth import configs, trace
    c = configs.CONFIGS[cfg]
    t = c["trace"]
    beta = configs.kv_bytes_per_token(c)
    eta = c["cap_bytes_per_gpu"] // beta
    e_ctx = t["mean_in"] + t["mean_out"] / 2
    n_conc = 0.6 * eta / e_ctx
    if lam0 is None:
        tau_ms = 0.63 + 0.0305 * n_conc          # attention-only Fig. 3 fit (7B), profiles/r01_paper_tables.json
        lam0 = n_conc / (t["mean_out"] * tau_ms / 1e3)
    segs = [(0, lam0), (60000, 2.5 * lam0), (90000, lam0)]
    n = int(lam0 * 60 + 2.5 * lam0 * 30 + lam0 * 60)
    tr = trace.make_trace(n, t["mean_in"], t["mean_out"], t["L_max"], t["seed"], dist=t["dist"],
                          arrival="piecewise", segments=segs)
    rows = []
    runs = [("static", b) for b in bs] + [(p, None) for p in policies]
    for pol, b in runs:
        gc.collect()
        torch.cuda.empty_cache()
        S = bench.setup_engine(cfg_name=cfg, policy=pol, b_static=b or 256, time_attention=False,
                               trace_override=tr, sla_ms=d_sla, eps_d_ms=eps_d)
        eng = S["eng"]
        bufs = eng.buffers(S["qd"], S["od"])
        t0 = time.time()
        recs, ms = bench.run_steps(S, 10 ** 9, bufs, torch.cuda.current_stream())
        adm, fin = eng.request_times()
        dev_s = sum(r["step_ns"] for r in recs) / 1e9
        clock_s = (recs[-1]["clock_ns"] + recs[-1]["step_ns"]) / 1e9
        rows.append(dict(policy=pol, b_static=b, steps=len(recs), tokens=int(sum(r["n_decode"] for r in recs)),
                         tokens_per_s_device=sum(r["n_decode"] for r in recs) / dev_s,
                         makespan_s=clock_s, preemptions=int(sum(r["n_preempted"] for r in recs)),
                         peak_pages=int(max(r["used_pages"] for r in recs)), cap_pages=S["cap_pages"],
                         p99_tbt_ms=_tbt_p99(recs), median_sched_delay_s=float(np.median(adm - tr.arrival_ns)) / 1e9,
                         p99_sched_delay_s=float(np.percentile(adm - tr.arrival_ns, 99)) / 1e9,
                         mean_b=float(np.mean([r["b_t"] for r in recs])), wall_s=time.time() - t0))
        print(json.dumps(rows[-1]), flush=True)
        S["eng"].close()
        S["pool"].close()
        S.clear()
        del eng, bufs
    return dict(config=cfg, lambda0_qps=lam0, segments=segs, n_requests=n, d_sla_ms=d_sla, eps_d_ms=eps_d,
                rows=rows)


def swap_table(cfg="llama2-7b", kv_gb=40.0, swap_gb=16.0, n_req=1500, b=256):
    """Whole trace (all-at-once) near the KV cap: recompute vs swap preemption (static b) and
    the memory-aware rule.  In this attention-only engine a recompute is the KV fill of the
    request's T tokens (no weights), i.e. a lower bound of the real re-prefill cost."""
    import gc

    import torch
    rows = []
    for pol, swap in (("static", 0), ("static", swap_gb), ("memory", 0)):
        gc.collect()
        torch.cuda.empty_cache()
        S = bench.setup_engine(cfg_name=cfg, policy=pol, b_static=b, time_attention=False, n_req=n_req,
                               cap_bytes=int(kv_gb * bench.GB), swap_bytes=int(swap * bench.GB))
        eng = S["eng"]
        bufs = eng.buffers(S["qd"], S["od"])
        t0 = time.time()
        recs, ms = bench.run_steps(S, 10 ** 9, bufs, torch.cuda.current_stream())
        dev_s = ms / 1e3
        sw = [r for r in recs if r["n_swap_out"] or r["n_swap_in"]]
        rows.append(dict(policy=pol, b_static=b if pol == "static" else None, preempt="swap" if swap else "recompute",
                         swap_gb=swap, kv_cap_pages=S["cap_pages"], steps=len(recs), device_s=dev_s,
                         tokens_per_s=sum(r["n_decode"] for r in recs) / dev_s,
                         mean_b=float(np.mean([r["n_decode"] for r in recs])),
                         preemptions=int(sum(r["n_preempted"] for r in recs)),
                         swapped_out=int(sum(r["n_swap_out"] for r in recs)),
                         swapped_in=int(sum(r["n_swap_in"] for r in recs)),
                         swap_gb_moved=sum(r["swap_bytes"] for r in recs) / bench.GB,
                         mean_step_ms=float(np.mean([r["step_ns"] for r in recs]) / 1e6),
                         mean_step_ms_with_swap=float(np.mean([r["step_ns"] for r in sw]) / 1e6) if sw else None,
                         wall_s=time.time() - t0))
        print(json.dumps(rows[-1]), flush=True)
        S["eng"].close()
        S["pool"].close()
        S.clear()
        del eng, bufs
    return dict(config=cfg, kv_gb=kv_gb, n_requests=n_req, rows=rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fig3", action="store_true")
    ap.add_argument("--table1", action="store_true")
    ap.add_argument("--sla", action="store_true")
    ap.add_argument("--capacity", action="store_true")
    ap.add_argument("--pd", action="store_true")
    ap.add_argument("--swap", action="store_true")
    ap.add_argument("--surge", action="store_true", help="configs[4]: traffic surge near the KV cap")
    ap.add_argument("--surge-lam0", type=float, default=None, help="base rate (qps); default from Little's law")
    ap.add_argument("--pd-model", action="store_true", help="PD table with prefill through the full model")
    ap.add_argument("--model", action="store_true", help="--fig3/--table1/--sla with the full decode step")
    ap.add_argument("--cap-lo", type=float, default=10.0, help="capacity bisection: lowest rate (qps)")
    ap.add_argument("--cap-hi", type=float, default=640.0, help="capacity bisection: highest rate (qps)")
    ap.add_argument("--cap-margin", type=float, default=0.0,
                    help="Alg. 2 steers to D_SLA - margin while capacity is judged at D_SLA (p99)")
    ap.add_argument("--cap-pd-only", action="store_true", help="capacity: the combined rule with PD fusion only")
    ap.add_argument("--cap-d", type=float, default=None, help="capacity: pin D_SLA (ms) instead of tau(b_mem/2)")
    ap.add_argument("--cap-config", default="llama2-13b-sla", help="capacity / SLA config (e.g. llama2-7b)")
    ap.add_argument("--cap-modes", default=None, help="capacity modes, e.g. static:pd,combined:pd,combined:nopd")
    ap.add_argument("--pd-token-budget", type=int, default=0,
                    help="PD fusion: fixed iteration token budget (R36) instead of b_t (R25)")
    ap.add_argument("--cap-tol", type=float, default=0.05, help="capacity bisection: relative tolerance")
    ap.add_argument("--cap-seeds", default=None, help="capacity: arrival seeds, e.g. 11,12,13 (one bisection each)")
    ap.add_argument("--cap-static-bs", default=None, help="capacity: static baselines to sweep, e.g. 128,192,256")
    ap.add_argument("--out", default="gpurun_out/paper_tables.json")
    a = ap.parse_args()
    global FULL_MODEL
    FULL_MODEL = a.model
    import torch
    torch.cuda.set_device(0)
    res = {}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)

    def save():  # after every section, so a time-out keeps what finished
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)

    if a.fig3:
        res["fig3"] = fig3()
        print(json.dumps(res["fig3"]["fit"]), flush=True)
        save()
    if a.table1:
        res["table1"] = table1()
        save()
    if a.pd:
        res["pd_table"] = pd_table()
        save()
    if a.pd_model:
        res["pd_table_model"] = pd_table(full_model=True, pd_token_budget=a.pd_token_budget)
        save()
    if a.swap:
        res["swap"] = swap_table()
        save()
    if a.surge:
        res["surge"] = surge_table(lam0=a.surge_lam0)
        save()
    if a.sla or a.capacity:
        res["fig3_13b"] = fig3(a.cap_config, bs=(32, 64, 128, 256))
        save()
        # binding SLA: the step latency at half the largest static batch; eps_D = 4 % of D
        b_mem = max(r["mean_batch"] for r in res["fig3_13b"]["rows"])
        d = round(res["fig3_13b"]["fit"]["a0_ms"] + res["fig3_13b"]["fit"]["a1_ms"] * b_mem / 2, 3)
        if a.sla:
            res["sla"] = sla(fit=d)
            save()
        if a.capacity:
            modes = (("combined", True),) if a.cap_pd_only else \
                (("static", False), ("combined", False), ("static", True), ("combined", True))
            if a.cap_modes:
                modes = tuple((m.split(":")[0], m.split(":")[1] == "pd") for m in a.cap_modes.split(","))
            if a.cap_d:
                d = a.cap_d
            res["capacity"] = capacity(cfg=a.cap_config, d_sla=d, eps_d=round(0.04 * d, 3), b_static=int(b_mem), lo=a.cap_lo,
                                       hi=a.cap_hi, ctrl_margin_ms=a.cap_margin, modes=modes,
                                       pd_token_budget=a.pd_token_budget, tol=a.cap_tol,
                                       seeds=tuple(int(x) for x in a.cap_seeds.split(",")) if a.cap_seeds else (None,),
                                       static_bs=[int(x) for x in a.cap_static_bs.split(",")] if a.cap_static_bs else None)
            save()
    print(json.dumps({k: (v.get("fit") if isinstance(v, dict) else None) for k, v in res.items()}))


if __name__ == "__main__":
    main()
