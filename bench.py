#!/usr/bin/env python
"""Benchmark: continuous-batching decode iterations of the Llama-2-7B-shaped workload
(BASELINE.json configs[1]) through the C-ABI engine on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

A step = one engine iteration = admission + prefill fill + page growth + KV append +
paged decode attention over all L layers (batch statistics fused into layer 0) +
statistics D2H + the host batch-size decision (Algorithm 1).  Prints one JSON line.
N > 1 (torchrun): request-sharded DP, per-GPU work fixed (weak scaling), the 128-byte
statistics records all-gathered over NCCL every step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import configs, trace  # noqa: E402

CFG_NAME = "llama2-7b"
METRIC = "decode tokens/s"
UNIT = "tokens/s"
GB = 1e9


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config, tp, kernel, model=False):
    """The committed ncu capture (profiles/ncu_traffic.json, written by profiles/run_ncu_traffic.sh
    on the current build) of THIS configuration's decode kernel: dram read + write bytes per
    launch and the algorithmic bytes of the same launches, or None if it has no entry."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    for e in d.get("entries", []):
        if e["config"] == config and e["tp"] == tp and e["kernel"] == kernel and bool(e.get("model")) == bool(model):
            return e
    return None


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (B200_PROFILING.md's clocks
    line): NVML polled every 5 ms from a thread (a 3 ms-step run still gets dozens of samples),
    else nvidia-smi every 100 ms."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80}

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []
        self.samples = []   # (sm_mhz, max_mhz, reasons bitmask) from NVML
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:  # the CUDA device's own NVML handle (CUDA_VISIBLE_DEVICES may renumber devices)
                import torch
                pr = torch.cuda.get_device_properties(self.device)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.nvml = (pynvml, h)

            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                while not self.stop.is_set():
                    try:
                        self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx,
                                             reasons_fn(h)))
                    except pynvml.NVMLError:
                        pass
                    self.stop.wait(0.005)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        if self.nvml:
            for clk, m, bits in self.samples:
                sm.append(float(clk))
                mx = float(m)
                reasons |= {nm for nm, b in self.BITS.items() if bits & b}
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml 5 ms"}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 100 ms"}


def make_workload(cfg_name=CFG_NAME, world=1, n_req=None):
    """The config's trace; DP runs generate world x n_requests (weak scaling), shard i % world."""
    c = configs.CONFIGS[cfg_name]
    t = c["trace"]
    n = (n_req or c["n_requests"]) * world
    tr = trace.make_trace(n, t["mean_in"], t["mean_out"], t["L_max"], t["seed"], dist=t["dist"])
    return c, tr


POLICIES = {"static": 0, "memory": 1, "sla": 2, "combined": 3}


def sched_kwargs(c, beta, policy=None, b_static=256, sla_ms=None, eps_d_ms=None, dp_world=1):
    """The scheduler's configuration.  B_max is the config's per-GPU batch bound (the pool's request
    slots): a job of dp_world request shards decides a GLOBAL b_t (Alg. 1 over the summed records
    and the global eta, R21), so its bound is dp_world x B_max and each rank's share stays at the
    one-GPU batch -- per-GPU work fixed (weak scaling).  A global 512 over 8 shards would leave 64
    requests per GPU."""
    pr = configs.prior_record(c)
    pol = POLICIES[policy or c["policy"]]
    return dict(policy=pol, b_static=b_static, b_min=c["b_min"], b_max=c["b_max"] * dp_world, b0=c["b_min"],
                eps_m=c["eps_m"], bytes_per_token=beta, page_size=c["page_size"], refresh_steps=100,
                w_len=256, w_sla=20, alpha=c.get("alpha", 8), delta=c.get("delta", 2),
                d_sla_ms=sla_ms or c.get("sla_ms", 50.0),
                eps_d_ms=eps_d_ms if eps_d_ms is not None else c.get("eps_d_ms", 2.0),
                prior=tuple(pr.values()))


def setup_engine(device=0, rank=0, world=1, cfg_name=CFG_NAME, cap_bytes=None, time_attention=True,
                 out_dtype=0, seed=2024, n_req=None, policy=None, b_static=256, sla_ms=None, tp=1,
                 trace_override=None, eps_d_ms=None, pd_fusion=False, swap_bytes=0, full_model=False,
                 free_bytes=None, pd_token_budget=0, tp_rank=0, per_layer_launches=False):
    """Pool sized from free HBM (cap = free - modeled fp16 weights of this GPU - reserve), or the
    config's fixed per-GPU cap; DP request shards (world) or KV-head TP (tp)."""
    import torch

    import paper_2503_05248_b200 as dbk
    c, tr = make_workload(cfg_name, world if tp == 1 else 1, n_req)
    if trace_override is not None:
        tr = trace_override
    L, Hq, Hkv, d, P = c["layers"], c["q_heads"] // tp, c["kv_heads"] // tp, c["head_dim"], c["page_size"]
    beta = configs.kv_bytes_per_token(c, tp=tp)
    max_req = c["b_max"] + 8
    io_bytes = 2 * L * max_req * Hq * d * 4 + 2 * max_req * L * Hkv * d * 2
    # free HBM: this GPU's, or the minimum over the ranks (every rank then derives the same cap,
    # eta and therefore the same b_t decisions)
    free = free_bytes if free_bytes is not None else torch.cuda.mem_get_info(device)[0]
    if cap_bytes is None and os.environ.get("DBK_BENCH_KV_GB"):  # profiling runs only (smaller pool)
        cap_bytes = int(float(os.environ["DBK_BENCH_KV_GB"]) * GB)
    if cap_bytes is None and "cap_bytes_per_gpu" in c:
        cap_bytes = c["cap_bytes_per_gpu"]
    if cap_bytes is None:
        cap_bytes = free - c["weights_bytes"] // tp - c["reserve_bytes"] - io_bytes
    cap_pages = int(cap_bytes // (P * beta))
    maxp = -(-c["trace"]["L_max"] // P)
    # KV-head TP: rank tp_rank holds global kv heads [tp_rank*Hkv, (tp_rank+1)*Hkv) (and their q heads);
    # the generator keys K/V/q by the global head, so the shards are disjoint slices of the TP1 job
    pool = dbk.KVPool(L, Hq, Hkv, d, cap_pages, max_req, maxp, "f16", device=device,
                      kv_head_offset=tp_rank * Hkv if tp > 1 else 0)
    if swap_bytes:  # swap preemption (R29-R31): pinned host swap space
        pool.swap_space_attach(torch.empty(int(swap_bytes), dtype=torch.uint8, pin_memory=True))
    # M_max of the whole job: DP shards add their pools; TP ranks hold the same tokens
    mem_cap_total = cap_pages * P * beta * (world if tp == 1 else 1)
    sched = dbk.Scheduler(**sched_kwargs(c, beta, policy, b_static, sla_ms, eps_d_ms,
                                         dp_world=world if tp == 1 else 1))
    eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, mem_cap_total, seed=seed,
                     out_dtype=out_dtype, time_attention=time_attention,
                     rank=rank if tp == 1 else 0, world=world if tp == 1 else 1, sla_ms=sla_ms or 0.0,
                     pd_fusion=pd_fusion, preempt_mode=1 if swap_bytes else 0, pd_token_budget=pd_token_budget,
                     per_layer_launches=per_layer_launches)
    model = None
    if full_model:  # NEXT row 3: QKV/O/MLP/LM-head GEMMs with synthetic fp16 weights around the attention
        if "model" not in c:
            raise SystemExit(f"--model: no model dimensions for config {cfg_name}")
        m = c["model"]
        model = dbk.Model(pool, m["hidden"], m["ffn"], m["vocab"], max_pos=c["trace"]["L_max"] + 16,
                          weight_seed=seed + 1)
        eng.attach_model(model)
    et = torch.float32 if out_dtype == 2 else torch.float16
    qd = torch.empty(L, max_req, Hq, d, dtype=torch.float16, device=f"cuda:{device}")
    od = torch.empty(L, max_req, Hq, d, dtype=et, device=f"cuda:{device}")
    kvd = torch.empty(2, L, max_req, Hkv, d, dtype=torch.float16, device=f"cuda:{device}")
    return dict(dbk=dbk, c=c, tr=tr, pool=pool, sched=sched, eng=eng, qd=qd, od=od, kvd=kvd, tp=tp, model=model,
                policy=policy, b_static=b_static, sla_ms=sla_ms, eps_d_ms=eps_d_ms,
                cap_pages=cap_pages, beta=beta, max_req=max_req, mem_cap_total=mem_cap_total, seed=seed,
                L=L, Hq=Hq, Hkv=Hkv, d=d, tp_rank=tp_rank)


def e2e_buffers(S, eng, args):
    """The engine's end-to-end buffers: attention-only -- pinned host q and new K/V rows in, every
    layer's output back; full model -- each step's input token ids in, greedy samples out."""
    import torch
    if not args.model:
        L, Hq, Hkv, d, mr = S["L"], S["Hq"], S["Hkv"], S["d"], S["max_req"]
        hq = torch.empty(L * mr * Hq * d, dtype=torch.float16, pin_memory=True).uniform_(-1, 1)
        hk = torch.empty(mr * L * Hkv * d, dtype=torch.float16, pin_memory=True).uniform_(-1, 1)
        hv = torch.empty(mr * L * Hkv * d, dtype=torch.float16, pin_memory=True).uniform_(-1, 1)
        ho = torch.empty(L * mr * Hq * d, dtype=torch.float16, pin_memory=True)
        S["_e2e_host"] = (hq, hk, hv, ho)  # keep the pinned buffers alive
        return eng.buffers(S["qd"], S["od"], S["kvd"], hq, hk, hv, ho)
    host_tok = torch.zeros(len(S["tr"]), dtype=torch.int32).pin_memory()
    S["_e2e_host"] = (host_tok,)
    return eng.buffers(S["qd"], S["od"], host_tokens=host_tok)


def run_steps(S, k, bufs, stream, comm_world=1, dist=None):
    """k engine steps; returns (records, device ms) timed with CUDA events on `stream`."""
    import torch
    eng = S["eng"]
    recs = []
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        if eng.done():
            break
        if S.get("exchange") is not None:  # caller-side exchange of the 128-B records
            local = eng.step_launch(bufs, stream)
            recs.append(eng.step_finish(S["exchange"](local)))
        else:
            recs.append(eng.step(bufs, stream))
    e1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    return recs, e0.elapsed_time(e1)


def oracle_sched_replay(S, recs):
    """The oracle's scheduler replay (O7: allocator + Alg. 1 / Alg. 2, Python) of the first
    steps of this very run from their logged step times: host time per step at full scale
    (SURVEY.md §8(d)), and whether every decision agreed bit for bit."""
    from oracle import engine as oeng
    from oracle import policy as opol
    if not recs or S.get("tp", 1) != 1:
        return {}
    c, tr, P = S["c"], S["tr"], S["c"]["page_size"]
    kw = sched_kwargs(c, S["beta"], S.get("policy"), S.get("b_static", 256), S.get("sla_ms"), S.get("eps_d_ms"))
    rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, S["cap_pages"], P)],
                     opol.SchedConfig(**kw), S["mem_cap_total"])
    agree = True
    t0 = time.perf_counter()
    for g in recs:
        o = rp.step(g["step_ns"])
        agree &= all(g[k] == o[k] for k in ("b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "sum_ctx",
                                            "used_pages"))
    dt = time.perf_counter() - t0
    return {"sched_replay_ms_per_step": round(dt / len(recs) * 1e3, 3), "sched_replay_steps": len(recs),
            "sched_replay_bit_exact": bool(agree)}


def cpu_model():
    """The host CPU's model name (/proc/cpuinfo), for the cpu_baseline record."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def toy_step_oracle(budget_s=3.0):
    """SURVEY.md §8(d) input (i): the oracle's whole toy decode step (BASELINE configs[0]: 8
    requests, 1 layer, 8 heads x d64, 256-page cap, memory rule) -- the replay's S1-S7 (admission,
    page growth, statistics, Alg. 1) plus fp64 paged attention of the step's batch on one thread,
    repeated over the toy trace until ~budget_s.  Inputs are built outside the timed calls."""
    from oracle import attention as oatt
    from oracle import engine as oeng
    from oracle import policy as opol
    c, tr = make_workload("toy")
    L, Hq, Hkv, d, P = c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["page_size"]
    cap = c["cap_tokens"] // P
    beta = configs.kv_bytes_per_token(c)
    kw = sched_kwargs(c, beta)
    secs, steps, toks = 0.0, 0, 0
    while secs < budget_s:
        rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, cap, P)],
                         opol.SchedConfig(**kw), cap * P * beta)
        while not rp.done() and secs < budget_s:
            t0 = time.perf_counter()
            rec = rp.step(1_000_000)
            dt = time.perf_counter() - t0
            rs, ctx, li, lo, pages = rec["batches"][0]
            if rs:
                bt, pk, pv, qq = oatt.synth_paged_batch(1, rs, ctx, pages, 0, Hq, Hkv, d, P, "f16")
                t0 = time.perf_counter()
                oatt.paged_decode_attention(np.asarray(ctx), bt, pk, pv, qq, "f16", nthreads=1)
                dt += time.perf_counter() - t0
            secs += dt
            steps += 1
            toks += len(rs)
    return {"toy_step_ms": round(1e3 * secs / max(steps, 1), 4), "toy_steps": steps,
            "toy_tokens_per_s": round(toks / secs, 1) if secs > 0 else None}


def cpu_baseline(S, budget_s=15.0, threads=None, single_budget_s=5.0):
    """The oracle (plain C, fp64) on a bounded sample of the current decode batch: all host
    cores, and one thread (SURVEY.md §8(d) "1 thread and nproc threads")."""
    from oracle import attention as oatt
    c = S["c"]
    L, Hq, Hkv, d, P = c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["page_size"]
    ids, ctx = S["eng"].last_batch()
    threads = threads or os.cpu_count() or 1
    # one fixed sample: k random requests of the timed batch at layer 0 (inputs regenerated
    # on the host from logical coordinates), timed repeatedly until ~budget_s of oracle work
    rng = np.random.default_rng(0)
    k = min(len(ids), 64)
    sel = rng.choice(len(ids), size=k, replace=False)
    pages, nxt = [], 0
    for cx in ctx[sel]:
        np_ = -(-int(cx) // P)
        pages.append(list(range(nxt, nxt + np_)))
        nxt += np_
    bt, pk, pv, qq = oatt.synth_paged_batch(S["seed"], [int(x) for x in ids[sel]], ctx[sel], pages, 0,
                                            Hq, Hkv, d, P, "f16")

    def timed(nth, budget):
        secs, reps = 0.0, 0
        while secs < budget:
            t0 = time.perf_counter()
            oatt.paged_decode_attention(ctx[sel], bt, pk, pv, qq, "f16", nthreads=nth)
            secs += time.perf_counter() - t0
            reps += 1
        return secs, reps
    secs, reps = timed(threads, budget_s)
    s1, r1 = timed(1, single_budget_s)
    kv_bytes = float(np.sum(ctx[sel])) * 2 * Hkv * d * 2   # the KV the sample reads, per repetition
    tok_s = k * reps / L / secs
    return {"value": round(tok_s, 3), "unit": UNIT, "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(),
            "single_thread_value": round(k * r1 / L / s1, 3),
            "kv_gbs_processed": round(kv_bytes * reps / secs / 1e9, 3),
            "sample": f"{k} random requests of the timed batch (mean ctx {float(np.mean(ctx[sel])):.0f}) x "
                      f"1 layer, fp64 paged attention, {reps} repetitions in {secs:.1f} s on {threads} threads "
                      f"({r1} in {s1:.1f} s on 1 thread); tokens/s = request-layers / L / time"}


def run_gpu(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # test harness only (tests/test_gpu_bench_multirank.py): every rank on cuda:0 with a gloo
    # process group, so the N > 1 bookkeeping of this script runs on a one-GPU box
    gloo_test = os.environ.get("DBK_BENCH_TEST_GLOO") == "1"
    if gloo_test:
        local = 0
    red = "cpu" if gloo_test else "cuda"  # device of the timing / token all-reduces
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if gloo_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # configs[3] (70B GQA) is sharded by KV heads (TP); the others by requests (DP)
    tp = world if args.config == "llama3-70b-gqa" else 1
    if args.tp_shard:  # one GPU runs exactly rank 0's share of a KV-head TP run of that width
        if world != 1 or args.config != "llama3-70b-gqa":
            raise SystemExit("--tp-shard: single-GPU emulation of the 70B KV-head TP shard only")
        tp = args.tp_shard
        if not 0 <= args.tp_rank < tp:
            raise SystemExit("--tp-rank must be in [0, tp-shard)")
    free_bytes = None
    if dist is not None:  # the same pool size on every rank (MIN of the ranks' free HBM)
        f_t = torch.tensor([float(torch.cuda.mem_get_info(local)[0])], dtype=torch.float64, device=red)
        dist.all_reduce(f_t, op=dist.ReduceOp.MIN)
        free_bytes = int(f_t.item())
    S = setup_engine(device=local, rank=rank, world=world, cfg_name=args.config, policy=args.policy,
                     b_static=args.b_static, sla_ms=args.sla_ms, tp=tp, full_model=args.model,
                     free_bytes=free_bytes, tp_rank=(args.tp_rank if args.tp_shard else rank) if tp > 1 else 0,
                     per_layer_launches=args.per_layer_launches)
    dbk = S["dbk"]
    eng = S["eng"]
    exchange_kind, comm = None, None
    if world > 1:
        mode = dbk._lib.MODE_TP if tp > 1 else dbk._lib.MODE_DP
        if gloo_test and args.exchange == "nccl":  # test harness only: NCCL refuses ranks sharing one GPU
            fields = dbk._lib.STATS_FIELDS

            def exchange(local_rec):
                t = torch.tensor([local_rec[f] for f in fields], dtype=torch.int64, device=red)
                out = [torch.zeros_like(t) for _ in range(world)]
                dist.all_gather(out, t)
                return dbk.stats_reduce([dict(zip(fields, o.tolist())) for o in out], mode)
            S["exchange"] = exchange
            exchange_kind = {"kind": "torch.distributed gloo all-gather (DBK_BENCH_TEST_GLOO test harness; "
                                     "--exchange nccl cannot run with ranks sharing one GPU)"}
        else:  # the product path: libdbk's own exchange (mailbox over peer memory, or NCCL)
            mb_err = None
            if args.exchange == "mailbox":
                try:
                    comm = dbk.Mailbox(dist, world, rank, local)
                    eng.attach_mbox(comm, mode)
                    exchange_kind = {"kind": "libdbk mailbox: one exchange kernel per step stores the 128-B "
                                             "record into every peer's IPC-mapped mailbox (dbk_engine_attach_mbox)",
                                     "ranks": world}
                    print(f"[bench] rank {rank}: libdbk mailbox exchange over {world} ranks "
                          f"mode={'TP' if tp > 1 else 'DP'}", file=sys.stderr, flush=True)
                except Exception as ex:  # loud, and recorded in the line: the NCCL transport instead
                    mb_err = f"{type(ex).__name__}: {ex}"
                    print(f"[bench] rank {rank}: MAILBOX SETUP FAILED ({mb_err}); using libdbk NCCL",
                          file=sys.stderr, flush=True)
                    comm = None
                # every rank must use the same transport: if the mailbox failed anywhere, all switch
                ok_t = torch.tensor([0 if comm is None else 1], dtype=torch.int32, device=red)
                dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
                if comm is not None and int(ok_t.item()) == 0:
                    eng.attach_mbox(None, mode)
                    comm.close()
                    comm = None
                    mb_err = mb_err or "a peer rank's mailbox setup failed"
            if comm is None:
                comm = dbk.Comm(dist, world, rank, local)
                nr, rk = comm.info()
                print(f"[bench] rank {rank}: libdbk NCCL communicator nranks={nr} rank={rk} "
                      f"mode={'TP' if tp > 1 else 'DP'}", file=sys.stderr, flush=True)
                if (nr, rk) != (world, rank):
                    raise SystemExit(f"NCCL communicator reports nranks={nr} rank={rk}, expected {world}/{rank}")
                eng.attach_comm(comm, mode)
                exchange_kind = {"kind": "libdbk ncclAllGather of the 128-B records (dbk_stats_allgather)",
                                 "nccl_nranks": nr}
                if mb_err:
                    exchange_kind["mailbox_setup_failed"] = mb_err
    stream = torch.cuda.current_stream()
    bufs = eng.buffers(S["qd"], S["od"])
    # fast-forward to the steady state (untimed), then W warm-up steps (untimed)
    ff_recs, _ = run_steps(S, args.ff, bufs, stream, dist=dist)
    # end-to-end through the same API (host buffers, copies inside the timed region): its steps
    # are split around the device-resident timed region -- half before the warm-up, half after --
    # so both measure the same stretch of the trace (contexts grow every step; an e2e run placed
    # entirely after the timed region would see ~5 % more KV per step)
    e2e_parts = []
    if not args.no_e2e and not args.ncu_step:
        ebufs = e2e_buffers(S, eng, args)
        run_steps(S, 2, ebufs, stream, dist=dist)
        e2e_parts.append(run_steps(S, args.steps // 2, ebufs, stream, dist=dist))
    run_steps(S, args.warmup, bufs, stream, dist=dist)
    eng.attn_timing(reset=True)
    if args.ncu_step:  # profiling: ONE step inside an NVTX range (ncu --nvtx --nvtx-include dbk_step/)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("dbk_step")
        rec = eng.step(bufs, stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        a_ms, a_launches, a_bytes = eng.attn_timing(reset=True)
        info = S["pool"].info()
        if rank == 0:
            print(json.dumps({"ncu_step": {"config": args.config, "tp": tp, "model": bool(args.model),
                                           "kernel": "decode_gqa_kernel" if info["decode_path"] == 2 else "decode_kernel",
                                           "attn_bytes": a_bytes, "attn_kernels": a_launches,
                                           "n_decode": rec["n_decode"], "chunk_pages": info["chunk_pages"],
                                           "per_layer_launches": bool(args.per_layer_launches or args.model)}}),
                  flush=True)
        return
    with ClockSampler(local) as clk:
        recs, ms = run_steps(S, args.steps, bufs, stream, dist=dist)
    att_ms, att_launches, att_bytes = eng.attn_timing(reset=True)
    info = S["pool"].info()
    xch = eng.last_exchange(reset=True) if comm is not None else None
    # every rank's own timed-region device time (ms), gathered for the line (max is `value`'s clock)
    per_rank_ms = [ms]
    if dist is not None:
        g = [torch.zeros(1, device=red) for _ in range(world)]
        dist.all_gather(g, torch.tensor([ms], device=red))
        per_rank_ms = [float(x.item()) for x in g]
    # decode tokens of the whole job: every rank's step record carries the GLOBAL counts (the
    # exchanged, reduced record: DP sums the disjoint shards, TP ranks serve the same requests),
    # so each rank contributes 1/world of it to the all-reduce
    ms_t = torch.tensor([ms], device=red)
    tok_t = torch.tensor([float(sum(r["n_decode"] for r in recs)) / world], device=red)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tok_t)
    ms_max, toks = float(ms_t.item()), float(tok_t.item())
    L, Hq, Hkv, d = S["L"], S["Hq"], S["Hkv"], S["d"]
    erecs, ems_t, etok_t = [], None, None
    if e2e_parts:
        e2e_parts.append(run_steps(S, args.steps - args.steps // 2, ebufs, stream, dist=dist))
        erecs = [r for part in e2e_parts for r in part[0]]
        ems_t = torch.tensor([sum(part[1] for part in e2e_parts)], device=red)
        etok_t = torch.tensor([float(sum(r["n_decode"] for r in erecs)) / world], device=red)
        if dist is not None:
            dist.all_reduce(ems_t, op=dist.ReduceOp.MAX)
            dist.all_reduce(etok_t)
    # read-only streaming probe over (part of) the KV pool on this GPU: the achievable
    # read bandwidth beside which the attention kernel's is reported
    import ctypes
    probe_ms = ctypes.c_double()
    probe_bytes = min(S["pool"].kv.numel(), 32 * 10 ** 9) // 16 * 16
    dbk._lib.dbk_probe_read_bandwidth(S["pool"].kv.data_ptr(), probe_bytes, local, stream.cuda_stream,
                                      ctypes.byref(probe_ms))
    probe_gbs = probe_bytes / 1e9 / (probe_ms.value / 1e3)
    if rank == 0:
        peak, peak_src = measured_peaks()
        achieved = att_bytes / 1e9 / (att_ms / 1e3) if att_ms > 0 else 0.0
        kern = "decode_gqa_kernel" if info["decode_path"] == 2 else "decode_kernel"
        traffic_rec = ncu_traffic(args.config, tp, kern, args.model)
        c = S["c"]
        n_steps = len(recs)
        # the decode tokens these steps could emit if every step only streamed its KV at `peak`
        kv_s = sum(r["sum_ctx"] for r in recs) * S["beta"] / (world if tp == 1 else 1) / (peak * 1e9)
        tok_roof = (toks / kv_s) if kv_s > 0 else 0.0
        kname = "decode_gqa_kernel (K2, tensor cores)" if info["decode_path"] == 2 else \
            "decode_kernel (K1, paged decode attention)"
        line = {
            "metric": METRIC, "value": round(toks / (ms_max / 1e3), 2), "unit": UNIT, "n_gpus": world,
            "steps": n_steps, "warmup": args.warmup, "ms_per_step": round(ms_max / max(n_steps, 1), 4),
            "higher_is_better": True, "scaling": "strong" if tp > 1 else "weak", "vs_baseline": None,
            "dtype": "f16",
            "data": ("synthetic (seeded lognormal trace; hash-generated fp16 weights and token ids; prompt KV "
                     "filled by the generator)") if args.model else
                    "synthetic (seeded lognormal trace, hash-generated q/K/V; no weights on this path)",
            "config": {"workload": c["name"], "layers": L, "q_heads": Hq, "kv_heads": Hkv, "head_dim": d,
                       "page_size": 16, "kv_dtype": "fp16", "out_dtype": "fp16",
                       "policy": args.policy or c["policy"], "sla_ms": args.sla_ms or c.get("sla_ms"),
                       "requests": len(S["tr"]),
                       "trace": f"all-at-once, lognormal CV=1, means {c['trace']['mean_in']}/{c['trace']['mean_out']}",
                       "cap_pages_per_gpu": S["cap_pages"],
                       "kv_cap_gb_per_gpu": round(S["cap_pages"] * 16 * S["beta"] / GB, 2),
                       "mean_batch": round(float(np.mean([r["n_decode"] for r in recs])), 1) if recs else 0,
                       "mean_ctx": round(float(np.mean([r["sum_ctx"] / max(r["n_decode"], 1) for r in recs])), 1) if recs else 0,
                       "fast_forward_steps": args.ff,
                       "parallelism": (f"rank {args.tp_rank} of tp{tp} (KV-head shard on one GPU; no exchange)"
                                       if args.tp_shard else
                                       f"tp{world} (KV-head shards)" if tp > 1 else f"dp{world} (request shards)"),
                       "decode_launches": ("one PDL-chained launch per layer" if args.per_layer_launches or args.model
                                           else "multi-layer persistent launches (dbk_decode_step_layers)"),
                       "decode_launches_per_step": (round(sum(r["launches"] for r in recs) / max(len(recs), 1), 2)),
                       "stats_exchange": (dict(exchange_kind or {}, **({
                           "host_us_per_step": (round(xch["us_total"] / max(xch["count"], 1), 2)
                                                if "nccl_nranks" in (exchange_kind or {}) else
                                                "inside the step's device time (exchange kernel)"),
                           "exchanges": xch["count"],
                           "last_step_ns_per_rank": [r["step_ns"] for r in xch["records"]]} if xch else {}))
                           if world > 1 else None),
                       "per_rank_ms": [round(x, 3) for x in per_rank_ms],
                       "l2": "inputs > L2 (~1e2 GB of KV read per step vs 126 MB L2)"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": traffic_rec["dram_bytes_per_launch"] if traffic_rec else None,
                         "traffic_source": ({k: traffic_rec[k] for k in ("file", "build", "launches",
                                                                          "algorithmic_bytes_per_launch",
                                                                          "traffic_over_algorithmic")}
                                            if traffic_rec else "no ncu entry for this configuration"),
                         "kernel": kname,
                         "bytes_per_launch": int(att_bytes / max(att_launches, 1)),
                         "ms_per_launch": round(att_ms / max(att_launches, 1), 4), "peak_source": peak_src,
                         "share_of_step": round(att_ms / max(ms, 1e-9), 4), "ctas_per_sm": info["ctas_per_sm"],
                         "chunk_pages": info["chunk_pages"], "read_probe_gbs": round(probe_gbs, 1),
                         "frac_of_read_probe": round(achieved / probe_gbs, 4),
                         # tokens/s roofline = BW * n / (sum_i ctx_i * beta) per step
                         "tokens_per_s_at_peak": round(tok_roof, 1),
                         "tokens_frac_of_roofline": round(toks / (ms_max / 1e3) / tok_roof, 4) if tok_roof else None},
            "e2e": {"value": round(float(etok_t.item()) / (float(ems_t.item()) / 1e3), 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(np.mean([r["h2d_bytes"] for r in erecs])) if erecs else 0,
                    "d2h_bytes_per_step": int(np.mean([r["d2h_bytes"] for r in erecs])) if erecs else 0,
                    "steps": len(erecs), "placement": "half the steps just before the warm-up, half just after the timed region"}
            if ems_t is not None else None,
            "gpu_launches": int(sum(r["launches"] for r in recs)),
            "clocks": clk.summary(),
            # time between tokens of the timed steps: every running request gets one token per
            # step, so a step's device-timed latency is its TBT (SURVEY §5 metrics)
            "tbt_ms": {q: round(float(np.percentile([r["step_ns"] / 1e6 for r in recs], p)), 3)
                       for q, p in (("p50", 50), ("p95", 95), ("p99", 99))} if recs else None,
        }
        if args.model:
            mc = c["model"]
            line["config"]["full_model"] = {"hidden": mc["hidden"], "ffn": mc["ffn"], "vocab": mc["vocab"],
                                            "weights_gb": round(S["model"].weights.numel() / GB, 2),
                                            "gemms": "dbk tcgen05 GEMM (gemm_tc.cu), fp16 x fp16 -> fp32 accumulate, fused RoPE/KV, SiLU, residual epilogues"}
            line["config"]["workload"] += " + full decode step (weights)"
            line["attention_share_of_step"] = line["roofline"]["share_of_step"]
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(S)
            line["cpu_baseline"].update(oracle_sched_replay(S, ff_recs[:60]))
            line["cpu_baseline"].update(toy_step_oracle())
        print(json.dumps(line), flush=True)
    if args.step_log:  # one JSON record per engine step of this rank, tagged by phase
        path = args.step_log if world == 1 else f"{args.step_log}.rank{rank}"
        with open(path, "w") as fh:
            for phase, rr in (("fast_forward", ff_recs), ("timed", recs), ("e2e", erecs)):
                for r in rr:
                    fh.write(json.dumps(dict(r, phase=phase, rank=rank)) + "\n")
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    """The oracle as the reference arm (no GPU): each step = fp64 paged attention on a bounded
    sample of one layer of the steady-state batch + the oracle's batch-size decision."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import attention as oatt
    from oracle import engine as oeng
    from oracle import policy as opol
    c, tr = make_workload(args.config)
    L, Hq, Hkv, d, P = c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["page_size"]
    beta = configs.kv_bytes_per_token(c)
    free = 178_000_000_000  # same sizing rule as the GPU arm on a 180 GB part
    cap_bytes = c.get("cap_bytes_per_gpu") or (free - c["weights_bytes"] - c["reserve_bytes"])
    cap_pages = int(cap_bytes // (P * beta))
    kw = sched_kwargs(c, beta, args.policy, args.b_static, args.sla_ms)
    kw["policy"] = min(kw["policy"], 1) if kw["policy"] != 3 else 1   # no device timing: memory rule
    rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, cap_pages, P)],
                     opol.SchedConfig(**kw), cap_pages * P * beta)
    for _ in range(args.ff):           # steady state: same fast-forward as the GPU arm (modeled 25 ms steps)
        rp.step(25_000_000)
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(1)
    per_step = 8
    times, toks = [], 0
    for s in range(args.warmup + args.steps):
        rec = rp.step(25_000_000)
        rs, ctx, li, lo, pages = rec["batches"][0]
        sel = rng.choice(len(rs), size=min(per_step, len(rs)), replace=False)
        cp, nxt = [], 0
        for i in sel:
            m = -(-ctx[i] // P)
            cp.append(list(range(nxt, nxt + m)))
            nxt += m
        bt, pk, pv, qq = oatt.synth_paged_batch(2024, [rs[i] for i in sel], [ctx[i] for i in sel], cp,
                                                s % L, Hq, Hkv, d, P, "f16")
        t0 = time.perf_counter()
        oatt.paged_decode_attention(np.asarray([ctx[i] for i in sel]), bt, pk, pv, qq, "f16", nthreads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            toks += len(sel)
    secs = sum(times)
    value = toks / L / secs
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * secs / max(len(times), 1), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (same trace and generator as the GPU arm)",
            "config": {"workload": c["name"], "layers": L, "q_heads": Hq, "kv_heads": Hkv, "head_dim": d},
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"per step {per_step} random requests of the steady-state batch at one "
                                       f"layer (fp64 C oracle); tokens/s = request-layers / L / time"},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ff", type=int, default=300, help="untimed fast-forward steps to the steady state")
    ap.add_argument("--impl", default="dbk", choices=["dbk", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default=CFG_NAME, choices=["llama2-7b", "llama2-13b-sla", "llama3-70b-gqa"])
    ap.add_argument("--policy", default=None, choices=[None, "static", "memory", "sla", "combined"])
    ap.add_argument("--b-static", type=int, default=256)
    ap.add_argument("--sla-ms", type=float, default=None)
    ap.add_argument("--tp-shard", type=int, default=0, choices=[0, 2, 4, 8],
                    help="70B GQA: run rank 0's KV-head shard of a TP-G job on this one GPU (per-GPU kernel rate)")
    ap.add_argument("--tp-rank", type=int, default=0, help="with --tp-shard: which rank's KV-head shard")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end (host buffers) run (profiling)")
    ap.add_argument("--step-log", default=None,
                    help="write every engine step's record (t, b_t, n_decode, sum_ctx, pages, step_ns, "
                         "admissions, preemptions, ...) as JSON lines here (per rank: PATH.rankR)")
    ap.add_argument("--exchange", default="mailbox", choices=["mailbox", "nccl"],
                    help="N > 1: the statistics exchange -- libdbk's mailbox over peer memory (default) or NCCL")
    ap.add_argument("--ncu-step", action="store_true",
                    help="profiling: after fast-forward + warm-up run ONE step inside the NVTX range dbk_step, "
                         "print its attention bytes and exit (profiles/run_ncu_traffic.sh)")
    ap.add_argument("--per-layer-launches", action="store_true",
                    help="one PDL-chained decode launch per layer (as a model's step issues them) instead of "
                         "multi-layer launches")
    ap.add_argument("--model", action="store_true",
                    help="full decode step: synthetic-weight QKV/O/MLP/LM-head GEMMs around the attention")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
