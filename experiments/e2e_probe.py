import sys, json, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
S = bench.setup_engine(cfg_name="llama2-7b")
eng = S["eng"]; stream = torch.cuda.current_stream()
bufs = eng.buffers(S["qd"], S["od"])
bench.run_steps(S, 300, bufs, stream)
L, Hq, Hkv, d, mr = S["L"], S["Hq"], S["Hkv"], S["d"], S["max_req"]
hq = torch.empty(L * mr * Hq * d, dtype=torch.float16, pin_memory=True).uniform_(-1, 1)
hk = torch.empty(mr * L * Hkv * d, dtype=torch.float16, pin_memory=True).uniform_(-1, 1)
hv = torch.empty(mr * L * Hkv * d, dtype=torch.float16, pin_memory=True).uniform_(-1, 1)
ho = torch.empty(L * mr * Hq * d, dtype=torch.float16, pin_memory=True)
out = {}
for name, b in [("resident", bufs), ("e2e", eng.buffers(S["qd"], S["od"], S["kvd"], hq, hk, hv, ho)),
                ("e2e_no_out", eng.buffers(S["qd"], S["od"], S["kvd"], hq, hk, hv, None)), ("resident2", bufs)]:
    bench.run_steps(S, 3, b, stream)
    eng.attn_timing(reset=True)
    recs, ms = bench.run_steps(S, 20, b, stream)
    a_ms, a_n, a_b = eng.attn_timing(reset=True)
    out[name] = dict(ms_per_step=ms / len(recs), attn_ms_per_step=a_ms / len(recs),
                     step_ns_mean=sum(r["step_ns"] for r in recs) / len(recs) / 1e6,
                     n=sum(r["n_decode"] for r in recs) / len(recs))
print(json.dumps(out, indent=1))
