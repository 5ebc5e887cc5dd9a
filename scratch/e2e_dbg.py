import sys, os, torch
sys.path.insert(0, ".")
os.environ["DBK_E2E_DEBUG"] = "1"
import bench
S = bench.setup_engine(cfg_name="llama2-7b")
eng = S["eng"]; stream = torch.cuda.current_stream()
bench.run_steps(S, 300, eng.buffers(S["qd"], S["od"]), stream)
L, Hq, Hkv, d, mr = S["L"], S["Hq"], S["Hkv"], S["d"], S["max_req"]
hq = torch.empty(L * mr * Hq * d, dtype=torch.float16, pin_memory=True)
hk = torch.empty(mr * L * Hkv * d, dtype=torch.float16, pin_memory=True)
hv = torch.empty(mr * L * Hkv * d, dtype=torch.float16, pin_memory=True)
ho = torch.empty(L * mr * Hq * d, dtype=torch.float16, pin_memory=True)
bench.run_steps(S, 6, eng.buffers(S["qd"], S["od"], S["kvd"], hq, hk, hv, ho), stream)
