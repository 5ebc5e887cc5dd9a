"""The README quick start, runnable (python experiments/quickstart.py on a B200)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch, paper_2503_05248_b200 as dbk

# paged KV pool over caller-owned HBM: 32 layers, 32 q / 32 kv heads x 128, 4096 pages of 16 tokens
pool = dbk.KVPool(32, 32, 32, 128, cap_pages=4096, max_requests=64, max_pages_per_req=256, kv_dtype="f16")
pool.request_begin(7, l_in=100, l_out=50)              # request id, prompt and target output length
pool.append_tokens([7], [101], seed=1)                  # K/V of 101 tokens (synthetic here; or k=, v= tensors)
q = torch.randn(1, 32, 128, dtype=torch.float16, device="cuda")
out = torch.empty(1, 32, 128, dtype=torch.float32, device="cuda")
pool.decode_step([7], layer=0, q=q, out=out, out_dtype=2, fuse_stats=True)   # K1/K2 + fused telemetry
stats = pool.batch_stats()                              # n_active, sum_ctx, pages vs cap, finishing sums ...

# Alg. 1 (memory, Eq. 11 buffer) / Alg. 2 (SLA feedback) / min -- integer-exact host C++
sched = dbk.Scheduler(policy=3, b_static=256, b_min=1, b_max=512, b0=1, eps_m=0.02,
                      bytes_per_token=2 * 32 * 32 * 128 * 2, page_size=16, d_sla_ms=50.0, eps_d_ms=2.0)
b_next, why = sched.choose(dict(stats, step_ns=16_000_000), mem_cap_bytes=4096 * 16 * 2 * 32 * 32 * 128 * 2)

# the whole loop: dbk.Engine(pool, sched, arrivals_ns, l_in, l_out, mem_cap) + engine.step(buffers);
# attach_model(dbk.Model(pool, hidden, ffn, vocab)) for the full decode step with weights,
# pd_fusion=True for chunked prefill (K7), preempt_mode=1 + pool.swap_space_attach(...) for swap.

print('readme ok', b_next, why, stats['n_active'])
