"""Observed model-step errors vs the fp64 oracle (for the R35 tolerance record)."""
import sys, json, numpy as np, torch
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, ROOT)
import paper_2503_05248_b200 as dbk
from oracle import model as om
from test_gpu_model import _setup, _read_kv, rel_l2
out = {}
for name, s, ctx in [("small-mha", om.ModelShape(2, 4, 4, 64, 256, 384, 300), [1, 2, 16, 17, 33, 100, 257]),
                     ("gqa-3layer", om.ModelShape(3, 8, 2, 128, 512, 640, 1000), [1, 2, 16, 17, 33, 100, 257]),
                     ("7b-1layer", om.ModelShape(1, 32, 32, 128, 4096, 11008, 32000), [3, 190, 573, 1100])]:
    pool, model, ids, ref = _setup(dbk, s, ctx, 5, 11)
    pool.reserve_tokens(ids, [1] * len(ids))
    logits = torch.empty(len(ids), s.vocab, dtype=torch.float32, device="cuda")
    model.step(ids, logits)
    want, nk, nv, _ = om.decode_step(s, 11, 5, ids, ctx)
    ke = max(rel_l2(_read_kv(pool, s, r, c - 1, l)[0], nk[l, i]) for l in range(s.layers) for i, (r, c) in enumerate(zip(ids, ctx)))
    ve = max(rel_l2(_read_kv(pool, s, r, c - 1, l)[1], nv[l, i]) for l in range(s.layers) for i, (r, c) in enumerate(zip(ids, ctx)))
    out[name] = dict(logits_rel_l2=float(rel_l2(logits.cpu().numpy(), want)), k_rel_l2=float(ke), v_rel_l2=float(ve))
    model.close(); pool.close()
print(json.dumps(out))
