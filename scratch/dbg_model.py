import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2503_05248_b200 as dbk
from oracle import model as om
from synth import hashgen
from test_gpu_model import _setup, _read_kv, rel_l2
s = om.ModelShape(layers=1, q_heads=4, kv_heads=4, head_dim=64, hidden=256, ffn=384, vocab=300)
ctx = [5]
pool, model, ids, ref = _setup(dbk, s, ctx, 5, 11)
pool.reserve_tokens(ids, [1])
model.step(ids)
torch.cuda.synchronize()
ptrs = (C.c_void_p * 8)()
dbk._lib.dbk_model_buffers(model.h, ptrs)
import glob, os, nvidia
rt = C.CDLL(glob.glob(os.path.join(os.path.dirname(nvidia.__path__[0] + "/"), "cuda_runtime/lib/libcudart.so*"))[0])
def grab(k, numel, dt):
    t = torch.empty(numel, dtype=dt, device="cuda")
    assert rt.cudaMemcpy(C.c_void_p(t.data_ptr()), C.c_void_p(ptrs[k]), C.c_size_t(numel * t.element_size()), 3) == 0
    return t.float().cpu().numpy()
W = om.weights(11, s, 0)
tok = int(hashgen.gen_token(11, ids[0], 4, s.vocab))
x0 = om.embed_rows(11, s, [tok])[0]
h0 = om.rmsnorm(x0, W["g1"], 1e-5)
qkv = grab(2, 768, torch.float16)
print("qkv got", qkv[:6], "want", (h0 @ W["w_qkv"].T)[:6])
wt = model.weights[:256 * 300 * 2].view(torch.float16).float().cpu().numpy().reshape(300, 256)
print("embed rows match", np.abs(wt - om.embed_rows(11, s, np.arange(300))).max())

print("h got", grab(1, 256, torch.float16)[:6])
x = grab(0, 256, torch.float32)
print("x got", x[:6])
