import ctypes as C, glob, os, json, torch, nvidia
rt = C.CDLL(glob.glob(os.path.join(nvidia.__path__[0], "cuda_runtime/lib/libcudart.so*"))[0])
L, n, row = 32, 512, 8192
hk = torch.empty(n * L * row, dtype=torch.uint8, pin_memory=True)
dk = torch.empty(n * L * row, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
def run(kind):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        e0.record()
        for rep in range(3):
            for l in range(L):
                if kind == "2d":
                    r = rt.cudaMemcpy2DAsync(C.c_void_p(dk.data_ptr() + l * row), C.c_size_t(L * row),
                                             C.c_void_p(hk.data_ptr() + l * row), C.c_size_t(L * row),
                                             C.c_size_t(row), C.c_size_t(n), 1, C.c_void_p(s.cuda_stream))
                    assert r == 0
                else:
                    off = l * n * row
                    dk[off:off + n * row].copy_(hk[off:off + n * row], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    return 3 * L * n * row / (e0.elapsed_time(e1) / 1e3) / 1e9
print(json.dumps({"1d_4MB_chunks_gbs": round(run("1d"), 1), "2d_8KB_rows_gbs": round(run("2d"), 1)}))
