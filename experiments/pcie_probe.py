"""Host<->device copy bandwidth on this box (pinned memory), alone and both directions at once:
the ceiling of bench.py's e2e number (q + new K/V in, outputs out every step)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch


def bw(fn, nbytes, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return nbytes * reps / (s.elapsed_time(e) / 1e3) / 1e9


def main():
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {"h2d_gbs": bw(lambda: d.copy_(h, non_blocking=True), n),
           "d2h_gbs": bw(lambda: h.copy_(d, non_blocking=True), n)}

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    out["bidir_total_gbs"] = bw(both, 2 * n)
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()


def under_load():
    """H2D bandwidth while an HBM-bound kernel (a 40 GB reduction) runs on another stream."""
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    big = torch.ones(20 << 30, dtype=torch.float16, device="cuda")
    s_copy, s_load = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1, l0, l1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(s_load):
        l0.record()
        for _ in range(3):
            big.sum()
        l1.record()
    with torch.cuda.stream(s_copy):
        e0.record()
        for _ in range(4):
            d.copy_(h, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    load_ms, copy_ms = l0.elapsed_time(l1), e0.elapsed_time(e1)
    print(json.dumps({"h2d_under_load_gbs": round(4 * n / (copy_ms / 1e3) / 1e9, 1),
                      "load_kernel_gbs": round(3 * big.numel() * 2 / (load_ms / 1e3) / 1e9, 1),
                      "copy_ms": round(copy_ms, 2), "load_ms": round(load_ms, 2)}))


if __name__ == "__main__":
    under_load()


def under_read_probe():
    """H2D bandwidth while libdbk's read-only streaming probe (~7 TB/s) saturates HBM."""
    import ctypes
    import paper_2503_05248_b200 as dbk
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    big = torch.ones(40 << 30, dtype=torch.uint8, device="cuda")
    s_copy, s_load = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_copy):
        e0.record()
        for _ in range(8):
            d.copy_(h, non_blocking=True)
        e1.record()
    ms = ctypes.c_double()
    dbk._lib.dbk_probe_read_bandwidth(big.data_ptr(), big.numel(), 0, s_load.cuda_stream, ctypes.byref(ms))
    torch.cuda.synchronize()
    copy_ms = e0.elapsed_time(e1)
    print(json.dumps({"h2d_while_read_probe_gbs": round(8 * n / (copy_ms / 1e3) / 1e9, 1),
                      "read_probe_gbs": round(big.numel() / (ms.value / 1e3) / 1e9, 1),
                      "copy_ms": round(copy_ms, 2), "probe_ms": round(ms.value, 2)}))


if __name__ == "__main__":
    under_read_probe()
