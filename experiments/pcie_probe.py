"""Host<->device copy bandwidth on this box (pinned memory), alone and both directions at once:
the ceiling of bench.py's e2e number (q + new K/V in, outputs out every step)."""
import json
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
