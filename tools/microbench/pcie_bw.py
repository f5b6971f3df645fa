"""Pinned host <-> device copy bandwidth on the GPU box (PCIe roofline for DESIGN.md)."""
import torch


def bw(n_bytes, direction, reps=5):
    host = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(n_bytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = 1e30
    with torch.cuda.stream(s):
        for _ in range(reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if direction == "h2d":
                dev.copy_(host, non_blocking=True)
            else:
                host.copy_(dev, non_blocking=True)
            e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
    return n_bytes / (best * 1e-3) / 1e9


if __name__ == "__main__":
    for mb in (16, 256, 2048):
        n = mb << 20
        print(f"{mb:5d} MiB  h2d {bw(n, 'h2d'):7.1f} GB/s   d2h {bw(n, 'd2h'):7.1f} GB/s")
    # simultaneous both directions
    n = 1 << 30
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    print(f"bidirectional 1 GiB each: {2 * n / t / 1e9:.1f} GB/s aggregate")
