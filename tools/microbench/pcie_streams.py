"""H2D throughput of 512 MiB of pinned 16 MiB buffers (the c2 leaves) over 1, 2 or 4 CUDA
streams (round-robin), and with a cuStreamWriteValue-like event between copies."""
import torch

dev = torch.device("cuda:0")
n, mb = 32, 16
host = [torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
devb = [torch.empty(mb << 20, dtype=torch.uint8, device=dev) for _ in range(n)]
for k in (1, 2, 4):
    ss = [torch.cuda.Stream(device=dev) for _ in range(k)]
    best = 1e9
    for rep in range(6):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ss[0])
        for s in ss[1:]:
            s.wait_event(e0)
        for i in range(n):
            with torch.cuda.stream(ss[i % k]):
                devb[i].copy_(host[i], non_blocking=True)
        for s in ss[1:]:
            ev = torch.cuda.Event()
            ev.record(s)
            ss[0].wait_event(ev)
        e1.record(ss[0])
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print("%d stream(s): %.3f ms for %d MiB = %.1f GB/s" % (k, best, n * mb, n * mb * 1048576 / best / 1e6))
