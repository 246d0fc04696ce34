"""H2D of 32 MiB under different conditions (GPU idle vs busy, page size)."""
import time

import torch

dev = torch.device("cuda", 0)
n = 32 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device=dev)
big = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def one(label, busy=False, reps=20):
    ts = []
    s2 = torch.cuda.Stream()
    for _ in range(reps):
        torch.cuda.synchronize()
        if busy:
            with torch.cuda.stream(s2):
                for _ in range(20):
                    big.mul_(1.0001)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{label}: median {ts[len(ts)//2]:.3f} ms ({32 / 1024 / (ts[len(ts)//2] / 1e3):.1f} GiB/s), best {ts[0]:.3f}")


one("idle")
one("busy", busy=True)
one("idle again")
# chunked
for chunks in (2, 8):
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        q = n // chunks
        for i in range(chunks):
            d[i * q:(i + 1) * q].copy_(h[i * q:(i + 1) * q], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{chunks} chunks: median {ts[10]:.3f} ms")
