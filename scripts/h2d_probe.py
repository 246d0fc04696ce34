"""Host->device copy bandwidth from pinned memory (e2e context)."""
import os
import time

import torch

try:
    import pynvml
    pynvml.nvmlInitWithFlags(0) if hasattr(pynvml, "nvmlInitWithFlags") else pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    aff = pynvml.nvmlDeviceGetCpuAffinity(h, 8)
    cpus = [w * 64 + b for w, word in enumerate(aff) for b in range(64) if word >> b & 1]
    print("gpu0 cpu affinity", cpus[:4], "...", len(cpus), "cpus; process affinity", len(os.sched_getaffinity(0)))
    print("numa nodes", sorted(os.listdir("/sys/devices/system/node")) if os.path.exists("/sys/devices/system/node") else None)
except Exception as e:
    print("nvml", e)
dev = torch.device("cuda", 0)
for mb in [int(x) for x in os.environ.get('SIZES', '32 128 640 32 8').split()]:
    n = mb * 1024 * 1024 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"H2D {mb} MiB: {mb / 1024 / dt:.1f} GiB/s back-to-back")
    iso = []
    for _ in range(5):
        torch.cuda.synchronize()
        time.sleep(0.002)
        t0 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        iso.append(time.perf_counter() - t0)
    print(f"H2D {mb} MiB isolated: {mb / 1024 / min(iso):.1f} GiB/s best, {mb / 1024 / max(iso):.1f} worst")
    # split over 4 streams
    ss = [torch.cuda.Stream() for _ in range(4)]
    q = n // 4
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        for i, s_ in enumerate(ss):
            with torch.cuda.stream(s_):
                d[i * q:(i + 1) * q].copy_(h[i * q:(i + 1) * q], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"H2D {mb} MiB on 4 streams: {mb / 1024 / dt:.1f} GiB/s")
    t0 = time.perf_counter()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"D2H {mb} MiB: {mb / 1024 / dt:.1f} GiB/s")
