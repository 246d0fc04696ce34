"""Trace one host-pointer pipeline call (SKYGPU_TRACE=1 prints device/host marks)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2412_02274_b200 as sk  # noqa: E402
from paper_2412_02274_b200 import skypar  # noqa: E402

gen, n, d = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
v = sk.generate(gen, n, d, 1)
pv = torch.from_numpy(v).pin_memory()
pi = torch.from_numpy(np.arange(n, dtype=np.int64)).pin_memory()
pos = torch.empty(n, dtype=torch.int64).pin_memory()
den = torch.empty(n, dtype=torch.int32).pin_memory()
plan = sk.make_plan("angular", 16, d)
for i in range(6):
    t0 = time.perf_counter()
    skypar.pipeline_raw(pv.data_ptr(), pi.data_ptr(), n, d, plan, 25, 0, 0, 1, 0, pos.data_ptr(),
                        den.data_ptr())
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for mode in ("flush+sync", "sync only", "sleep 1ms"):
    ts = []
    for i in range(10):
        if mode == "flush+sync":
            flush.zero_()
        torch.cuda.synchronize()
        if mode == "sleep 1ms":
            time.sleep(0.001)
        t0 = time.perf_counter()
        skypar.pipeline_raw(pv.data_ptr(), pi.data_ptr(), n, d, plan, 25, 0, 0, 1, 0, pos.data_ptr(),
                            den.data_ptr())
        ts.append(1e3 * (time.perf_counter() - t0))
    ts.sort()
    print(f"{mode}: median {ts[5]:.3f} ms min {ts[0]:.3f}", file=sys.stderr, flush=True)
