import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2412_02274_b200 as sk
v = sk.generate("ant", 1_000_000, 3, 1)
ids = np.arange(len(v), dtype=np.int64)
for p in (1, 16):
    pids = (np.arange(len(v)) % p).astype(np.int64)
    for rep in range(3):
        t0 = time.perf_counter()
        a = sk.sfs_accounting(v, ids, pids, p)
        print(p, rep, f"{1e3*(time.perf_counter()-t0):.1f} ms", int(a.per_partition.max()), a.final_tests, flush=True)
