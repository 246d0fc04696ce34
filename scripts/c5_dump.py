"""GPU side of the full-scale C5 CPU-oracle check: run the pipeline on the
10 M-tuple, d = 7 config and dump the skyline (membership bitmask over the
input) and the denominators aligned with ascending input position."""
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_2412_02274_b200 as sk  # noqa: E402

v = sk.generate("ant", 10_000_000, 7, 1)
res = sk.pipeline(v, None, sk.make_plan("angular", 64, 7), cap=25)
order = np.argsort(res.positions)
pos = res.positions[order]
den = res.den[order].astype(np.uint8)
mask = np.zeros(len(v), dtype=bool)
mask[pos] = True
np.savez_compressed("gpurun_out/c5_full_gpu.npz", mask=np.packbits(mask), den=den,
                    g_max=res.g_max, engine=res.stats["gres_engine"])
print("S", len(pos), "g_max", res.g_max, "gres_engine", res.stats["gres_engine"])
