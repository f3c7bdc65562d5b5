"""Black-Scholes at 2^26 options: two reference-precision launches, then two fast-tier ones (for ncu)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import bench as B, repro
n = 1 << 26
rt = sr.Runtime(1)
cols = []
for k, (lo, hi) in enumerate(B.BS_RANGES.values()):
    v = sr.DistributedVector(rt, n, dtype=np.float32); repro.fill_uniform(v, 1, k * n, lo, hi); cols.append(v)
out = sr.DistributedVector(rt, n, dtype=np.float32)
for _ in range(2):
    B.black_scholes_prices(out, *cols)
for _ in range(2):
    B.black_scholes_prices(out, *cols, precision="fast")
rt.synchronize()
