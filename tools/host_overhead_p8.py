"""Host cost of one inclusive_scan over 8 segments on one GPU (2^20 elements each, so the
device time is small): wall time per call and a cProfile of the host path."""
import cProfile, os, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A, repro
rt = sr.Runtime(8)
n = 8 << 20
x = sr.DistributedVector(rt, n, dtype=np.float32); repro.fill_mod(x, 1, 0, 3, -1)
y = sr.DistributedVector(rt, n, dtype=np.float32)
for _ in range(20): A.inclusive_scan(x, y)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): A.inclusive_scan(x, y)
torch.cuda.synchronize()
print("us per call", round((time.perf_counter() - t0) / 200 * 1e6, 1))
pr = cProfile.Profile(); pr.enable()
for _ in range(200): A.inclusive_scan(x, y)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
