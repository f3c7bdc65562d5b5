import os, sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A, repro
n = 1 << 30
rt = sr.Runtime(8)
x = sr.DistributedVector(rt, n, dtype=np.float32); repro.fill_mod(x, 1, 0, 3, -1)
y = sr.DistributedVector(rt, n, dtype=np.float32)
for chain in (True, False, True):
    A._CHAIN_SCANS = chain
    A.inclusive_scan(x, y); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10): A.inclusive_scan(x, y)
    torch.cuda.synchronize()
    print("chain" if chain else "plain", round((time.perf_counter() - t0) / 10 * 1e3, 3), "ms", flush=True)
