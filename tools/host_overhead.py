"""Host overhead per API call at small n (one GPU): wall time of reduce / transform /
inclusive_scan / dot on 2^16-element fp32 vectors (device time is ~1-3 us, so the wall time
is the host path), and a cProfile of each.

    python tools/host_overhead.py [--profile]
"""
import cProfile
import json
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, bench as B, repro  # noqa: E402

n = 1 << 16
rt = sr.Runtime(1)
x = sr.DistributedVector(rt, n, dtype=np.float32)
repro.fill_mod(x, 1, 0, 3, -1)
y = sr.DistributedVector(rt, n, dtype=np.float32)
a = sr.DistributedVector(rt, n, dtype=np.float32)
ops = {
    "reduce": lambda: A.reduce(x, 0.0),
    "transform": lambda: A.transform(x, y, lambda v: v * 2.0 + 1.0),
    "scan": lambda: A.inclusive_scan(x, y),
    "dot": lambda: B.dot_product(x, y),
    "triad": lambda: B.stream_triad(a, x, y),
}
out = {}
for name, f in ops.items():
    for _ in range(50):
        f()
    torch.cuda.synchronize()
    reps = 2000
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    out[name] = round((time.perf_counter() - t0) / reps * 1e6, 1)
# C1: dot at 2^24 over 2 segments (one batched launch), per API call and kernel alone
rt2 = sr.Runtime(2, devices=[0])
n1 = 1 << 24
cx = sr.DistributedVector(rt2, n1, dtype=np.float32)
cy = sr.DistributedVector(rt2, n1, dtype=np.float32)
repro.fill_unit(cx, 1, 0)
repro.fill_unit(cy, 1, n1)
for _ in range(50):
    B.dot_product(cx, cy)
torch.cuda.synchronize()
reps = 1000
t0 = time.perf_counter()
for _ in range(reps):
    B.dot_product(cx, cy)
out["c1_dot_2^24_p2"] = round((time.perf_counter() - t0) / reps * 1e6, 1)
from paper_2406_00158_b200 import kernels  # noqa: E402
with kernels.profile() as prof:
    for _ in range(200):
        B.dot_product(cx, cy)
    torch.cuda.synchronize()
ks = prof.summary()
out["c1_kernel_us"] = {k: round(v[1] / v[0] * 1e3, 1) for k, v in ks.items()}
print(json.dumps({"us_per_call": out, "n": n}), flush=True)
if "--profile" in sys.argv:
    for name, f in ops.items():
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(500):
            f()
        pr.disable()
        print(f"===== {name}")
        pstats.Stats(pr).sort_stats("tottime").print_stats(14)
