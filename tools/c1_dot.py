"""C1 (BASELINE configs[0]): dot_product via zip|transform|reduce on two fp32 vectors,
n = 2^24, 2 segments — time per API call (host overhead included) and per kernel."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import bench as B, kernels
from oracle import segrange_port as O

n, p = 1 << 24, 2
x = O.unit_doubles(1, 0, n).astype(np.float32)
y = O.unit_doubles(1, n, n).astype(np.float32)
rt = sr.Runtime(p)
vx, vy = sr.DistributedVector.from_numpy(rt, x), sr.DistributedVector.from_numpy(rt, y)
for _ in range(20):
    d = B.dot_product(vx, vy)
reps = 200
t0 = time.perf_counter()
for _ in range(reps):
    d = B.dot_product(vx, vy)
api_us = (time.perf_counter() - t0) / reps * 1e6
with kernels.profile() as prof:
    for _ in range(50):
        B.dot_product(vx, vy)
torch.cuda.synchronize()
summ = prof.summary()
name = "drk_dot_batch" if "drk_dot_batch" in summ else "drk_dot"  # one batched launch when both segments share a GPU
cnt, ms, el = summ[name]
kern_us = ms / 50 * 1e3  # device time per API call
want = O.dot(x, y, p)
# CPU reference path (oracle port of segrange, numpy, 2 segments on 2 threads)
t0 = time.perf_counter()
for _ in range(5):
    O.dot(x, y, p, threads=p)
cpu_ms = (time.perf_counter() - t0) / 5 * 1e3
print(json.dumps({"config": "C1 dot fp32 n=2^24 P=2 (both segments on GPU 0)", "result": d, "oracle": want,
                  "rel_err": abs(d - want) / want, "api_us_per_call": round(api_us, 1),
                  "kernel": name, "kernel_us_per_call": round(kern_us, 2),
                  "GB/s_api": round(8 * n / (api_us * 1e-6) / 1e9, 1),
                  "GB/s_kernels": round(8 * n / (kern_us * 1e-6) / 1e9, 1),
                  "cpu_port_ms": round(cpu_ms, 2)}))

if os.environ.get("C1_PROFILE"):
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        B.dot_product(vx, vy)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
