"""Reduce combine modes (Runtime reduce_combine = host / device / nccl): API time per call of
C1 (dot, 2^24 fp32, 2 segments) and of a 2^16-element reduce over 8 segments, on the visible
GPUs (one GPU: every segment on GPU 0, a one-rank NCCL communicator)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, bench as B, repro  # noqa: E402


def per_call(f, reps):
    for _ in range(20):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t0) / reps * 1e6


for mode in ("host", "device", "nccl", "fused"):
    rt = sr.Runtime(2, reduce_combine=mode)
    n = 1 << 24
    x = sr.DistributedVector(rt, n, dtype=np.float32)
    y = sr.DistributedVector(rt, n, dtype=np.float32)
    repro.fill_unit(x, 1, 0)
    repro.fill_unit(y, 1, n)
    c1 = per_call(lambda: B.dot_product(x, y), 500)
    d = B.dot_product(x, y)
    rt8 = sr.Runtime(8, reduce_combine=mode)
    v = sr.DistributedVector(rt8, 1 << 16, dtype=np.float32)
    repro.fill_unit(v, 1, 0)
    r8 = per_call(lambda: A.reduce(v, 0.0), 2000)
    print(json.dumps({"mode": mode, "c1_dot_us": round(c1, 1), "reduce_2^16_p8_us": round(r8, 1), "dot": d}),
          flush=True)
    rt.close()
    rt8.close()
