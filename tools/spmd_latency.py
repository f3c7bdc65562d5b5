"""Latency of the one-process-per-GPU reduce (C1-like dot, 2^20 fp32 per rank) with the
exchange as an NCCL all-gather vs the peer-memory mailbox kernel (run under torchrun; with
one rank on one GPU both paths run their full code)."""
import json, os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, repro, spmd, views  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rt = sr.Runtime(1, devices=[local])
n = 1 << 20
x = sr.DistributedVector(rt, n, dtype=np.float32)
y = sr.DistributedVector(rt, n, dtype=np.float32)
repro.fill_unit(x, 1, 0)
repro.fill_unit(y, 1, n)
z = views.transform(views.zip(x, y), lambda t: t[0] * t[1])
out = sr.DistributedVector(rt, n, dtype=np.float32)
for combine in ("collective", "ipc"):
    g = spmd.Group(combine=combine)
    for name, f in (("dot", lambda: spmd.reduce(z, 0.0, A.add, g)), ("scan", lambda: spmd.inclusive_scan(x, out, g))):
        for _ in range(20):
            f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            f()
        torch.cuda.synchronize()
        us = (time.perf_counter() - t0) / 200 * 1e6
        if dist.get_rank() == 0:
            print(json.dumps({"combine": combine, "op": name, "us_per_call": round(us, 1)}), flush=True)
if "--profile" in sys.argv and dist.get_rank() == 0:
    import cProfile, pstats
    g = spmd.Group(combine="ipc")
    for name, f in (("dot", lambda: spmd.reduce(z, 0.0, A.add, g)), ("scan", lambda: spmd.inclusive_scan(x, out, g))):
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(200):
            f()
        pr.disable()
        print("=====", name)
        pstats.Stats(pr).sort_stats("tottime").print_stats(12)
dist.destroy_process_group()
