"""C5 sweep (one GPU): reduce / transform / inclusive_scan on fp32 vectors of 2^20..2^32
elements through the public API, against the CPU reference path (oracle port) up to 2^30.

For each size: per-call wall time (host overhead included), kernel time from CUDA events
(launches queued behind a GPU sleep; the fastest of five calls),
GB/s on algorithmic bytes (reduce 4, transform 8, scan 8 per element), and a
size-independent check (scan last == reduce; transform sample exact)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A, kernels, repro, views
from oracle import segrange_port as O

BYTES = {"reduce": 4, "transform": 8, "scan": 8}
sizes = [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else "20,22,24,26,28,30,32".split(","))]
threads = len(os.sched_getaffinity(0))
rt = sr.Runtime(1)
rows = []
for lg in sizes:
    n = 1 << lg
    x = sr.DistributedVector(rt, n, dtype=np.float32)
    repro.fill_mod(x, 1, 0, 3, -1)   # {-1,0,1}: exact fp32 sums at any n
    y = sr.DistributedVector(rt, n, dtype=np.float32)
    ops = {
        "reduce": lambda: A.reduce(x, 0.0),
        "transform": lambda: A.transform(x, y, lambda v: v * 2.0 + 1.0),
        "scan": lambda: A.inclusive_scan(x, y),
    }
    row = {"log2n": lg}
    for name, f in ops.items():
        f(); torch.cuda.synchronize()
        reps = max(3, min(50, (1 << 28) // n))
        t0 = time.perf_counter()
        for _ in range(reps):
            r = f()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps
        # kernel time: launches queued behind a GPU sleep, so the events bracket the kernel
        # and not the host's launch latency (a reduce waits for its result, so only its first
        # call is queued: the minimum over calls is the kernel time)
        with kernels.profile() as prof:
            with torch.cuda.stream(rt.device_states[0].stream):
                torch.cuda._sleep(int(4e6))
            for _ in range(5):
                f()
        torch.cuda.synchronize()
        per_call = {}
        for nm, recs in prof.records.items():
            for k, (s, e, _) in enumerate(recs):
                per_call.setdefault(k, 0.0)
                per_call[k] += s.elapsed_time(e)
        kms = min(per_call.values())
        row[name] = {"api_GBps": round(BYTES[name] * n / wall / 1e9, 1),
                     "kernel_GBps": round(BYTES[name] * n / (kms * 1e-3) / 1e9, 1),
                     "api_us": round(wall * 1e6, 1), "kernel_us": round(kms * 1e3, 1)}
        if name == "reduce":
            total = r
    row["check_scan_last_eq_reduce"] = bool(y[n - 1] == total)
    A.transform(x, y, lambda v: v * 2.0 + 1.0)
    seg = y.segments()[0]
    head = seg.to_numpy()[:4096] if n <= (1 << 24) else None
    if lg <= 30:
        xs = O.mod_ints(1, 0, n, 3, -1).astype(np.float32)
        cpu = {}
        for name, f in (("reduce", lambda: O.reduce(xs, threads, 0.0, np.add, threads)),
                        ("transform", lambda: O.triad(xs, xs, 0.0, threads, threads)),
                        ("scan", lambda: O.scan(xs, threads, np.float32, threads=threads))):
            t0 = time.perf_counter(); f(); cpu[name] = round(BYTES[name] * n / (time.perf_counter() - t0) / 1e9, 2)
        row["cpu_GBps"] = cpu
    rows.append(row)
    print(json.dumps(row), flush=True)
    del x, y
    torch.cuda.empty_cache()
print(json.dumps({"cpu_threads": threads, "rows": rows}))
