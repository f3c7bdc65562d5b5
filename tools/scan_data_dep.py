"""Does the scan's time at 2^30 depend on the data?  fp32 / int32 inclusive scans of zeros,
{-1, 0, 1} and uniform data (kernel time from CUDA events, GPU queue kept full)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, kernels, repro  # noqa: E402

n = 1 << 30
rt = sr.Runtime(1)
st = rt.device_states[0]
for dt in (np.float32, np.int32):
    x = sr.DistributedVector(rt, n, dtype=dt)
    out = sr.DistributedVector(rt, n, dtype=dt)
    for name, fill in (("zeros", lambda: sr.fill(x, 0)), ("mod3", lambda: repro.fill_mod(x, 1, 0, 3, -1)),
                       ("wide", lambda: repro.fill_mod(x, 1, 0, 2001, -1000) if dt == np.int32
                        else repro.fill_unit(x, 1, 0))):
        fill()
        for _ in range(3):
            A.inclusive_scan(x, out)
        rt.synchronize()
        with kernels.profile() as prof:
            with torch.cuda.stream(st.stream):
                torch.cuda._sleep(int(4e6))
            for _ in range(10):
                A.inclusive_scan(x, out)
            rt.synchronize()
        t = sorted(s.elapsed_time(e) for recs in prof.records.values() for s, e, _ in recs)
        print(json.dumps({"dtype": np.dtype(dt).name, "data": name, "ms": round(t[len(t) // 2], 4)}), flush=True)
    del x, out
