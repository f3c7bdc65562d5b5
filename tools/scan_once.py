"""One inclusive scan (fp32) of 2^log2n elements after two warm-ups: a short command to run
under ncu (tools for profiles/).  --view affine|product scans a fused view instead."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, repro, views  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
view = sys.argv[2] if len(sys.argv) > 2 else ""
DTYPE = {"f32": np.float32, "i32": np.int32, "f64": np.float64}[sys.argv[3] if len(sys.argv) > 3 else "f32"]
n = 1 << lg
rt = sr.Runtime(1)
x = sr.DistributedVector(rt, n, dtype=DTYPE)
y = sr.DistributedVector(rt, n, dtype=DTYPE)
repro.fill_mod(x, 1, 0, 3, -1)
repro.fill_mod(y, 2, 0, 3, -1)
out = sr.DistributedVector(rt, n, dtype=DTYPE)
src = {"-": x, "": x, "affine": views.transform(x, lambda v: 2.5 * v + 1.0),
       "product": views.transform(views.zip(x, y), lambda t: t[0] * t[1])}[view]
for _ in range(3):
    A.inclusive_scan(src, out)
rt.synchronize()
