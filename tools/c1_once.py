"""C1 (dot fp32, 2^24 elements, 2 segments on one GPU) three times: a short command for ncu."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import bench as B, repro  # noqa: E402

n = 1 << 24
rt = sr.Runtime(2, devices=[0])
x = sr.DistributedVector(rt, n, dtype=np.float32)
y = sr.DistributedVector(rt, n, dtype=np.float32)
repro.fill_unit(x, 1, 0)
repro.fill_unit(y, 1, n)
for _ in range(3):
    B.dot_product(x, y)
