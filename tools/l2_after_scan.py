"""Why is dot slower right after a scan?  Times drk_dot on 2^30 fp32 alone, after drk_triad,
after drk_scan, and after drk_scan followed by cudaCtxResetPersistingL2Cache (which returns
evict_last / persisting L2 lines to normal priority).

    python tools/l2_after_scan.py
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_00158_b200 import _lib  # noqa: E402

n = 1 << 30
lib = _lib.load()
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
a = torch.empty(n, dtype=torch.float32, device=dev)
b = torch.rand(n, dtype=torch.float32, device=dev)
c = torch.rand(n, dtype=torch.float32, device=dev)
red = torch.zeros(lib.drk_reduce_scratch_bytes(), dtype=torch.uint8, device=dev)
res = torch.zeros(4, dtype=torch.float64, device=dev)
sb = lib.drk_scan_scratch_bytes(_lib.F32, _lib.ADD, n)
scr = torch.zeros(sb + 4096, dtype=torch.uint8, device=dev)
alpha = _lib.scalar_buffer(3.0, np.float32)
cudart = None
for cand in ("libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so"):
    try:
        cudart = ctypes.CDLL(cand)
        break
    except OSError:
        pass


def dot():
    _lib.call("drk_dot", _lib.F32, b.data_ptr(), c.data_ptr(), n, res.data_ptr(), red.data_ptr(), 0, s)


def triad():
    _lib.call("drk_triad", _lib.F32, a.data_ptr(), b.data_ptr(), c.data_ptr(), n, alpha, 0, s)


def scan():
    _lib.call("drk_scan", _lib.F32, _lib.ADD, 0, c.data_ptr(), a.data_ptr(), n, None, None, None, None, None,
              scr.data_ptr(), scr.numel(), 0, s)


def reset():
    torch.cuda.synchronize()
    rc = cudart.cudaCtxResetPersistingL2Cache() if cudart is not None else -1
    torch.cuda.synchronize()
    return rc


def timed_dot(before, reps=10):
    ts = []
    for _ in range(reps):
        before()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dot()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(float(np.median(ts)), 4)


out = {
    "alone": timed_dot(lambda: None),
    "after_triad": timed_dot(triad),
    "after_scan": timed_dot(scan),
    "after_scan_sync": timed_dot(lambda: (scan(), torch.cuda.synchronize())),
    "after_scan_reset": timed_dot(lambda: (scan(), reset())),
    "after_triad_sync": timed_dot(lambda: (triad(), torch.cuda.synchronize())),
}
print(json.dumps(out))
