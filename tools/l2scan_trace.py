"""Per-iteration phases of the L2-resident scan (debug trace in libdrk)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_00158_b200 import _lib

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dt = sys.argv[2] if len(sys.argv) > 2 else "float32"
n = 1 << log2n
lib = _lib.load()
for kv in (sys.argv[3].split(",") if len(sys.argv) > 3 else []):
    k, v = kv.split("="); lib.drk_tune(k.encode(), int(v))
dev = torch.device("cuda", 0)
code = {"float32": _lib.F32, "int32": _lib.I32, "float64": _lib.F64}[dt]
x = (torch.rand(n, device=dev) * 10).to(getattr(torch, dt))
y = torch.empty_like(x)
sb = lib.drk_scan_scratch_bytes(code, _lib.ADD, n)
scratch = torch.zeros(sb + 4096, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream().cuda_stream
call = lambda: _lib.call("drk_scan", code, _lib.ADD, 0, x.data_ptr(), y.data_ptr(), n, None, None, None, None, None,
                         scratch.data_ptr(), scratch.numel(), 0, stream)
call(); torch.cuda.synchronize()
nmax = (sb - 128) // 16
tr = torch.zeros(nmax * 8, dtype=torch.int64, device=dev)
lib.drk_scan_set_trace(tr.data_ptr()); call(); torch.cuda.synchronize(); lib.drk_scan_set_trace(None)
t = tr.cpu().numpy().reshape(nmax, 8).astype(np.float64)
nt = int((t[:, 5] > 0).sum()); t = t[:nt]
t0 = t[:, 2].min()
dur = (t[:, 5].max() - t0) / 1e3
print(f"{dt} n=2^{log2n} tiles={nt} span {dur:.1f} us -> {2*n*x.element_size()/dur/1e3:.0f} GB/s")
lb = (t[:, 3] - t[:, 2]) / 1e3
rs = (t[:, 5] - t[:, 3]) / 1e3
print(f"  lookback  mean {lb.mean():.3f} p50 {np.percentile(lb,50):.3f} p90 {np.percentile(lb,90):.3f} us; rounds mean {t[:,6].mean():.2f} max {t[:,6].max():.0f}")
print(f"  rescan    mean {rs.mean():.3f} p50 {np.percentile(rs,50):.3f} p90 {np.percentile(rs,90):.3f} us")
for G in (444, 296, 148):
    if nt > 2 * G:
        red = (t[G:, 2] - t[:-G, 5]) / 1e3
        if np.percentile(red, 10) > 0:
            print(f"  G={G}: reduce-next mean {red.mean():.3f} p50 {np.percentile(red,50):.3f} p90 {np.percentile(red,90):.3f} us")
