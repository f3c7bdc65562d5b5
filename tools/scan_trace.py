"""Per-tile timeline of the decoupled look-back scan (debug trace in libdrk)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_00158_b200 import _lib

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
dt = sys.argv[2] if len(sys.argv) > 2 else "float32"
n = 1 << log2n
lib = _lib.load()
for kv in (sys.argv[3].split(",") if len(sys.argv) > 3 else []):
    k, v = kv.split("=")
    lib.drk_tune(k.encode(), int(v))
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
ntiles = (sb - 128) // 16  # upper bound (SUB=1 tiles); unused rows stay 0

tr = torch.zeros(ntiles * 8, dtype=torch.int64, device=dev)
lib.drk_scan_set_trace(tr.data_ptr())
call(); torch.cuda.synchronize()
lib.drk_scan_set_trace(None)
t = tr.cpu().numpy().reshape(ntiles, 8).astype(np.float64)
t = t[t[:, 5] > 0]
ntiles = len(t)
t0 = t[:, 0].min()
T = t[:, :6] - t0
dur = (T[:, 5].max()) / 1e3
print(f"{dt} n=2^{log2n} tiles={ntiles} total {dur:.1f} us  -> {2*n*x.element_size()/dur/1e3:.0f} GB/s")
names = ["load", "local scan+publish", "lookback", "outputs", "store+exit"]
for k, nm in enumerate(names):
    d = (T[:, k + 1] - T[:, k]) / 1e3
    print(f"  {nm:20s} mean {d.mean():7.3f}  p50 {np.percentile(d,50):7.3f}  p90 {np.percentile(d,90):7.3f}  p99 {np.percentile(d,99):7.3f} us")
life = (T[:, 5] - T[:, 0]) / 1e3
print(f"  {'lifetime':20s} mean {life.mean():7.3f}  p50 {np.percentile(life,50):7.3f}  p90 {np.percentile(life,90):7.3f}")
r = t[:, 6]
print("  lookback rounds: mean %.2f max %d" % (r.mean(), r.max()))
# concurrency: tiles alive at the middle of the run
mid = T[:, 5].max() / 2
alive = ((T[:, 0] <= mid) & (T[:, 5] >= mid)).sum()
print(f"  tiles alive at midpoint: {alive}  (per SM {alive/148:.1f})")
# how late is the predecessor's aggregate relative to my data-ready?
pub = T[:, 2]
lag = (pub[:-1] - T[1:, 1]) / 1e3
print(f"  pred agg published minus my data-ready: p50 {np.percentile(lag,50):.3f} p90 {np.percentile(lag,90):.3f} us")
inc = T[:, 3]
lag2 = (inc[:-1] - T[1:, 2]) / 1e3
print(f"  pred INC published minus my agg: p50 {np.percentile(lag2,50):.3f} p90 {np.percentile(lag2,90):.3f} us")
# start order vs tile order
st = T[:, 0]
print(f"  ticket start spread per 1000 tiles: {np.median(np.diff(st[::1000]))/1e3:.3f} us")
