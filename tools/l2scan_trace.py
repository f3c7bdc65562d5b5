"""Per-CTA phases of the L2 two-touch scan (debug trace in libdrk):
stamp 0 ticket, 1 reduce done, 2 aggregate published + TMA issued, 3 prefix resolved, 5 end."""
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
x = (torch.rand(n, device=dev) * 10).to(getattr(torch, dt)); y = torch.empty_like(x)
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
t0 = t[:, 0].min()
T = (t - t0) / 1e3
T[:, 6] = t[:, 6]
span = T[:, 5].max()
print(f"{dt} n=2^{log2n} tiles={nt} span {span:.1f} us -> {2*n*x.element_size()/span/1e3:.0f} GB/s")
for nm, a, b in (("reduce", 0, 1), ("publish+TMA", 1, 2), ("lookback", 2, 3), ("rescan", 3, 5), ("life", 0, 5)):
    d = T[:, b] - T[:, a]
    print(f"  {nm:12s} mean {d.mean():7.3f} p50 {np.percentile(d,50):7.3f} p90 {np.percentile(d,90):7.3f} p99 {np.percentile(d,99):7.3f} us")
print(f"  lookback rounds mean {T[:,6].mean():.2f} max {T[:,6].max():.0f}")
for frac in (0.25, 0.5, 0.75):
    m = span * frac
    alive = ((T[:, 0] <= m) & (T[:, 5] >= m)).sum()
    inred = ((T[:, 0] <= m) & (T[:, 1] >= m)).sum()
    inlb = ((T[:, 2] <= m) & (T[:, 3] >= m)).sum()
    inres = ((T[:, 3] <= m) & (T[:, 5] >= m)).sum()
    print(f"  at {frac:.2f}: alive {alive} ({alive/148:.2f}/SM) reduce {inred} lookback {inlb} rescan {inres}")
# gaps: time between a CTA slot freeing and the next ticket start (approx via start-time density)
st = np.sort(T[:, 0])
print(f"  start rate {nt/span:.1f} tiles/us; first/last start {st[0]:.1f}/{st[-1]:.1f} us; tail {span-st[-1]:.1f} us")
