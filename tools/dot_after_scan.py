"""Dot time right after a scan, with an idle gap of G us between them (GPU sleep), against the
dot right after a triad: is the slowdown a transient of the scan's end?"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, bench as B, kernels, repro, views  # noqa: E402

n = 1 << 30
rt = sr.Runtime(1)
st = rt.device_states[0]
a, b, c = (sr.DistributedVector(rt, n, dtype=np.float32) for _ in range(3))
repro.fill_unit(b, 1, 0)
repro.fill_unit(c, 1, n)
dot = lambda: A.reduce(views.transform(views.zip(b, c), lambda t: t[0] * t[1]), 0.0, A.add)
from paper_2406_00158_b200 import _lib  # noqa: E402
lib = _lib.load()
for kv in filter(None, (sys.argv[1] if len(sys.argv) > 1 else "").split(",")):
    k, v = kv.split("=")
    lib.drk_tune(k.encode(), int(v))
befores = (sys.argv[2] if len(sys.argv) > 2 else "scan,triad").split(",")
gaps = [int(g) for g in (sys.argv[3] if len(sys.argv) > 3 else "0,20,100,500").split(",")]
PRE = {"scan": lambda: A.inclusive_scan(c, a), "triad": lambda: B.stream_triad(a, b, c),
       "copy": lambda: A.copy(c, a), "reduce": lambda: A.reduce(c, 0.0), "dot": dot}
for before in befores:
    for gap_us in gaps:
        ts = []
        for rep in range(8):
            PRE[before]()
            if gap_us:
                with torch.cuda.stream(st.stream):
                    torch.cuda._sleep(int(gap_us * 1965))
            with kernels.profile() as prof:
                dot()
            rt.synchronize()
            if rep >= 2:
                ts += [s.elapsed_time(e) for recs in prof.records.values() for s, e, _ in recs]
        print(json.dumps({"tune": sys.argv[1] if len(sys.argv) > 1 else "", "before": before, "gap_us": gap_us, "dot_ms": round(float(np.median(ts)), 4)}), flush=True)
