"""Where the e2e step's time goes: bench.py's e2e loop (upload b,c -> dot, triad, scan ->
download a,o) with CUDA events around every transfer and kernel phase, printed per step
as start/end offsets (ms) on each stream.

    python tools/e2e_timeline.py [--log2n 30] [--steps 4]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, bench as B, views  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=30)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--no-dot", action="store_true")
    a = ap.parse_args()
    n = 1 << a.log2n
    dt = np.float32
    rt = sr.Runtime(1)
    st = rt.device_states[0]
    hb, hc = sr.pinned_empty(n, dt), sr.pinned_empty(n, dt)
    ha, ho = sr.pinned_empty(n, dt), sr.pinned_empty(n, dt)
    hb[...] = 1.0
    hc[...] = 2.0
    sets = [tuple(sr.DistributedVector(rt, n, dtype=dt) for _ in range(4)) for _ in range(2)]
    h2d, d2h = st.copy_stream("h2d"), st.copy_stream("d2h")
    marks = []

    def mark(name, stream):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        marks.append((name, ev))

    tickets = []

    def step(i):
        av, bv, cv, ov = sets[i % 2]
        tickets.append(bv.upload(hb, wait=False))
        tickets.append(cv.upload(hc, wait=False))
        mark(f"{i}:h2d_end", h2d)
        if not a.no_dot:
            z = views.transform(views.zip(bv, cv), lambda t: t[0] * t[1])
            A.reduce(z, 0.0, A.add)
            mark(f"{i}:dot_end", st.stream)
        B.stream_triad(av, bv, cv)
        tickets.append(av.to_numpy(out=ha, wait=False)[1])
        A.inclusive_scan(cv, ov)
        mark(f"{i}:scan_end", st.stream)
        tickets.append(ov.to_numpy(out=ho, wait=False)[1])
        mark(f"{i}:d2h_end", d2h)

    step(0)
    for tk in tickets:
        tk.wait()
    tickets.clear()
    torch.cuda.synchronize()
    marks.clear()
    mark("t0", st.stream)
    t0 = time.perf_counter()
    for i in range(1, a.steps + 1):
        step(i)
    for tk in tickets:
        tk.wait()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.steps
    base = marks[0][1]
    out = {name: round(base.elapsed_time(ev), 2) for name, ev in marks[1:]}
    print(json.dumps({"wall_ms_per_step": round(wall * 1e3, 2), "marks_ms": out}))


if __name__ == "__main__":
    main()
