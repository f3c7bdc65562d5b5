"""Batched reduce/dot kernel time (CUDA events, GPU queue kept full) against the grid cap
(drk_tune reduce_grid) at small n: where the fixed cost of the last-CTA fold sits."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import _lib, algorithms as A, kernels, repro, views  # noqa: E402

lib = _lib.load()
rt = sr.Runtime(1)
st = rt.device_states[0]
for lg in (20, 22, 24):
    n = 1 << lg
    x = sr.DistributedVector(rt, n, dtype=np.float32)
    y = sr.DistributedVector(rt, n, dtype=np.float32)
    repro.fill_unit(x, 1, 0)
    repro.fill_unit(y, 1, n)
    for kind in ("reduce", "dot"):
        r = x if kind == "reduce" else views.transform(views.zip(x, y), lambda t: t[0] * t[1])
        plan = A._ReducePlan(rt, A._pieces(r), A.add)
        row = {"log2n": lg, "kind": kind}
        for g in (148, 296, 444, 592, 888, 0):
            lib.drk_tune(b"reduce_grid", g)
            for _ in range(5):
                plan.batch.launch()
            st.synchronize()
            with kernels.profile() as prof:
                with torch.cuda.stream(st.stream):
                    torch.cuda._sleep(int(2e6))
                for _ in range(40):
                    plan.batch.launch()
                st.synchronize()
            t = sorted(s.elapsed_time(e) for recs in prof.records.values() for s, e, _ in recs)
            row[f"g{g or 'auto'}"] = round(t[len(t) // 2] * 1e3, 2)
        lib.drk_tune(b"reduce_grid", 0)
        print(json.dumps(row), flush=True)
