"""Batched reduce / dot kernel time by size and grid waves (drk_tune reduce_waves), CUDA events
with the GPU queue kept full: how close the reduce gets to the read roofline at mid sizes."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import _lib, algorithms as A, kernels, repro, views  # noqa: E402

lib = _lib.load()
rt = sr.Runtime(1)
st = rt.device_states[0]
peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "MEASURED_PEAKS.json")))["hbm_gbs"])
for lg in (22, 24, 26, 28, 30):
    n = 1 << lg
    x = sr.DistributedVector(rt, n, dtype=np.float32)
    repro.fill_unit(x, 1, 0)
    plan = A._ReducePlan(rt, A._pieces(x), A.add)
    row = {"log2n": lg}
    for w in (1, 2, 4, 8):
        lib.drk_tune(b"reduce_waves", w)
        for _ in range(3):
            plan.batch.launch()
        st.synchronize()
        with kernels.profile() as prof:
            with torch.cuda.stream(st.stream):
                torch.cuda._sleep(int(3e6))
            for _ in range(20):
                plan.batch.launch()
            st.synchronize()
        t = sorted(s.elapsed_time(e) for recs in prof.records.values() for s, e, _ in recs)
        ms = t[len(t) // 2]
        row[f"w{w}"] = (round(ms * 1e3, 1), round(4 * n / (ms * 1e-3) / 1e9 / peak, 3))
    lib.drk_tune(b"reduce_waves", 1)
    print(json.dumps(row), flush=True)
    del x
