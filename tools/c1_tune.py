"""C1 (dot fp32, n = 2^24, 2 segments on one GPU): API time per call and the batched dot
kernel's device time with the GPU queue kept full (so CUDA events bracket kernel time, not
host launch gaps), for reduce-grid wave counts (drk_tune reduce_waves)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import _lib, bench as B, kernels, repro  # noqa: E402

n = 1 << 24
rt = sr.Runtime(2, devices=[0])
x = sr.DistributedVector(rt, n, dtype=np.float32)
y = sr.DistributedVector(rt, n, dtype=np.float32)
repro.fill_unit(x, 1, 0)
repro.fill_unit(y, 1, n)
st = rt.device_states[0]
lib = _lib.load()
for waves in [int(w) for w in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4").split(",")]:
    lib.drk_tune(b"reduce_waves", waves)
    for _ in range(50):
        B.dot_product(x, y)
    torch.cuda.synchronize()
    reps = 500
    t0 = time.perf_counter()
    for _ in range(reps):
        B.dot_product(x, y)
    api = (time.perf_counter() - t0) / reps * 1e6
    # device time: enqueue the batched kernel alone, back to back behind a sleep
    from paper_2406_00158_b200 import algorithms as A, views
    plan = A._ReducePlan(rt, A._pieces(views.transform(views.zip(x, y), lambda t: t[0] * t[1])), A.add)
    with kernels.profile() as prof:
        with torch.cuda.stream(st.stream):
            torch.cuda._sleep(int(4e6))
        for _ in range(100):
            plan.batch.launch()
        st.synchronize()
    times = sorted(s.elapsed_time(e) for s, e, _ in prof.records["drk_dot_batch"])
    kus = times[len(times) // 2] * 1e3
    print(json.dumps({"reduce_waves": waves, "api_us": round(api, 1), "kernel_us": round(kus, 2),
                      "kernel_GB/s": round(8 * n / (kus * 1e-6) / 1e9, 1)}), flush=True)
