"""Where C1's API time goes (dot fp32 2^24, 2 segments, one GPU): the full API call, the
cached plan's run() alone, the raw batched launch + stream sync through ctypes, and the
kernel's device time (CUDA events, queue kept full)."""
import ctypes, json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import _lib, algorithms as A, bench as B, kernels, plans, repro, views  # noqa: E402


def per_call(f, reps=1000):
    for _ in range(50):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    return round((time.perf_counter() - t0) / reps * 1e6, 2)


n = 1 << 24
rt = sr.Runtime(2, devices=[0])
x = sr.DistributedVector(rt, n, dtype=np.float32)
y = sr.DistributedVector(rt, n, dtype=np.float32)
repro.fill_unit(x, 1, 0)
repro.fill_unit(y, 1, n)
st = rt.device_states[0]
out = {"api_us": per_call(lambda: B.dot_product(x, y))}
z = views.transform(views.zip(x, y), lambda t: t[0] * t[1])
key, dvs, plan = plans.lookup("reduce", z, A._op_key(A.add))
plan = plan or A._ReducePlan(rt, A._pieces(z), A.add)
out["plan_run_us"] = per_call(plan.run)
b = plan.batch
scratch = st.reduce_batch_scratch(b.m)
lib = _lib.load()
fn, sync = lib.drk_dot_batch, lib.drk_stream_synchronize
res = st.host_result_dev_ptr(0)


def raw():
    fn(b.code, b.m, b.xs, b.ys, b.ns, res, scratch.data_ptr(), st.index, st.handle)
    sync(st.index, st.handle)


out["raw_launch_sync_us"] = per_call(raw)
out["raw_launch_only_us"] = per_call(lambda: fn(b.code, b.m, b.xs, b.ys, b.ns, res, scratch.data_ptr(), st.index,
                                                st.handle), 200)
torch.cuda.synchronize()
with kernels.profile() as prof:
    with torch.cuda.stream(st.stream):
        torch.cuda._sleep(int(4e6))
    for _ in range(100):
        b.launch()
    st.synchronize()
t = sorted(s.elapsed_time(e) for s, e, _ in prof.records["drk_dot_batch"])
out["kernel_us"] = round(t[len(t) // 2] * 1e3, 2)
# the same kernel with its result in device memory instead of mapped pinned host memory
dres = st.result_dev_ptr(0)
torch.cuda.synchronize()
evs = []
with torch.cuda.stream(st.stream):
    torch.cuda._sleep(int(4e6))
for _ in range(100):
    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_.record(st.stream)
    fn(b.code, b.m, b.xs, b.ys, b.ns, dres, scratch.data_ptr(), st.index, st.handle)
    e_.record(st.stream)
    evs.append((s_, e_))
st.synchronize()
t = sorted(a.elapsed_time(c) for a, c in evs)
out["kernel_devres_us"] = round(t[len(t) // 2] * 1e3, 2)
for waves in (1, 2):
    lib.drk_tune(b"reduce_waves", waves)
    out[f"raw_launch_sync_w{waves}_us"] = per_call(raw)
print(json.dumps(out), flush=True)
