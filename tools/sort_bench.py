"""Radix sort (drk_sort_keys / drk_sort_pairs) time by size and dtype on one GPU, device time
from CUDA events around each call (keys re-filled between reps), plus a numpy check."""
import ctypes, json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_00158_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream().cuda_stream
for name, tdt, code in (("uint64", torch.int64, 5), ("float32", torch.float32, 0), ("int32", torch.int32, 2)):
    for lg in (20, 24, 27):
        n = 1 << lg
        g = torch.Generator(device=dev).manual_seed(1)
        if name == "float32":
            src = torch.randn(n, device=dev, generator=g)
        else:
            src = torch.randint(-2**31 if name == "int32" else 0, 2**31 - 1, (n,), device=dev, generator=g,
                                dtype=tdt)
        keys = src.clone()
        alt = torch.empty_like(keys)
        need = ctypes.c_size_t(0)
        _lib.call("drk_sort_keys", code, keys.data_ptr(), alt.data_ptr(), n, None, ctypes.byref(need), 0, stream)
        scratch = torch.empty(need.value, dtype=torch.uint8, device=dev)
        times = []
        for r in range(6):
            keys.copy_(src)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            _lib.call("drk_sort_keys", code, keys.data_ptr(), alt.data_ptr(), n, scratch.data_ptr(),
                      ctypes.byref(need), 0, stream)
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
        ms = sorted(times[1:])[len(times[1:]) // 2]
        ok = None
        if lg <= 24:
            got = keys.cpu().numpy()
            want = np.sort(src.cpu().numpy().view(np.uint64) if name == "uint64" else src.cpu().numpy())
            ok = bool(np.array_equal(got.view(np.uint64) if name == "uint64" else got, want))
        print(json.dumps({"dtype": name, "log2n": lg, "ms": round(ms, 3), "Gkeys/s": round(n / ms / 1e6, 2),
                          "ok": ok}), flush=True)
