import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2406_00158_b200 import _lib
for dt, code in ((np.float32, 0), (np.float64, 1)):
    x = np.array([3.0, np.nan, -1.0, -np.nan, 0.0, -0.0, np.inf, -np.inf, 1e-38, 5e-324], dtype=dt)
    x = np.tile(x, 3)
    k = torch.from_numpy(x.copy()).cuda(); alt = torch.empty_like(k)
    need = ctypes.c_size_t(0); s = torch.cuda.current_stream().cuda_stream
    _lib.call("drk_sort_keys", code, k.data_ptr(), alt.data_ptr(), len(x), None, ctypes.byref(need), 0, s)
    sc = torch.zeros(need.value, dtype=torch.uint8, device="cuda")
    _lib.call("drk_sort_keys", code, k.data_ptr(), alt.data_ptr(), len(x), sc.data_ptr(), ctypes.byref(need), 0, s)
    torch.cuda.synchronize()
    print(dt.__name__, k.cpu().numpy())
