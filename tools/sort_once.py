"""One drk_sort_keys of 2^24 int32 keys after a warm-up (a short command for ncu)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_00158_b200 import _lib  # noqa: E402

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 24)
kind = sys.argv[2] if len(sys.argv) > 2 else "int32"
dev = torch.device("cuda", 0)
if kind == "float32":
    src = torch.randn(n, device=dev)
else:
    src = torch.randint(-2**31, 2**31 - 1, (n,), device=dev, dtype=torch.int32)
code = 0 if kind == "float32" else 2
keys, alt = src.clone(), torch.empty_like(src)
need = ctypes.c_size_t(0)
s = torch.cuda.current_stream().cuda_stream
_lib.call("drk_sort_keys", code, keys.data_ptr(), alt.data_ptr(), n, None, ctypes.byref(need), 0, s)
scratch = torch.empty(need.value, dtype=torch.uint8, device=dev)
for _ in range(2):
    keys.copy_(src)
    _lib.call("drk_sort_keys", code, keys.data_ptr(), alt.data_ptr(), n, scratch.data_ptr(), ctypes.byref(need), 0, s)
torch.cuda.synchronize()
