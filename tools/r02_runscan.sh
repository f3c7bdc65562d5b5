timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_config_parity_gpu.py tests/test_fused_scan_gpu.py tests/test_large_gpu.py -x -q -p no:cacheprovider -k "scan or Scan" 2>&1 | tail -1
python tools/scan_sizes.py --sizes 22,24,26,27,28,30 --kinds f32,i32,f64 --queue 5 --reps 10 | grep log2n | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['log2n'], d['kind'], d['ms'], d['frac'])" | paste - - -
