for cfg in "scan_sub=1" "scan_sub=2" "scan_sub=3" "scan_sub=4" "scan_sub=1,scan_l2_min=4194304" "scan_sub=2,scan_l2_min=8388608"; do
  echo "== $cfg"; DRK_TUNE="$cfg" python tools/scan_sizes.py --sizes 18,19,20,21,22,23 --kinds f32,i32 --queue 5 --reps 20 2>&1 | grep log2n | python -c "
import json,sys
print(' '.join(f\"{d['log2n']}{d['kind'][0]}:{d['ms']*1e3:.1f}\" for d in map(json.loads, sys.stdin)))"
done
