for cfg in "scan_stagger=-1" "scan_stagger=0" "scan_stagger=20" "scan_stagger=60" "scan_stagger=90"; do
  echo "== $cfg"; DRK_TUNE="$cfg" python tools/scan_sizes.py --sizes 25,26,27,28 --kinds f32,i32 --queue 5 --reps 10 2>&1 | grep log2n | python -c "
import json,sys
print(' '.join(f\"{d['log2n']}{d['kind'][0]}:{d['ms']*1e3:.1f}/{d['frac']}\" for d in map(json.loads, sys.stdin)))"
done
