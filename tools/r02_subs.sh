for cfg in "" "scan_l2_subs=4" "scan_l2_subs=8"; do
  echo "== $cfg"; DRK_TUNE="$cfg" python tools/scan_sizes.py --sizes 23,24,25,26,27 --kinds f32,i32 --queue 5 --reps 10 2>&1 | grep log2n | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['log2n'], d['kind'], d['ms'], d['frac'])" | paste - - - - - - - - - -
done
