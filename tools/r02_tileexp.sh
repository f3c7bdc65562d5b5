#!/bin/bash
# Tile-shape experiments of the fp32 L2 scan (drk_tune scan_exp): time by size + DRAM bytes at 2^30.
mkdir -p gpurun_out/tileexp
for cfg in "" "scan_exp=1" "scan_exp=1,scan_smem_pad=20480" "scan_exp=2" "scan_exp=3" "scan_exp=4" "scan_exp=4,scan_smem_pad=20480" "scan_l2_subs=8"; do
  tag=$(echo "x$cfg" | tr ',=' '__')
  DRK_TUNE="$cfg" timeout 300 python tools/scan_sizes.py --sizes 21,22,23,24,25,26,27,28,30 --kinds f32 --queue 5 --reps 10 > gpurun_out/tileexp/t_$tag.jsonl 2>&1
  DRK_TUNE="$cfg" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:scan -c 2 --csv python tools/scan_once.py 30 > gpurun_out/tileexp/n_$tag.csv 2>&1
  echo "== $cfg"; python - "$tag" <<'PY'
import json,sys
tag=sys.argv[1]
rows=[json.loads(l) for l in open(f"gpurun_out/tileexp/t_{tag}.jsonl") if l.startswith('{"log2n')]
print(" ".join(f"{r['log2n']}:{r['ms']*1e3:.1f}us/{r['frac']}" for r in rows))
PY
  grep -E '"(dram__bytes_read|gpu__time)' gpurun_out/tileexp/n_$tag.csv | awk -F'","' '{printf "%s ", $NF}'; echo
done
