#!/bin/bash
# keep_tail scan experiment: parity under the knob, then time by size and DRAM bytes at 2^30.
mkdir -p gpurun_out/keep
DRK_TUNE=scan_keep_tail=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_gpu.py tests/test_config_parity_gpu.py tests/test_fused_scan_gpu.py -x -q -p no:cacheprovider -k "scan or Scan" > gpurun_out/keep/tests.log 2>&1; tail -3 gpurun_out/keep/tests.log
for cfg in "" "scan_keep_tail=1" "scan_keep_tail=1,scan_l2_subs=8" "scan_keep_tail=1,scan_stagger=0"; do
  tag=$(echo "x$cfg" | tr ',=' '__')
  DRK_TUNE="$cfg" timeout 300 python tools/scan_sizes.py --sizes 22,23,24,25,26,27,28,30 --kinds f32,i32,f64 --queue 5 --reps 10 > gpurun_out/keep/t_$tag.jsonl 2>&1
  DRK_TUNE="$cfg" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:scan -c 2 --csv python tools/scan_once.py 30 > gpurun_out/keep/n_$tag.csv 2>&1
  echo "== $cfg"; python - "$tag" <<'PY'
import json,sys
tag=sys.argv[1]
rows=[json.loads(l) for l in open(f"gpurun_out/keep/t_{tag}.jsonl") if l.startswith('{"log2n')]
for k in ("f32","i32","f64"):
    print(k, " ".join(f"{r['log2n']}:{r['ms']*1e3:.1f}/{r['frac']}" for r in rows if r['kind']==k))
PY
  grep -E '"(dram__bytes_read|gpu__time)' gpurun_out/keep/n_$tag.csv | awk -F'","' '{printf "%s ", $NF}'; echo
done
