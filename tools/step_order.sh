#!/bin/bash
# Per-kernel time by what runs before it: the two cyclic orders of the bench step and each
# workload alone (bench.py lines without e2e / CPU legs).
mkdir -p gpurun_out/order
B="python bench.py --no-e2e --no-cpu --steps 20"
for w in dot,triad,scan dot,scan,triad dot triad scan; do
  $B --workloads $w > gpurun_out/order/$w.json 2>&1
  tail -1 gpurun_out/order/$w.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], {k:(v['avg_ms'],v['frac']) for k,v in d['workloads'].items()})"
done
