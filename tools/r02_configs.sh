#!/bin/bash
# Round-2 bench lines for the BASELINE configs on one GPU (C1 dot 2^24 x 2 segments, C2 STREAM,
# C3 scan 8 x 2^27 segments and one 2^30 segment, C3 fused-view scans, C4 both precisions).
mkdir -p gpurun_out/cfg
B="python bench.py --no-e2e --no-cpu --steps 20"
$B --workloads dot --log2n 24 --segments 2 > gpurun_out/cfg/c1.json 2>&1
$B --workloads copy,scale,add,triad > gpurun_out/cfg/c2.json 2>&1
$B --workloads scan --segments 8 > gpurun_out/cfg/c3_8seg.json 2>&1
$B --workloads scan,scan_affine,scan_product > gpurun_out/cfg/c3_views.json 2>&1
$B --workloads black_scholes,black_scholes_fast --log2n 28 > gpurun_out/cfg/c4.json 2>&1
for f in gpurun_out/cfg/*.json; do echo "== $f"; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['workload'], {k:(v['kernel'],v['avg_ms'],v['GB/s'],v['frac']) for k,v in d['workloads'].items()})"; done
