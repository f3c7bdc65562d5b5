#!/bin/bash
# Round-2 ncu captures (one launch each, --set full): scan 2^30 fp32 (keep_tail), Black-Scholes both
# precisions at 2^26, the radix sort passes at 2^24, the C1 batched dot; plus the bench launch list.
mkdir -p gpurun_out/ncu2
N="ncu --set full --clock-control none --import-source on"
$N -k regex:scan_l2 --launch-skip 2 -c 1 -o gpurun_out/ncu2/scan30 python tools/scan_once.py 30 > gpurun_out/ncu2/scan30.log 2>&1
$N -k regex:map_vec --launch-skip 5 -c 1 -o gpurun_out/ncu2/bsref python tools/bs_once.py > gpurun_out/ncu2/bsref.log 2>&1
$N -k regex:radix --launch-skip 8 -c 2 -o gpurun_out/ncu2/radix python tools/sort_once.py 24 > gpurun_out/ncu2/radix.log 2>&1
$N -k regex:reduce_batch --launch-skip 2 -c 1 -o gpurun_out/ncu2/c1dot python tools/c1_once.py > gpurun_out/ncu2/c1dot.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu2/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu2/bench.log 2>&1
ls -la gpurun_out/ncu2
