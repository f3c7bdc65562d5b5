#!/bin/bash
# Round-2 measurement pass: scan size sweep, host overhead per call, C1 tuning, scan ncu at 2^24 and 2^30.
mkdir -p gpurun_out
timeout 900 python tools/scan_sizes.py --sizes 20,21,22,23,24,25,26,27,28,30 --kinds f32,i32,f64,affine_f32,copy_f32 --queue 5 > gpurun_out/scan_sizes.jsonl 2>&1
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.json 2>&1
timeout 300 python tools/c1_tune.py 1,2,3,4 > gpurun_out/c1_tune.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan -c 2 -o gpurun_out/scan24 python tools/scan_once.py 24 > gpurun_out/ncu24.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan -c 2 -o gpurun_out/scan30 python tools/scan_once.py 30 > gpurun_out/ncu30.log 2>&1
cat gpurun_out/scan_sizes.jsonl gpurun_out/host_overhead.json gpurun_out/c1_tune.jsonl
