#!/bin/bash
mkdir -p gpurun_out/g9
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g9/gputests.log 2>&1; tail -5 gpurun_out/g9/gputests.log
timeout 600 python bench.py --workloads black_scholes,black_scholes_fast --log2n 28 --no-e2e --steps 20 > gpurun_out/g9/bench_c4.json 2>gpurun_out/g9/bench_c4.err; cat gpurun_out/g9/bench_c4.json
timeout 600 python bench.py --no-cpu > gpurun_out/g9/bench_n1.json 2>gpurun_out/g9/bench_n1.err; cat gpurun_out/g9/bench_n1.json
timeout 300 python tools/scan_sizes.py --sizes 24,25,26,27,28,30 --kinds f32,i32,f64 --queue 5 --reps 10 > gpurun_out/g9/scan_sizes.jsonl 2>&1
