#!/bin/bash
# Round-2 final pass on the last build: GPU tests, smoke, bench N=1 (both arms), the bench launch
# list and one ncu --set full capture of the scan (the kernel furthest below its roofline).
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final/gputests.txt 2>&1
echo "PYTEST_RC=$?" >> gpurun_out/final/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/final/smoke.txt 2>&1
timeout 400 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err
timeout 400 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/final/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_l2 --launch-skip 2 -c 1 \
  -o gpurun_out/final/scan30 python tools/scan_once.py 30 > gpurun_out/final/scan30.log 2>&1
ls -la gpurun_out/final; tail -3 gpurun_out/final/gputests.txt
