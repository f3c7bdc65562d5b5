#!/bin/bash
# Small-n scan overhead: ncu full of the 2^20 / 2^22 scans and the 2^22 copy, and a trace at 2^20.
mkdir -p gpurun_out/small
timeout 300 ncu --set full --clock-control none --import-source on -k regex:scan -c 1 -o gpurun_out/small/scan20 python tools/scan_once.py 20 > gpurun_out/small/n20.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:scan -c 1 -o gpurun_out/small/scan22 python tools/scan_once.py 22 > gpurun_out/small/n22.log 2>&1
timeout 300 ncu --section SpeedOfLight --section LaunchStats --clock-control none -k regex:map -c 1 -o gpurun_out/small/copy22 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A
rt=sr.Runtime(1); x=sr.DistributedVector(rt,1<<22,dtype=np.float32); y=sr.DistributedVector(rt,1<<22,dtype=np.float32)
for _ in range(3): A.copy(x,y)
rt.synchronize()" > gpurun_out/small/c22.log 2>&1
timeout 120 python tools/scan_trace.py 20 float32 > gpurun_out/small/trace20.txt 2>&1
cat gpurun_out/small/trace20.txt
