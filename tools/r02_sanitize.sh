#!/bin/bash
mkdir -p gpurun_out/san
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize.py > gpurun_out/san/memcheck.log 2>&1; tail -3 gpurun_out/san/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize.py --small > gpurun_out/san/racecheck.log 2>&1; tail -3 gpurun_out/san/racecheck.log
timeout 1500 compute-sanitizer --tool synccheck python tools/sanitize.py --small > gpurun_out/san/synccheck.log 2>&1; tail -3 gpurun_out/san/synccheck.log
