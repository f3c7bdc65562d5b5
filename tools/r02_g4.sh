mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_reduce_combine_gpu.py -x -q -p no:cacheprovider > gpurun_out/combine_tests.log 2>&1; tail -15 gpurun_out/combine_tests.log
timeout 300 python tools/combine_bench.py > gpurun_out/combine_bench.jsonl 2>&1; cat gpurun_out/combine_bench.jsonl
for lg in 22 24 26 28 30; do timeout 120 python tools/scan_trace.py $lg float32; done > gpurun_out/scan_trace.txt 2>&1; cat gpurun_out/scan_trace.txt
