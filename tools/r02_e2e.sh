#!/bin/bash
# e2e transfer chunking experiment: PCIe probe, then the bench e2e leg with whole and chunked copies.
python tools/pcie_probe.py --reps 3
for c in 0 256 64; do
  DRK_TUNE=memcpy_chunk_mb=$c python bench.py --workloads dot,triad,scan --steps 5 --warmup 3 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunk', $c, d['e2e'])"
done
