python tools/pcie_probe.py --reps 3 | head -1
for r in 1 2; do python bench.py --workloads dot,triad,scan --steps 5 --warmup 3 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
