python tools/bs_parity.py
python bench.py --workloads black_scholes,black_scholes_fast --log2n 28 --no-e2e --no-cpu --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:(v['avg_ms'],v['GB/s']) for k,v in d['workloads'].items()})"
