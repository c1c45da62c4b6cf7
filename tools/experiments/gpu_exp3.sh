timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "concat or cfg4" 2>&1 | tail -1
for c in cfg4 cfg5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],4), 'ms', 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3) if d.get('roofline') else None)"; done
timeout 300 python tools/launch_breakdown.py --config cfg4 --top 5 2>&1 | head -12
