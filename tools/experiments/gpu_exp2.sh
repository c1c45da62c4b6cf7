timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for s in "4096 4096 4096" "10240 784 256" "1024 2048 64 256" "256 2048 1024" "256 1024 2048" "1024 256 256" "784 256 128" "128 256 784"; do
  for f in 4 3; do timeout 60 python tools/gemm_probe.py --graph --force $f --shape $s --iters 10 2>&1 | tail -1; done
done
for c in cfg2_mlp cfg1_batch cfg1_full cfg4 cfg5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],4), 'ms', 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3) if d.get('roofline') else None)"; done
