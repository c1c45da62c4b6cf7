timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --config cfg2_mlp --steps 20 --warmup 5 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | cut -c1-700
bash tools/launch_list.sh cfg2_mlp | tail -16
timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | cut -c1-400
timeout 300 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | cut -c1-400
