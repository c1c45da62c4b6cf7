timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/e2e_profile.py --config cfg2_mlp --n 200 2>&1 | head -4
timeout 300 python bench.py --config cfg2_mlp --steps 20 --warmup 5 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | cut -c1-700
