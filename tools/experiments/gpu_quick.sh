timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/e2e_profile.py --config cfg2_mlp --n 200 2>&1 | head -4
timeout 300 python bench.py --config cfg2_mlp --steps 20 --warmup 5 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | cut -c1-760
bash tools/launch_list.sh cfg2_mlp | tail -22
timeout 300 ncu --set full --clock-control none -k regex:fused_kernel -s 12 -c 3 -o gpurun_out/fused6 python bench.py --config cfg2_mlp --steps 1 --warmup 3 --no-cpu-baseline --no-sweep --minimal > /dev/null 2>&1
