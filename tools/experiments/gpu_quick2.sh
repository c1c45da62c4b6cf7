timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for s in "128 256 784" "784 256 128" "128 10 256" "256 10 128" "1024 256 256" "32 256 784" "320 784 256"; do timeout 60 python tools/gemm_probe.py --graph --force 1 --shape $s --iters 20 2>&1 | tail -1; done
timeout 300 python bench.py --config cfg2_mlp --steps 20 --warmup 5 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | cut -c1-760
bash tools/launch_list.sh cfg2_mlp | tail -16
