export PFB_TC_TRACE=1
for s in "784 256 128" "1024 256 256" "256 2048 1024"; do
  for f in 4 3; do echo "== force=$f $s"; timeout 60 python tools/tc_trace.py --force $f --shape $s 2>&1 | tail -1; done
done
unset PFB_TC_TRACE
for s in "1024 256 256" "256 2048 1024" "256 1024 2048" "128 256 784" "784 256 128" "10240 784 256" "4096 4096 4096" "1024 2048 64 256"; do
  for f in 4 3 6; do timeout 60 python tools/gemm_probe.py --graph --force $f --shape $s --iters 20 2>&1 | tail -1; done
done
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3
