for s in "1024 256 256" "256 2048 1024" "256 1024 2048" "128 256 784" "784 256 128"; do
  for k in 1 4; do
    for f in 4 3; do
      r=$(PFB_TC_KSPLIT=$k timeout 60 python tools/gemm_probe.py --graph --force $f --shape $s --iters 20 2>&1 | tail -1)
      echo "ksplit=$k $r"
    done
  done
done
for s in "1024 256 256" "128 256 784" "10240 784 256" "1024 2048 64 256"; do timeout 60 python tools/gemm_probe.py --graph --force 1 --shape $s --iters 20 2>&1 | tail -1; done
