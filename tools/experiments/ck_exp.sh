cd paper_1903_04243_b200; cp libpfb.so libpfb_ck2.so; cd ..
for c in 2 4 8; do
  cp paper_1903_04243_b200/libpfb_ck$c.so paper_1903_04243_b200/libpfb.so
  echo "CHUNK_KB=$c"
  for s in "10240 784 256" "4096 4096 4096" "1024 256 512" "256 2048 1024"; do timeout 60 python tools/gemm_probe.py --graph --force 3 --shape $s --iters 10 2>&1 | tail -1; done
  timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "bias or accurate or error_scale" 2>&1 | tail -1
done
