cp paper_1903_04243_b200/libpfb.so /tmp/libpfb_sw4.so
for w in 4 6 8; do
  if [ $w != 4 ]; then cp paper_1903_04243_b200/libpfb_sw$w.so paper_1903_04243_b200/libpfb.so; else cp /tmp/libpfb_sw4.so paper_1903_04243_b200/libpfb.so; fi
  echo "SPLIT_WARPS=$w"
  for s in "10240 784 256" "1024 2048 64 256" "2048 2048 256"; do timeout 60 python tools/gemm_probe.py --graph --force 6 --shape $s --iters 5 | tail -1; done
done
