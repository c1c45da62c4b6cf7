export PFB_TC_TRACE=1
for s in "784 256 128" "1024 256 256" "256 2048 1024" "128 256 784"; do
  for f in 4 3; do echo "== force=$f $s"; timeout 60 python tools/tc_trace.py --force $f --shape $s 2>&1 | tail -2; done
done
echo "== ksplit 4"; PFB_TC_KSPLIT=4 timeout 60 python tools/tc_trace.py --force 4 --shape 784 256 128 | tail -2
