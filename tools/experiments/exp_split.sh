for f in 4 8 7; do for e in 0 2 16 18; do
  echo "== force $f exp $e"
  PFB_TC_EXP=$e PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force $f --shape 256 2048 1024 --planes --graph 20 2>&1 | grep "deltas\|rep 2" | tail -2
  PFB_TC_EXP=$e timeout 60 python tools/gemm_probe.py --graph --planes --force $f --shape 256 2048 1024 --iters 20 2>&1 | tail -1
done; done
echo "== products=1 force 8"; PFB_TC_PRODUCTS=1 timeout 60 python tools/gemm_probe.py --graph --planes --force 8 --shape 256 2048 1024 --iters 20 2>&1 | tail -1
