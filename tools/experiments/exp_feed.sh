# is the per-step GEMM's k-loop bound by the TMA feed?  PFB_TC_EXP=1: no TMA after the first ring fill
for e in 0 1 3; do
  echo "== force 8 exp $e"
  PFB_TC_EXP=$e PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force 8 --shape 256 2048 1024 --planes --graph 20 2>&1 | grep "deltas\|rep 2" | tail -2
  PFB_TC_EXP=$e timeout 60 python tools/gemm_probe.py --graph --planes --force 8 --shape 256 2048 1024 --iters 20 2>&1 | tail -1
done
for e in 0 1; do
  echo "== force 4 4096^3 exp $e"
  PFB_TC_EXP=$e timeout 60 python tools/gemm_probe.py --graph --planes --force 4 --shape 4096 4096 4096 --iters 5 2>&1 | tail -1
done
