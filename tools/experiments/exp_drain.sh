# per-k-block cost vs. the accumulator drain (PFB_TC_EXP bit 4: no drain) and chunk depth
for f in 8; do for e in 0 4 6; do for ch in 2 4 8; do
  echo "== force $f exp $e chunk $ch"
  PFB_TC_CHUNK=$ch PFB_TC_EXP=$e PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force $f --shape 256 2048 1024 --planes --graph 20 2>&1 | grep "deltas\|rep 2" | tail -2
  PFB_TC_CHUNK=$ch PFB_TC_EXP=$e timeout 60 python tools/gemm_probe.py --graph --planes --force $f --shape 256 2048 1024 --iters 20 2>&1 | tail -1
done; done; done
for ch in 2 4 8; do echo "== no planes force 8 chunk $ch"; PFB_TC_CHUNK=$ch timeout 60 python tools/gemm_probe.py --graph --force 8 --shape 256 2048 1024 --iters 20 2>&1 | tail -1; done
