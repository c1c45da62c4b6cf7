#!/bin/bash
# One GPU pass: the GPU suite (or $TESTS), bench lines for $CONFIGS (our arm,
# no CPU leg), launch lists for $LL.  Outputs under gpurun_out/$TAG/.
TAG=${TAG:-quick}; OUT=gpurun_out/$TAG; mkdir -p $OUT
TESTS=${TESTS:-tests}
if [ "$TESTS" != "none" ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
fi
for c in ${CONFIGS:-cfg4}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-sweep --steps 10 > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err
  python - $OUT/bench_$c.jsonl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print(d["config"]["workload"], f"value={d['value']:.4g} {d['unit']} ms/step={d['ms_per_step']:.4f} e2e={d['e2e']['value']:.4g} launches={d['gpu_launches']}",
          f"roof={r.get('kernel')} frac={r.get('frac', 0):.3f} share={r.get('share_of_step', 0):.2f}")
except Exception as e:
    print("bench failed", sys.argv[1], e)
PY
  tail -2 $OUT/bench_$c.err
done
for c in ${LL:-}; do
  bash tools/launch_list.sh $c > $OUT/ll_$c.txt 2>&1; head -30 $OUT/ll_$c.txt
done
