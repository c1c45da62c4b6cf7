#!/bin/bash
# F16 tests again (row kernel launch bounds) + partials split-count sweep on cfg5 / cfg4
OUT=gpurun_out/r02y; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parts.py -m gpu -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for smax in 2 4 8; do
  for c in cfg5 cfg4; do
    PFB_PARTS_SMAX=$smax timeout 300 python bench.py --config $c --no-cpu-baseline --no-sweep --minimal --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('smax=$smax', d['config']['workload'], round(d['ms_per_step'],4))"
  done
done
PFB_PARTS_BN=256 timeout 300 python bench.py --config cfg5 --no-cpu-baseline --no-sweep --minimal --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bn256', d['config']['workload'], round(d['ms_per_step'],4))"
