#!/bin/bash
# post-profile validation: the GPU suite, smoke, and bench lines + launch lists
# of the configs changed after tools/final_round.sh ran ($CONFIGS)
OUT=gpurun_out/val; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
: > $OUT/bench_lines.jsonl
for c in ${CONFIGS:-cfg2_mlp cfg2_conv}; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 3 2> $OUT/bench_$c.err | tail -1 >> $OUT/bench_lines.jsonl
  bash tools/launch_list.sh $c > /dev/null 2>&1
  python tools/summarize_launches.py gpurun_out/ll_$c.csv > $OUT/launches_$c.txt 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/val/bench_lines.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], round(d["value"]), d["unit"], round(d["ms_per_step"] * 1000, 1), "us", d["gpu_launches"], "launches")
PY
