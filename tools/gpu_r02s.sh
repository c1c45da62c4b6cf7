#!/bin/bash
# Session re-entry check: GPU suite, default bench line, every config (our arm), cfg4 launch list
OUT=gpurun_out/r02s; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 300 python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err; tail -c 600 $OUT/bench_default.jsonl
: > $OUT/bench_lines.jsonl
for c in cfg2_mlp cfg1_batch cfg1_full cfg2_conv cfg3 cfg5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2> $OUT/bench_$c.err | tail -1 >> $OUT/bench_lines.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/r02s/bench_lines.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    r=d.get("roofline",{})
    print(d["config"]["workload"], round(d["value"],1), d["unit"], "ms/step", round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"],1), "launches", d.get("gpu_launches"), "dom", r.get("kernel"), round(r.get("frac",0),3))
PY
bash tools/launch_list.sh cfg4 > $OUT/ll_cfg4.txt 2>&1; tail -30 $OUT/ll_cfg4.txt
