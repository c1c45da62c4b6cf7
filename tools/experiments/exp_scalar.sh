# cfg4 step with the fused programs at one element per thread (PFB_FUSED_SCALAR=1)
for sc in 0 1; do
  PFB_FUSED_SCALAR=$sc timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('scalar', $sc, d['ms_per_step'], d['roofline']['kinds_eager_ms'])"
done
PFB_FUSED_SCALAR=1 bash tools/launch_list.sh cfg4 2>&1 | tail -8
