for cfg in "PFB_PARTS_BN=128" "PFB_PARTS_BN=256" "PFB_PARTS_BN=128 PFB_PARTS_SMAX=8" "PFB_PARTS_BN=128 PFB_PARTS_SMAX=4" "PFB_NO_PARTS=1"; do
  echo "$cfg: $(env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["gpu_launches"])')"
done
