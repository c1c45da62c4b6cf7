# per-launch durations (warm caches) of one config: gpurun_out/ll_<cfg>.txt
c=${1:-cfg2_mlp}
mkdir -p gpurun_out
# GEMM autotune choices from an unprofiled run (timings under ncu are meaningless)
export PFB_GEMM_TUNE_FILE=gpurun_out/tune_ll_$c.txt
rm -f $PFB_GEMM_TUNE_FILE
timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sweep --minimal > /dev/null 2>&1
cat $PFB_GEMM_TUNE_FILE
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/ll_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-sweep --minimal > /dev/null 2>&1
python - "$c" <<'PY'
import csv, sys
c = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/ll_{c}.csv")) if len(r) > 10]
rows = [rows[0]] + [r for r in rows[1:] if r[0] != rows[0][0]]
hdr = rows[0]; data = rows[1:]
ik, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
seq = [(int(r[iid]), r[ik], float(r[iv].replace(",", ""))) for r in data]
# last step only: launches after the last L2 flush (FillFunctor<unsigned char>)
last = max(i for i, (_, k, _) in enumerate(seq) if "FillFunctor<unsigned char>" in k)
step = seq[last + 1:]
tot = sum(t for _, _, t in step)
print(f"{c}: {len(step)} launches in the last step, sum {tot/1e3:.1f} us (units ns->us)")
import collections
agg = collections.defaultdict(lambda: [0.0, 0])
for i, k, t in step:
    a = agg[k[:80]]
    a[0] += t
    a[1] += 1
if len(step) > 40:
    for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"  {t/1e3:9.1f} us  n={n:4d}  mean={t/n/1e3:6.2f} us  {k}")
else:
    for i, k, t in step:
        print(f"  {t/1e3:8.2f} us  {k[:90]}")
PY
