"""Print the live nodes of a workload program after passes.optimize (small sizes)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import sys, collections
from paper_1903_04243_b200 import workloads as WL, passes
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
kw = {"cfg4": dict(n=4, steps=3, units=64), "cfg2": dict(n=128, model=sys.argv[2] if len(sys.argv) > 2 else "mlp")}.get(cfg, {})
w = WL.BUILDERS[cfg](WL.this_api(), **kw)
keys=[tuple(o) for o in w.graph.outputs]
dst, m = passes.optimize(w.graph, keys)
keep=[m[k] for k in keys]
live = passes.live_set(dst, keep)
c = collections.Counter()
for n in dst.topo_order():
    if n.id not in live or n.kind in ("constant","placeholder","reshape","transpose","gather_rows","tile_leading"): continue
    c[n.kind]+=1
    ins=[(i[0], i[1], dst.ref_shape(i)) for i in n.inputs]
    attrs = {k:v for k,v in n.attrs.items() if k not in ('program','value','out_dtypes')}
    print(n.id, n.kind, dst.ref_shape((n.id,0)), ins[:8], attrs, len(n.attrs.get('program',())))
print(c)
