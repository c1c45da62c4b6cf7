"""Print the live nodes of a workload program after passes.optimize, including
the nested cond/while sub-graphs (small sizes)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1903_04243_b200 import passes, workloads as WL  # noqa: E402
from paper_1903_04243_b200.vectorize import vectorize_graph  # noqa: E402

SKIP = {"constant", "placeholder", "reshape", "transpose", "gather_rows", "tile_leading",
        "capture", "carried", "loop_var"}


def show(g, keep, ind=""):
    live = passes.live_set(g, keep)
    for n in g.topo_order():
        if n.id not in live or n.kind in SKIP:
            continue
        attrs = {k: v for k, v in n.attrs.items() if k not in ("program", "value", "out_dtypes")}
        print(ind, n.id, n.kind, g.ref_shape((n.id, 0)),
              [(i[0], g.ref_shape(i)) for i in n.inputs][:6], str(attrs)[:100])
        if n.block is not None:
            for name, sg in n.block.subgraphs.items():
                print(ind, "  --", name)
                show(sg, [tuple(o) for o in sg.outputs], ind + "    ")


if __name__ == "__main__":
    cfg = sys.argv[1]
    kw = eval("dict(" + (sys.argv[2] if len(sys.argv) > 2 else "") + ")")
    w = WL.BUILDERS[cfg](WL.this_api(), **kw)
    g, rm = w.graph, {}
    gv, _ = vectorize_graph(g, refmap_out=rm)
    keys = [(rm[tuple(o)].nid, rm[tuple(o)].port) if tuple(o) in rm else tuple(o) for o in g.outputs]
    dst, m = passes.optimize(gv, keys)
    show(dst, [m[k] for k in keys])
