"""Accept graphs built by the reference `pforvec` package itself.

`import_graph(g)` translates a reference `Graph` (any object with the same
structure: `nodes` / `topo_order()` / `outputs` / `variables`, nodes with
`kind` / `attrs` / `inputs` / `control_deps` / `block`) into this package's
IR, recursively through cond / while / parfor blocks, re-running shape
inference.  Dtype tags and constant payloads are mapped by value, so the
executor can run graphs the reference's own `GraphBuilder` / `pfor` /
`jacobian` produced -- the drop-in path described in INTEGRATION.md.
"""

from __future__ import annotations

from .graph import Block, Graph
from .tensor import DType, TensorValue


def _dtype(d):
    if d is None or isinstance(d, DType):
        return d
    return DType(getattr(d, "value", d))


def _value(v):
    if isinstance(v, TensorValue):
        return v
    return TensorValue(_dtype(v.dtype), v.data)


def _attrs(kind, attrs):
    out = {}
    for k, v in attrs.items():
        if k == "value":
            out[k] = _value(v)
        elif k in ("dtype", "out_dtype"):
            out[k] = _dtype(v)
        else:
            out[k] = v
    return out


def is_native(g) -> bool:
    return isinstance(g, Graph)


def import_graph(src) -> Graph:
    if isinstance(src, Graph):
        return src
    dst = Graph()
    dst.variables = {k: _value(v) for k, v in getattr(src, "variables", {}).items()}
    dst.outer_variables = {k: _value(v) for k, v in getattr(src, "outer_variables", {}).items()}
    idmap = {}
    for node in src.topo_order():
        blk = None
        if node.block is not None:
            b = node.block
            blk = Block(b.kind, {name: import_graph(sg) for name, sg in b.subgraphs.items()},
                        b.num_carried, b.out_arity)
        ins = [(idmap[n], p) for n, p in node.inputs]
        new = dst.add_node(node.kind, ins, _attrs(node.kind, node.attrs),
                           control_deps=[idmap[c] for c in node.control_deps], block=blk)
        idmap[node.id] = new.id
    dst.set_outputs([(idmap[n], p) for n, p in src.outputs])
    dst._import_idmap = idmap
    return dst


def translate_ref(src_graph, dst_graph, ref):
    """Map an output reference of the source graph onto the imported graph."""
    if hasattr(ref, "nid"):
        nid, port = ref.nid, ref.port
    elif isinstance(ref, tuple):
        nid, port = ref
    else:
        nid, port = int(ref), 0
    return (dst_graph._import_idmap[nid], port)
