"""Post-vectorization graph rewrites (SURVEY.md §8a "Required fusions").

The converter pass emits, per op, what the reference's greedy conversion
emits (PAPER.md:534-546 notes such graphs want follow-up fusion passes).
Per-example gradients of dense layers come out as stacked K=1 batched
matmuls -- rank-1 outer products a_i b_i^T -- which the reference then
squares, reduces, scales and sums elementwise over a [n, p, q] tensor.  These
rewrites compute the same values without that tensor:

F1a  reduce_sum(square(a (x) b), (1, 2))       ->  |a_i|^2 * |b_i|^2
F1b  reduce_sum((a (x) b) * s, (0,))            ->  A^T diag(s) B   (one K=n GEMM)
F2   (a_1 (x) b_1) + ... + (a_T (x) b_T)        ->  [a_1..a_T] [b_1..b_T]^T
                                                    (one batched K=T GEMM; B laid
                                                    out K-major for tcgen05)

Each rewrite adds nodes to a private copy of the graph and redirects the
consumers; the now-unread outer products are removed by the executor's
dead-code elimination.  Results agree with the unfused graph to fp32
rounding (tests/test_passes.py checks against the oracle).
"""

from __future__ import annotations

from .builder import GraphBuilder
from .graph import Ref


def copy_with_map(src):
    """Deep copy (blocks included) returning (graph, {(nid, port): (nid', port)})."""
    from .vectorize import copy_graph
    dst = copy_graph(src)
    # copy_graph walks topo order and assigns fresh ids in that order
    mapping = {}
    for old, new in zip(src.topo_order(), dst.topo_order()):
        for p in range(old.output_arity):
            mapping[(old.id, p)] = (new.id, p)
    return dst, mapping


class _Rewriter:
    def __init__(self, g, keep):
        self.g = g
        self.b = GraphBuilder(graph=g)
        self.keep = set(keep)  # (nid, port) that must stay materialised (requested outputs)
        self._users = None

    def users(self):
        if self._users is None:
            u = {}
            for n in self.g.nodes.values():
                for i, src in enumerate(n.inputs):
                    u.setdefault(src, []).append((n, i))
            self._users = u
        return self._users

    def node(self, key):
        return self.g.nodes[key[0]]

    def redirect(self, old_key, new_ref):
        for n, i in self.users().get(old_key, []):
            n.inputs[i] = (new_ref.nid, new_ref.port)
        if old_key in self.keep:
            self.keep.discard(old_key)
            self.keep.add((new_ref.nid, new_ref.port))
            self.replaced[old_key] = (new_ref.nid, new_ref.port)
        self._users = None
        self.g._topo_cache = None

    # -- pattern helpers ---------------------------------------------------------

    def outer(self, key):
        """(A [n,p,1] ref, B [n,1,q] ref) if `key` is a K=1 batched matmul."""
        n = self.node(key)
        if n.kind != "matmul" or key[1] != 0:
            return None
        sa = self.g.ref_shape(n.inputs[0])
        sb = self.g.ref_shape(n.inputs[1])
        if sa is None or sb is None or len(sa) != 3 or len(sb) != 3 or sa[2] != 1:
            return None
        if None in sa or None in sb:
            return None
        return Ref(self.g, *n.inputs[0]), Ref(self.g, *n.inputs[1])

    def single_use(self, key):
        return len(self.users().get(key, [])) == 1 and key not in self.keep


def fuse_outer_products(g, keep=()):
    """Apply F1a/F1b/F2 in place on `g` (a private copy).  Returns the number
    of rewrites and a map of requested outputs that moved."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    count = 0
    for node in list(g.topo_order()):
        if node.id not in g.nodes:
            continue
        if node.kind == "add":
            count += _f2(rw, node)
        elif node.kind == "reduce_sum":
            count += _f1(rw, node)
    return count, rw.replaced


def _f1(rw, node):
    g, b = rw.g, rw.b
    axes = tuple(node.attrs["axes"])
    src = node.inputs[0]
    inner = rw.node(src)
    # F1a: reduce_sum(square(outer), (1, 2))
    if inner.kind == "square" and axes in ((1, 2), (-2, -1), (1, -1)):
        ab = rw.outer(inner.inputs[0])
        if ab is None:
            return 0
        a, bb = ab
        na = b.reduce_sum(b.square(a), (1, 2))
        nb = b.reduce_sum(b.square(bb), (1, 2))
        rw.redirect((node.id, 0), b.mul(na, nb))
        return 1
    # F1b: reduce_sum(outer * s, (0,)) with s [n,1,1]
    if inner.kind == "mul" and axes in ((0,), (-3,)):
        for k in (0, 1):
            ab = rw.outer(inner.inputs[k])
            if ab is None:
                continue
            s_key = inner.inputs[1 - k]
            ss = g.ref_shape(s_key)
            sm = g.ref_shape(inner.inputs[k])
            if ss is None or len(ss) != 3 or ss[1:] != (1, 1) or ss[0] != sm[0]:
                continue
            a, bb = ab
            n, p, _ = g.ref_shape(a)
            q = g.ref_shape(bb)[2]
            a2 = b.reshape(a, [n, p])
            bs = b.mul(b.reshape(bb, [n, q]), b.reshape(Ref(g, *s_key), [n, 1]))
            rw.redirect((node.id, 0), b.matmul(b.transpose(a2, [1, 0]), bs))
            return 1
    return 0


def _f2(rw, node):
    """Collapse a single-use add tree whose leaves are same-shape K=1 outer
    products into one batched GEMM with K = number of leaves."""
    g, b = rw.g, rw.b
    leaves, stack, inner_adds = [], [(node.id, 0)], []
    while stack:
        key = stack.pop()
        n = rw.node(key)
        if n.kind == "add" and (key == (node.id, 0) or rw.single_use(key)):
            if g.ref_shape(n.inputs[0]) != g.ref_shape(n.inputs[1]):
                return 0
            inner_adds.append(key)
            stack.extend([n.inputs[1], n.inputs[0]])
            continue
        ab = rw.outer(key)
        if ab is None or not rw.single_use(key):
            return 0
        leaves.append(ab)
    if len(leaves) < 3:
        return 0
    # the root must not itself feed a larger add tree (handled from the top)
    users = rw.users().get((node.id, 0), [])
    if len(users) == 1 and users[0][0].kind == "add" and (node.id, 0) not in rw.keep:
        up = users[0][0]
        if g.ref_shape(up.inputs[0]) == g.ref_shape(up.inputs[1]):
            return 0
    # leaves were pushed right-first; restore left-to-right order
    leaves.reverse()
    a_cat = b.concat([a for a, _ in leaves], 2)                       # [n, p, T]
    bt = b.concat([b.transpose(bb, [0, 2, 1]) for _, bb in leaves], 2)  # [n, q, T]
    out = b.matmul(a_cat, b.transpose(bt, [0, 2, 1]))                  # K-major B view
    rw.redirect((node.id, 0), out)
    return 1


def optimize(g, keep_keys):
    """Copy `g`, apply the rewrites, return (graph, key map old->new)."""
    dst, mapping = copy_with_map(g)
    keep = [mapping[k] for k in keep_keys]
    _, moved = fuse_outer_products(dst, keep)
    final = {}
    for k, v in mapping.items():
        final[k] = moved.get(v, v)
    return dst, final
