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
F3   chains of elementwise ops (binary / unary / f32<->bool cast) whose interior
     values have no other live consumer  ->  one `fused_ew` launch running a
     small register program (the same fp32 ops in the same order).
F4   reduce_sum(square(x)) / reduce_sum(x * y)  ->  reduce_dot(x, y): the
     product is formed in registers inside the reduction.
F6   independent reduce_dot row-reductions over the same leading dim (the
     per-parameter-block |g_i|^2 of per-example norms)  ->  one
     `row_dots` launch with one output per reduction.
F5   GEMM prologue / epilogue (SURVEY.md §8a F3 "GEMM epilogues"):
     matmul(A, B * s[K,1]) -> [reshape] -> add(., bias[N]) -> [reshape] ->
     tanh | sigmoid | relu   ->  one `matmul_ep` launch (kscale scales B's
     rows as the operand is read; bias + activation in the store epilogue).

Each rewrite adds nodes to a private copy of the graph and redirects the
consumers; the now-unread outer products are removed by the executor's
dead-code elimination.  Results agree with the unfused graph to fp32
rounding (tests/test_passes.py checks against the oracle).
"""

from __future__ import annotations

import numpy as np

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
    for node in list(g.topo_order()):  # after F2 has claimed its outer-product trees
        if node.id in g.nodes and node.kind == "add":
            count += _f11(rw, node)
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


def _f11(rw, node, min_leaves=9):
    """F11: a single-use add tree over T >= 9 same-shape leaves -> one
    reduce_sum over the leaves stacked on a trailing axis (one launch instead
    of T-1; smaller trees are left to F3, whose fused kernels take up to 8
    inputs).  cfg4's per-example bias gradient dBg = sum_t dz_t: for [n,1,q]
    leaves the stack is built exactly like F2's K-major B operand (the
    transposed dz_t columns), so CSE then shares that concat and the sum
    only reads it.  Summation order changes (fp32 rounding only)."""
    g, b = rw.g, rw.b
    shape = g.ref_shape((node.id, 0))
    if shape is None or None in shape or not shape:
        return 0
    users = rw.users().get((node.id, 0), [])
    if len(users) == 1 and users[0][0].kind == "add" and (node.id, 0) not in rw.keep:
        up = users[0][0]
        if g.ref_shape(up.inputs[0]) == g.ref_shape(up.inputs[1]) == shape:
            return 0  # handled from the top of the tree
    leaves, stack = [], [(node.id, 0)]
    while stack:
        key = stack.pop()
        n = rw.node(key)
        if n.kind == "add" and (key == (node.id, 0) or rw.single_use(key)) and \
                g.ref_shape(n.inputs[0]) == g.ref_shape(n.inputs[1]) == shape:
            stack.extend([n.inputs[1], n.inputs[0]])
            continue
        leaves.append(key)
    if len(leaves) < min_leaves or g.ref_dtype((node.id, 0)) != g.ref_dtype(leaves[0]):
        return 0
    leaves.reverse()
    refs = [Ref(g, *k) for k in leaves]
    if len(shape) == 3 and shape[1] == 1:
        cat = b.concat([b.transpose(r, [0, 2, 1]) for r in refs], 2)  # [n, q, T]
        out = b.reshape(b.reduce_sum(cat, [2]), list(shape))
    else:
        cat = b.concat([b.reshape(r, list(shape) + [1]) for r in refs], len(shape))
        out = b.reduce_sum(cat, [len(shape)])
    rw.redirect((node.id, 0), out)
    return 1


def live_set(g, keep):
    """Nodes the requested outputs depend on (plus stateful nodes and control
    deps) -- what the executor will actually run."""
    from .graph import STATEFUL_KINDS
    live = set()
    todo = [k[0] for k in keep] + [n.id for n in g.nodes.values()
                                   if n.kind in STATEFUL_KINDS or n.block is not None]
    while todo:
        nid = todo.pop()
        if nid in live:
            continue
        live.add(nid)
        node = g.nodes[nid]
        todo.extend(src for src, _ in node.inputs)
        todo.extend(node.control_deps)
    return live


def fuse_reductions(g, keep=()):
    """F4: reduce_sum(square(x)) and reduce_sum(mul(x, y)) (y broadcast to x)
    -> reduce_dot(x, y): the product is never written to HBM."""
    keep = set(keep)
    live = live_set(g, keep)
    users = {}
    for n in g.nodes.values():
        if n.id in live:
            for src in n.inputs:
                users.setdefault(src, []).append(n)
    moved = {}
    count = 0
    from .tensor import DType
    for node in list(g.topo_order()):
        if node.kind != "reduce_sum" or node.id not in live:
            continue
        src = node.inputs[0]
        inner = g.nodes[src[0]]
        if len(users.get(src, [])) != 1 or src in keep or inner.out_dtypes[0] != DType.F64:
            continue
        if inner.kind == "square":
            x = y = inner.inputs[0]
        elif inner.kind == "mul":
            a, b = inner.inputs
            out_sh = inner.out_shapes[0]
            if g.ref_shape(a) == out_sh:
                x, y = a, b
            elif g.ref_shape(b) == out_sh:
                x, y = b, a
            else:
                continue
        else:
            continue
        new = g.add_node("reduce_dot", [x, y], {"axes": tuple(node.attrs["axes"])})
        for u in users.get((node.id, 0), []):
            u.inputs = [(new.id, 0) if s_ == (node.id, 0) else s_ for s_ in u.inputs]
        if (node.id, 0) in keep:
            moved[(node.id, 0)] = (new.id, 0)
            keep.discard((node.id, 0))
            keep.add((new.id, 0))
        count += 1
    g._topo_cache = None
    return count, moved


_ACT_KINDS = ("tanh", "sigmoid", "relu")


def fuse_matmul_epilogues(g, keep=()):
    """F5 in place on `g` (a private copy).  Returns (count, moved outputs)."""
    from .tensor import DType
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    count = 0
    for node in list(g.topo_order()):
        if node.id not in g.nodes or node.kind not in ("matmul", "matmul2"):
            continue
        if node.out_dtypes[0] != DType.F64:
            continue
        if node.kind == "matmul2" and node.attrs.get("has_bias"):
            continue
        count += _f5(rw, node)
    return count, rw.replaced


def _const_is(g, key, value):
    n = g.nodes[key[0]]
    if n.kind != "constant" or key[1] != 0:
        return False
    v = n.attrs["value"]
    return v.rank == 0 and float(v.data) == value


def _dop_pattern(g, key):
    """("dtanh", y) for sub(1, mul(y, y)); ("dsigmoid", y) for mul(y, sub(1, y))
    (either operand order) -- the cotangent factors autodiff emits for the
    tanh / sigmoid VJPs (autodiff.py, reference autodiff.py:108-111)."""
    n = g.nodes[key[0]]
    if key[1] != 0:
        return None
    if n.kind == "sub" and _const_is(g, n.inputs[0], 1.0):
        m = g.nodes[n.inputs[1][0]]
        if m.kind == "mul" and n.inputs[1][1] == 0 and tuple(m.inputs[0]) == tuple(m.inputs[1]):
            return "dtanh", tuple(m.inputs[0])
    if n.kind == "mul":
        for j in (0, 1):
            sn = g.nodes[n.inputs[1 - j][0]]
            if (sn.kind == "sub" and n.inputs[1 - j][1] == 0 and _const_is(g, sn.inputs[0], 1.0)
                    and tuple(sn.inputs[1]) == tuple(n.inputs[j])):
                return "dsigmoid", tuple(n.inputs[j])
    return None


def _strip_units(shape):
    return tuple(d for d in shape if d != 1)


def _f5(rw, node):
    import math
    g, b = rw.g, rw.b
    sm = g.ref_shape((node.id, 0))
    sa, sbb = g.ref_shape(node.inputs[0]), g.ref_shape(node.inputs[1])
    if None in (sm, sa, sbb) or None in sm or None in sa or None in sbb or sa[-1] == 0:
        return 0
    A, B = Ref(g, *node.inputs[0]), Ref(g, *node.inputs[1])
    kscale = None
    dual = node.kind == "matmul2"
    bn = rw.node(node.inputs[1])
    if (not dual and bn.kind == "mul" and node.inputs[1][1] == 0
            and rw.single_use(node.inputs[1])):
        for j in (0, 1):
            s_key, b0_key = bn.inputs[1 - j], bn.inputs[j]
            ss, s0 = g.ref_shape(s_key), g.ref_shape(b0_key)
            if (ss is not None and s0 is not None and tuple(s0) == tuple(sbb)
                    and len(ss) == len(s0) and ss[-1] == 1 and tuple(ss[:-1]) == tuple(s0[:-1])
                    and g.ref_dtype(s_key) == g.ref_dtype(b0_key)):
                kscale = b.reshape(Ref(g, *s_key), list(ss[:-1]))
                B = Ref(g, *b0_key)
                break
    n_cols = sm[-1]
    key = (node.id, 0)
    end = key
    bias = act = None
    dop = dy = None
    while True:
        us = rw.users().get(key, [])
        if len(us) != 1 or key in rw.keep:
            break
        un, idx = us[0]
        osh = g.ref_shape((un.id, 0))
        if osh is None or None in osh:
            break
        if un.kind == "reshape":
            unfold = (len(osh) == 3 and len(sm) == 2 and osh[0] * osh[1] == sm[0]
                      and osh[2] == sm[1])  # the fold path's [n*x, z] -> [n, x, z]
            if not unfold and (_strip_units(osh) != _strip_units(sm) or not osh
                               or osh[-1] != n_cols):
                break
            key = (un.id, 0)
            continue
        if un.kind == "add" and bias is None and act is None:
            other = un.inputs[1 - idx]
            bsh = g.ref_shape(other)
            if (bsh is None or None in bsh or tuple(osh) != tuple(g.ref_shape(key))
                    or g.ref_dtype(other) != g.ref_dtype(key)):
                break
            nb = math.prod(bsh)
            if not (nb == 1 or (nb == n_cols and bsh and bsh[-1] == n_cols)):
                break
            bias = b.reshape(Ref(g, *other), [nb])
            key = end = (un.id, 0)
            continue
        if un.kind in _ACT_KINDS and act is None:
            act = un.kind
            key = end = (un.id, 0)
            continue
        if un.kind == "mul" and dop is None and not dual and tuple(osh) == tuple(g.ref_shape(key)):
            pat = _dop_pattern(g, tuple(un.inputs[1 - idx]))
            if pat is not None and g.ref_dtype(pat[1]) == g.ref_dtype(key):
                ysh = g.ref_shape(pat[1])
                if ysh is not None and None not in ysh and len(ysh) <= len(osh) and all(
                        a in (1, o) for a, o in zip(ysh[::-1], tuple(osh)[::-1])):
                    dop, dy = pat[0], Ref(g, *pat[1])
                    end_before_dop = end
                    key = end = (un.id, 0)
                    continue
        break
    if kscale is None and bias is None and act is None and dop is None:
        return 0
    esh = tuple(g.ref_shape(end))
    if dop is not None:
        # the epilogue addresses y in the GEMM's output coordinates
        ysh = tuple(g.ref_shape(tuple((dy.nid, dy.port))))
        ypad = (1,) * (len(esh) - len(ysh)) + ysh
        if _strip_units(esh) == _strip_units(sm) and len(sm) == len(_strip_units(sm)):
            keep_ax = [i for i, d in enumerate(esh) if d != 1]
            dy = b.reshape(dy, [ypad[i] for i in keep_ax] or [1])
        else:  # y does not map onto the GEMM's output rows: stop before the mul
            dop = dy = None
            end = end_before_dop
            if kscale is None and bias is None and act is None:
                return 0
            esh = tuple(g.ref_shape(end))
    if dual:
        ins = [A, B, Ref(g, *node.inputs[2]), Ref(g, *node.inputs[3])] + (
            [bias] if bias is not None else [])
        new = g.add_node("matmul2", [(r.nid, r.port) for r in ins],
                         {"act": act, "has_bias": bias is not None})
    else:
        ins = [A, B] + ([kscale] if kscale is not None else []) + (
            [bias] if bias is not None else []) + ([dy] if dy is not None else [])
        new = g.add_node("matmul_ep", [(r.nid, r.port) for r in ins],
                         {"act": act, "has_kscale": kscale is not None,
                          "has_bias": bias is not None, "dop": dop})
    out = Ref(g, new.id, 0)
    if tuple(esh) != tuple(g.ref_shape((new.id, 0))):
        out = b.reshape(out, list(esh))
    rw.redirect(end, out)
    return 1


# ----------------------------------------------------------------------------
# F12: per-example conv filter gradients without the im2col buffer

def fuse_conv_filter_grads(g, keep=()):
    """F12 in place on `g` (a private copy): the conv2d VJP's filter gradient
    matmul(transpose(reshape(im2col(x))), reshape(gy)) -- per example
    im2col(x_i)^T gy_i, reference autodiff.py conv2d VJP over tensor.py:209-229
    -- becomes one `conv_filter_grad(x, gy)` node: a kernel that reads each
    image window in shared memory and reduces the k1*k2*c x o filter gradient
    in registers, so the [n, h, w, k1*k2*c] im2col buffer (9x the image for a
    3x3 filter) is never written (cfg2 ConvNet).  Same sums, different order
    (fp32 rounding).  Returns (count, moved outputs)."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    count = 0
    for node in list(g.topo_order()):
        if node.id in g.nodes and node.kind == "matmul":
            count += _f12(rw, node)
    return count, rw.replaced


def _f12(rw, node):
    g, b = rw.g, rw.b
    out_sh = g.ref_shape((node.id, 0))
    t = rw.node(node.inputs[0])
    if out_sh is None or None in out_sh or t.kind != "transpose" or node.inputs[0][1] != 0:
        return 0
    batched = len(out_sh) == 3
    if tuple(t.attrs["perm"]) != ((0, 2, 1) if batched else (1, 0)):
        return 0
    key = tuple(t.inputs[0])
    flat = g.ref_shape(key)
    while rw.node(key).kind == "reshape" and key[1] == 0:
        key = tuple(rw.node(key).inputs[0])
    im = rw.node(key)
    if im.kind != "im2col" or key[1] != 0:
        return 0
    xsh = g.ref_shape(tuple(im.inputs[0]))
    if xsh is None or None in xsh or len(xsh) != 4:
        return 0
    n, h, w, c = xsh
    k1, k2 = im.attrs["k1"], im.attrs["k2"]
    kc = k1 * k2 * c
    if tuple(flat) != ((n, h * w, kc) if batched else (h * w, kc)) or (not batched and n != 1):
        return 0
    bsh = g.ref_shape(node.inputs[1])
    if bsh is None or None in bsh or tuple(bsh[:-1]) != ((n, h * w) if batched else (h * w,)):
        return 0
    o = bsh[-1]
    gy = b.reshape(Ref(g, *node.inputs[1]), [n, h, w, o])
    new = g.add_node("conv_filter_grad", [tuple(im.inputs[0]), (gy.nid, gy.port)],
                     {"k1": k1, "k2": k2})
    out = Ref(g, new.id, 0)
    if not batched:
        out = b.reshape(out, [kc, o])
    rw.redirect((node.id, 0), out)
    return 1


# ----------------------------------------------------------------------------
# F10: common-subexpression elimination

_NO_CSE = frozenset({"read_variable", "assign", "assign_add", "random_uniform", "placeholder",
                     "loop_var", "carried", "capture"})


def _freeze(v):
    """Hashable, value-exact key of an attribute value."""
    from .tensor import TensorValue
    if isinstance(v, TensorValue):
        a = np.ascontiguousarray(v.data)
        return ("T", v.dtype.value, a.dtype.str, a.shape, a.tobytes())
    if isinstance(v, np.ndarray):
        a = np.ascontiguousarray(v)
        return ("A", a.dtype.str, a.shape, a.tobytes())
    if isinstance(v, dict):
        return ("D",) + tuple(sorted((k, _freeze(x)) for k, x in v.items()))
    if isinstance(v, (list, tuple)):
        return ("L",) + tuple(_freeze(x) for x in v)
    if hasattr(v, "value") and hasattr(v, "name"):  # enums (DType)
        return ("E", type(v).__name__, v.name)
    return ("V", repr(v))


def eliminate_common_subexpressions(g, keep=()):
    """F10 in place on `g` (a private copy): pure, block-free nodes with the
    same kind, attributes and (already merged) inputs -- constants compared by
    value -- are computed once; their readers are redirected to the first.
    `jacobian(y, W_l)` for several l (cfg3) builds one pfor per call, each
    re-deriving the same backward chain from y (reference apps.py:59-80,
    autodiff.py:181-200); after conversion those chains are identical
    subgraphs and collapse into one.  Values are unchanged.  Returns
    (count, moved outputs)."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    seen = {}
    canon = {}  # (nid, port) -> canonical (nid, port)
    count = 0
    for node in list(g.topo_order()):
        ins = tuple(canon.get(tuple(src), tuple(src)) for src in node.inputs)
        if ins != tuple(tuple(x) for x in node.inputs):
            node.inputs = list(ins)
            g._topo_cache = None
        if (node.kind in _NO_CSE or node.block is not None or node.control_deps
                or node.output_arity == 0):
            continue
        try:
            key = (node.kind, _freeze(node.attrs), ins)
        except Exception:
            continue
        first = seen.get(key)
        if first is None:
            seen[key] = node.id
            continue
        for p in range(node.output_arity):
            canon[(node.id, p)] = (first, p)
            if (node.id, p) in rw.keep:
                rw.keep.discard((node.id, p))
                rw.keep.add((first, p))
                rw.replaced[(node.id, p)] = (first, p)
        count += 1
    # readers created before a later duplicate was seen are already redirected
    # (topological order); outputs of the graph itself:
    g.outputs = [tuple(canon.get(tuple(o), tuple(o))) for o in g.outputs] if g.outputs else g.outputs
    dup = {k[0]: v[0] for k, v in canon.items()}
    for n in g.nodes.values():
        if n.control_deps & dup.keys():
            n.control_deps = {dup.get(d, d) for d in n.control_deps}
    for nid in dup:  # the duplicates: no reader is left
        g.nodes.pop(nid, None)
    rw._users = None
    g._topo_cache = None
    return count, rw.replaced


# ----------------------------------------------------------------------------
# F9: a column slice of a GEMM result -> a GEMM over the sliced columns

_VIEW_KINDS = frozenset({"reshape", "transpose"})


def _nonunit(shape):
    return [(i, d) for i, d in enumerate(shape) if d != 1]


def slice_matmul_columns(g, keep=()):
    """F9 in place on `g` (a private copy).  matmul(A, B) whose only live
    reader is a chain of views (reshape / transpose) ending in
    gather_rows(., idx) along the GEMM's column axis, idx a constant vector,
    becomes matmul(A, B[..., idx]) followed by the same views: only the
    gathered columns are computed.  Each output element is the same dot
    product as before (the K reduction does not depend on N), so values are
    bit-identical.  In the LSTM backward (cfg4) the GEMM dz_t Wg^T yields the
    cotangent of [x_t, h_{t-1}]; only the h half is live, so this halves
    every backward-step GEMM.  Returns (count, moved outputs)."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    live = live_set(g, set(keep))
    count = 0
    for node in list(g.topo_order()):
        if node.id in g.nodes and node.kind == "matmul" and node.id in live:
            count += _f9(rw, node, live)
    return count, rw.replaced


def _f9(rw, node, live):
    g = rw.g
    key = (node.id, 0)
    ysh = node.out_shapes[0]
    if ysh is None or None in ysh or len(ysh) not in (2, 3) or key in rw.keep:
        return 0
    naxis = len(ysh) - 1  # the GEMM's column axis in the current value
    chain = []
    cur, shape = key, tuple(ysh)
    while True:
        us = [(n, i) for n, i in rw.users().get(cur, []) if n.id in live]
        if len(us) != 1 or cur in rw.keep and cur != key:
            return 0
        u, _ = us[0]
        if u.kind == "transpose":
            perm = tuple(u.attrs["perm"])
            naxis = perm.index(naxis)
            chain.append(u)
            cur, shape = (u.id, 0), tuple(u.out_shapes[0])
        elif u.kind == "reshape":
            osh = u.out_shapes[0]
            if osh is None or None in osh:
                return 0
            a, b_ = _nonunit(shape), _nonunit(osh)
            if [d for _, d in a] != [d for _, d in b_]:
                return 0  # merges or splits real axes
            pos = [j for j, (i, _) in enumerate(a) if i == naxis]
            if not pos:
                return 0
            naxis = b_[pos[0]][0]
            chain.append(u)
            cur, shape = (u.id, 0), tuple(osh)
        elif u.kind == "gather_rows" and u.inputs[0] == cur and naxis == 0:
            idx_node = g.nodes[u.inputs[1][0]]
            if idx_node.kind != "constant":
                return 0
            idx = np.asarray(idx_node.attrs["value"].data)
            if idx.ndim != 1 or len(idx) >= ysh[-1] or u.id in rw.keep:
                return 0
            break
        else:
            return 0
    b = rw.b
    k = len(idx)
    B = Ref(g, *node.inputs[1])
    bsh = g.ref_shape(node.inputs[1])
    r = len(bsh)
    # B[..., idx]: bring the column axis to the front, gather, move it back
    front = [r - 1] + list(range(r - 1))
    back = list(range(1, r)) + [0]
    Bs = b.transpose(b.gather(b.transpose(B, front), Ref(g, *u.inputs[1])), back)
    y = b.matmul(Ref(g, *node.inputs[0]), Bs)
    # replay the view chain with the column extent k
    nax = len(ysh) - 1
    for v in chain:
        if v.kind == "transpose":
            perm = tuple(v.attrs["perm"])
            y = b.transpose(y, list(perm))
            nax = perm.index(nax)
        else:
            osh = list(v.out_shapes[0])
            cur_sh = g.ref_shape((y.nid, y.port))
            a = _nonunit(cur_sh) if k != 1 else [(i, d) for i, d in enumerate(cur_sh)
                                                  if d != 1 or i == nax]
            j = [t for t, (i, _) in enumerate(a) if i == nax][0]
            tgt = [i for i, d in enumerate(osh) if d != 1]
            newax = tgt[j]
            osh[newax] = k
            y = b.reshape(y, osh)
            nax = newax
    if tuple(g.ref_shape((y.nid, y.port))) != tuple(u.out_shapes[0]):
        return 0  # (leaves the added nodes dead; the executor's DCE drops them)
    rw.redirect((u.id, 0), y)
    return 1


# ----------------------------------------------------------------------------
# F8: loop-invariant code motion out of while bodies

_NO_LICM = frozenset({"read_variable", "assign", "assign_add", "random_uniform", "placeholder",
                      "loop_var", "carried", "capture", "constant"})
# ops that raise on their data (index out of range, scatter collision /
# incomplete cover): hoisted out of a while body they would run -- and raise
# -- on a zero-trip loop whose body the reference never evaluates
_MAY_RAISE = frozenset({"gather_rows", "gather_stacked", "scatter_rows", "scatter_add_rows"})


def _provably_safe(g, wnode, body, n):
    """A raising op may still move when it cannot raise: a gather by a
    constant index (in the body, or captured from a constant of the
    enclosing graph) that is in range of x's static leading dimension."""
    if n.kind != "gather_rows":
        return False
    src = body.nodes[n.inputs[1][0]]
    if src.kind == "capture":
        pref = wnode.inputs[wnode.block.num_carried + src.attrs["index"]]
        src = g.nodes[pref[0]]
    xs = body.ref_shape(tuple(n.inputs[0]))
    if src.kind != "constant" or not xs or xs[0] is None:
        return False
    v = np.asarray(src.attrs["value"].data)
    return bool(((v >= 0) & (v < xs[0])).all())


def hoist_loop_invariants(g):
    """F8 in place on `g` (a private copy), nested blocks first: every pure
    node of a `while` body whose inputs are all captures, constants or other
    such nodes is evaluated once in the enclosing graph and reaches the body
    as a new capture (the reference re-evaluates it every trip, e.g. the
    row-index iota of the per-example gathers in cfg5's body).  Values are
    unchanged.  Returns the number of nodes moved."""
    moved_total = 0
    for node in list(g.topo_order()):
        if node.block is None:
            continue
        for sg in node.block.subgraphs.values():
            moved_total += hoist_loop_invariants(sg)
        if node.block.kind != "while":
            continue
        moved_total += _licm_while(g, node)
    return moved_total


def _licm_while(g, wnode):
    body = wnode.block.subgraphs["body"]
    nc = wnode.block.num_carried
    inv = set()
    movable = []
    for n in body.topo_order():
        if n.kind in ("capture", "constant"):
            inv.add(n.id)
        elif (n.kind not in _NO_LICM and n.block is None and n.inputs and not n.control_deps
              and all(src in inv for src, _ in n.inputs)
              and (n.kind not in _MAY_RAISE or _provably_safe(g, wnode, body, n))):
            inv.add(n.id)
            movable.append(n)
    if not movable:
        return 0
    users = {}
    for n in body.nodes.values():
        for src in n.inputs:
            users.setdefault(tuple(src), []).append(n)
    outs = {tuple(o) for o in body.outputs}
    pmap = {}  # body (nid, port) -> parent (nid, port)

    def parent_ref(src):
        sn = body.nodes[src[0]]
        if sn.kind == "capture":
            return tuple(wnode.inputs[nc + sn.attrs["index"]])
        if sn.kind == "constant":
            if src not in pmap:
                c = g.add_node("constant", [], dict(sn.attrs))
                pmap[src] = (c.id, 0)
            return pmap[src]
        return pmap[src]

    moved_ids = {n.id for n in movable}
    for n in movable:
        pn = g.add_node(n.kind, [parent_ref(tuple(s_)) for s_ in n.inputs], dict(n.attrs))
        for p in range(n.output_arity):
            pmap[(n.id, p)] = (pn.id, p)
    count = 0
    for n in movable:
        for p in range(n.output_arity):
            key = (n.id, p)
            ext = [u for u in users.get(key, []) if u.id not in moved_ids]
            if not ext and key not in outs:
                continue
            idx = len(wnode.inputs) - nc
            pref = pmap[key]
            pnode = g.nodes[pref[0]]
            cap = body.add_node("capture", [], {"index": idx, "dtype": pnode.out_dtypes[p],
                                                "shape": pnode.out_shapes[p]})
            wnode.inputs.append(pref)
            for u in ext:
                u.inputs = [(cap.id, 0) if tuple(s_) == key else s_ for s_ in u.inputs]
            if key in outs:
                body.outputs = [(cap.id, 0) if tuple(o) == key else o for o in body.outputs]
            count += 1
    body._topo_cache = None
    g._topo_cache = None
    return len(movable)


# ----------------------------------------------------------------------------
# F7: two GEMMs into one output -> one dual-operand GEMM launch

def fuse_dual_matmuls(g, keep=()):
    """F7 in place on `g` (a private copy).  Two patterns become one
    `matmul2(a1, b1, a2, b2)` node (out = a1 @ b1 + a2 @ b2, one launch that
    accumulates both K ranges):
      * add(M1, M2) of two single-use rank-2 matmuls (through reshapes) with
        the same output shape -- e.g. the RNN cell z = x_t Wx + h Wh (cfg5);
      * matmul(reshape(concat([a1, a2], -1)), B) with a single-use concat:
        B's rows split at K1 (zero-cost view gathers), no concat copy.
    Returns (count, moved outputs)."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    count = 0
    for node in list(g.topo_order()):
        if node.id not in g.nodes:
            continue
        if node.kind == "add":
            count += _f7_sum(rw, node)
        elif node.kind == "matmul":
            count += _f7_cat(rw, node)
    return count, rw.replaced


def _through_reshapes(rw, key):
    """Follow single-use reshapes upward from `key`; the first non-reshape key."""
    while True:
        n = rw.node(key)
        if n.kind != "reshape" or not rw.single_use(key):
            return key
        key = n.inputs[0]


def _f7_sum(rw, node):
    from .tensor import DType
    g, b = rw.g, rw.b
    osh = g.ref_shape((node.id, 0))
    if osh is None or None in osh:
        return 0
    if any(g.ref_shape(i) is None or tuple(g.ref_shape(i)) != tuple(osh) for i in node.inputs):
        return 0
    mms = []
    for i in node.inputs:
        k = _through_reshapes(rw, i)
        n = rw.node(k)
        if n.kind != "matmul" or k[1] != 0 or not rw.single_use(k) or n.out_dtypes[0] != DType.F64:
            return 0
        sa, sb = g.ref_shape(n.inputs[0]), g.ref_shape(n.inputs[1])
        if sa is None or sb is None or len(sa) != 2 or len(sb) != 2 or None in sa or None in sb:
            return 0
        if sa[1] == 0:
            return 0
        mms.append(n)
    m1, m2 = mms
    if tuple(g.ref_shape((m1.id, 0))) != tuple(g.ref_shape((m2.id, 0))):
        return 0
    new = g.add_node("matmul2", [m1.inputs[0], m1.inputs[1], m2.inputs[0], m2.inputs[1]],
                     {"act": None, "has_bias": False})
    out = Ref(g, new.id, 0)
    if tuple(g.ref_shape((new.id, 0))) != tuple(osh):
        out = b.reshape(out, list(osh))
    rw.redirect((node.id, 0), out)
    return 1


def _f7_cat(rw, node):
    from .tensor import DType
    g, b = rw.g, rw.b
    if node.out_dtypes[0] != DType.F64:
        return 0
    sa, sb = g.ref_shape(node.inputs[0]), g.ref_shape(node.inputs[1])
    if sa is None or sb is None or len(sa) != 2 or len(sb) != 2 or None in sa or None in sb:
        return 0
    ck = _through_reshapes(rw, node.inputs[0])
    cn = rw.node(ck)
    if cn.kind != "concat" or len(cn.inputs) != 2 or not rw.single_use(ck):
        return 0
    csh = g.ref_shape(ck)
    if csh is None or None in csh or not csh:
        return 0
    ax = cn.attrs["axis"]
    if ax < 0:
        ax += len(csh)
    if ax != len(csh) - 1 or csh[-1] != sa[1]:
        return 0
    parts = []
    for i in cn.inputs:
        ps = g.ref_shape(i)
        if ps is None or None in ps or ps[-1] == 0 or g.ref_dtype(i) != DType.F64:
            return 0
        parts.append((Ref(g, *i), ps[-1]))
    k1 = parts[0][1]
    rows = sa[0]
    a1 = b.reshape(parts[0][0], [rows, k1])
    a2 = b.reshape(parts[1][0], [rows, sa[1] - k1])
    B = Ref(g, *node.inputs[1])
    b1 = b.gather(B, b.const(np.arange(0, k1, dtype=np.int64)))
    b2 = b.gather(B, b.const(np.arange(k1, sa[1], dtype=np.int64)))
    new = g.add_node("matmul2", [(a1.nid, a1.port), (b1.nid, b1.port), (a2.nid, a2.port),
                                 (b2.nid, b2.port)], {"act": None, "has_bias": False})
    rw.redirect((node.id, 0), Ref(g, new.id, 0))
    return 1


MAX_ROW_DOTS = 8


def fuse_row_dots(g, keep=()):
    """F6 in place on `g`: group reduce_dot nodes that reduce every
    non-leading axis of same-shape operands and share the leading extent into
    `row_dots` nodes (<= 8 each).  A node joins a group only if no member is
    its ancestor or descendant, so the grouped node cannot create a cycle."""
    from .tensor import DType
    keep = set(keep)
    live = live_set(g, keep)
    cands = []
    for node in g.topo_order():
        if node.kind != "reduce_dot" or node.id not in live:
            continue
        x, y = node.inputs
        sx, sy = g.ref_shape(x), g.ref_shape(y)
        if sx is None or None in sx or len(sx) < 2 or tuple(sx) != tuple(sy):
            continue
        if node.out_dtypes[0] != DType.F64:
            continue
        from .tensor import normalize_axes
        if tuple(sorted(normalize_axes(node.attrs["axes"], len(sx)))) != tuple(range(1, len(sx))):
            continue
        cands.append(node)
    if len(cands) < 2:
        return 0, {}
    anc_memo = {}

    def ancestors(nid):
        if nid in anc_memo:
            return anc_memo[nid]
        out, todo = set(), [nid]
        while todo:
            k = todo.pop()
            for src, _ in g.nodes[k].inputs:
                if src not in out:
                    out.add(src)
                    todo.append(src)
        anc_memo[nid] = out
        return out

    groups = []
    for node in cands:
        lead = g.ref_shape(node.inputs[0])[0]
        anc = ancestors(node.id)
        placed = False
        for grp in groups:
            if grp["lead"] != lead or len(grp["nodes"]) >= MAX_ROW_DOTS:
                continue
            if any(m.id in anc or node.id in ancestors(m.id) for m in grp["nodes"]):
                continue
            grp["nodes"].append(node)
            placed = True
            break
        if not placed:
            groups.append({"lead": lead, "nodes": [node]})
    users = {}
    for n in g.nodes.values():
        for i, src in enumerate(n.inputs):
            users.setdefault(src, []).append((n, i))
    moved, count = {}, 0
    for grp in groups:
        members = grp["nodes"]
        if len(members) < 2:
            continue
        ins = []
        for m in members:
            ins.extend(m.inputs)
        new = g.add_node("row_dots", ins, {"n": len(members)})
        for j, m in enumerate(members):
            for u, i in users.get((m.id, 0), []):
                u.inputs[i] = (new.id, j)
            if (m.id, 0) in keep:
                moved[(m.id, 0)] = (new.id, j)
        count += 1
    g._topo_cache = None
    return count, moved


def _pipeline(elementwise):
    seq = [eliminate_common_subexpressions, stack_onehot_sums, place_scatter_sums,
           slice_matmul_columns,
           fuse_outer_products, fuse_conv_filter_grads, eliminate_common_subexpressions,
           fuse_reductions, fuse_row_dots, fuse_dual_matmuls, fuse_matmul_epilogues]
    if elementwise:
        seq += [sink_unit_reshapes, fuse_elementwise, place_concats, fuse_row_sums]
    seq += [merge_sibling_gathers, merge_sibling_reduce_dots]
    return seq


def _optimize_in_place(g, keep, elementwise=True):
    """Run the rewrites on `g`; returns (new keep keys, composed key map)."""
    moved_all = []
    for fn in _pipeline(elementwise):
        _, moved = fn(g, keep)
        keep = [moved.get(k, k) for k in keep]
        moved_all.append(moved)
    return keep, moved_all


def _optimize_blocks(g, elementwise=True):
    """Apply the rewrites inside every cond / while sub-graph (outputs kept)."""
    for node in list(g.nodes.values()):
        if node.block is None:
            continue
        for sg in node.block.subgraphs.values():
            _optimize_blocks(sg, elementwise)
            sg.set_outputs(_optimize_in_place(sg, [tuple(o) for o in sg.outputs], elementwise)[0])


def optimize(g, keep_keys, elementwise=True):
    """Copy `g`, apply the rewrites, return (graph, key map old->new)."""
    dst, mapping = copy_with_map(g)
    hoist_loop_invariants(dst)
    _optimize_blocks(dst, elementwise)
    keep = [mapping[k] for k in keep_keys]
    _, moved_all = _optimize_in_place(dst, keep, elementwise)
    final = {}
    for k, v in mapping.items():
        for moved in moved_all:
            v = moved.get(v, v)
        final[k] = v
    return dst, final


# ----------------------------------------------------------------------------
# F14: unit-dim reshapes of elementwise results move onto their operands
#
# reshape(less(r, 0), [n, 1, 1]) == less(reshape(r, [n, 1, 1]), 0): with the
# reshape on the operand, the elementwise op has the broadcast shape of the
# group that reads it and F3 absorbs it (the op is evaluated per element of
# the group's output on the broadcast operand -- the same values).  cfg5's
# per-step `reduce_sum(z) < 0` mask then costs no launch of its own.

def _nonunit_dims(shape):
    return [d for d in shape if d != 1]


def sink_unit_reshapes(g, keep=()):
    """F14 in place on `g` (a private copy).  Returns (count, moved outputs)."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    live = live_set(g, keep)
    count = 0
    for node in list(g.topo_order()):
        if node.id not in g.nodes or node.kind != "reshape" or node.id not in live:
            continue
        count += _f14(rw, node, live)
    return count, rw.replaced


def _f14(rw, node, live):
    g = rw.g
    src = tuple(node.inputs[0])
    e = rw.node(src)
    readers = [n for n, _ in rw.users().get(src, []) if n.id in live]
    if src[1] != 0 or len(readers) != 1 or src in rw.keep or e.output_arity != 1:
        return 0
    if e.kind not in _CHEAP_BCAST or not (_ew_eligible(g, e, "float") or _ew_eligible(g, e, "int")):
        return 0
    es, rs = g.ref_shape(src), g.ref_shape((node.id, 0))
    if es is None or rs is None or None in es or None in rs or tuple(es) == tuple(rs):
        return 0
    # only for a broadcast operand of an elementwise reader (what F3 can then
    # absorb); a reshape feeding a concat or a GEMM keeps the op where it is
    rr = [n for n, _ in rw.users().get((node.id, 0), []) if n.id in live]
    if not rr or not all((_ew_eligible(g, n, "float") or _ew_eligible(g, n, "int"))
                         and tuple(n.out_shapes[0] or ()) != tuple(rs) for n in rr):
        return 0
    if _nonunit_dims(es) != _nonunit_dims(rs):
        return 0
    ins = []
    for k in e.inputs:
        sk = g.ref_shape(tuple(k))
        if sk is None or None in sk:
            return 0
        if len(sk) == 0:
            ins.append(tuple(k))
        elif tuple(sk) == tuple(es):
            r = g.add_node("reshape", [tuple(k)], {"shape": list(rs)})
            ins.append((r.id, 0))
        else:
            return 0
    new = g.add_node(e.kind, ins, dict(e.attrs))
    rw.redirect((node.id, 0), Ref(g, new.id, 0))
    return 1


# ----------------------------------------------------------------------------
# F3: elementwise chains -> one fused_ew launch

_BIN_CODE = {"add": 0, "sub": 1, "mul": 2, "div": 3, "max": 4, "min": 5, "less": 6, "equal": 7}
_UN_CODE = {"neg": 0, "exp": 1, "log": 2, "relu": 3, "tanh": 4, "sigmoid": 5, "square": 6,
            "logical_not": 7}
OP_LOAD, OP_CONST, OP_TOBOOL, OP_MOV, OP_SELECT = 64, 65, 66, 67, 68
MAX_INPUTS, MAX_STEPS, MAX_REGS = 16, 96, 32


_INT_BIN = frozenset({"add", "sub", "mul", "max", "min", "less", "equal"})
_INT_UN = frozenset({"neg", "square", "logical_not"})


def _ew_eligible(g, node, domain="float"):
    """Can `node` join an elementwise group of `domain`: "float" (fp32 / bool
    registers, `fused_ew[m]`) or "int" (int64 / bool registers, `fused_int`:
    loop counters, index arithmetic, masks)."""
    from .tensor import DType
    k = node.kind
    allowed = (DType.F64, DType.BOOL) if domain == "float" else (DType.I64, DType.BOOL)
    if domain == "float":
        if k not in _BIN_CODE and k not in _UN_CODE and k not in ("cast", "select"):
            return False
    elif k not in _INT_BIN and k not in _INT_UN and k not in ("cast", "select"):
        return False
    if node.output_arity != 1:
        return False
    if node.out_dtypes[0] not in allowed:
        # an integer group may end in cast(i64 / bool -> f64) (one-hot and
        # mask factors): its f64 output can only be the group's root, since
        # no integer-domain op takes an f64 operand
        if not (domain == "int" and k == "cast" and node.out_dtypes[0] == DType.F64):
            return False
    sh = node.out_shapes[0]
    if sh is None or any(d is None for d in sh):
        return False
    for src in node.inputs:
        if g.ref_dtype(src) not in allowed:
            return False
    if k == "select" and g.ref_dtype(node.inputs[0]) != DType.BOOL:
        return False
    return True


_CHEAP_BCAST = frozenset({"less", "equal", "add", "sub", "mul", "neg", "logical_not", "select"})


def _broadcasts_to(sh, shape):
    if sh is None or len(sh) > len(shape):
        return False
    sh = (1,) * (len(shape) - len(sh)) + tuple(sh)
    return all(a == b or a == 1 for a, b in zip(sh, shape))


def _domains(g, node):
    """Domains a group rooted at `node` can use (bool-only roots: both)."""
    from .tensor import DType
    if node.output_arity != 1:
        return ()
    dts = [node.out_dtypes[0]] + [g.ref_dtype(s_) for s_ in node.inputs]
    if node.kind == "cast" and dts[0] == DType.F64 and dts[1] in (DType.I64, DType.BOOL):
        return ("int", "float")  # i64 / bool -> f64: the end of an integer group
    if any(d == DType.I64 for d in dts):
        return ("int",)
    if any(d == DType.F64 for d in dts):
        return ("float",)
    return ("int", "float")


def _const_scalar_i(g, key):
    import numpy as np
    from .tensor import DType
    n = g.nodes[key[0]]
    if n.kind == "constant" and key[1] == 0:
        v = n.attrs["value"]
        if v.rank == 0 and v.dtype in (DType.I64, DType.BOOL):
            x = int(np.asarray(v.data).item())
            if -2 ** 31 <= x < 2 ** 31:
                return x
    return None


def _const_scalar_f(g, key):
    import numpy as np
    from .tensor import DType
    n = g.nodes[key[0]]
    if n.kind == "constant" and key[1] == 0:
        v = n.attrs["value"]
        if v.rank == 0 and v.dtype == DType.F64:
            return float(np.float32(v.item()))
    return None


def _program(g, order, root, externals, outputs=(), domain="float"):
    """Register program for the group `order` (topo order, root last).
    Registers of `outputs` (node ids) are kept to the end of the program.
    domain "int": constants are int32 immediates, casts bool<->i64."""
    import struct
    from .tensor import DType
    ext_index = {k: i for i, k in enumerate(externals)}
    last_use = {}
    for i, n in enumerate(order):
        for src in n.inputs:
            last_use[src] = i
    free = list(range(MAX_REGS - 1, -1, -1))
    reg = {}
    steps = []
    pinned = {(i, 0) for i in outputs}

    def operand(src):
        if src in reg:
            return reg[src]
        if not free:
            raise OverflowError
        r = free.pop()
        c = _const_scalar_f(g, src) if domain == "float" else _const_scalar_i(g, src)
        if c is not None:
            bits = struct.unpack("<i", struct.pack("<f", c))[0] if domain == "float" else c
            steps.append((OP_CONST, r, bits, 0))
        else:
            steps.append((OP_LOAD, r, ext_index[src], 0))
        reg[src] = r
        return r

    for i, n in enumerate(order):
        ops = [operand(src) for src in n.inputs]
        k = n.kind
        if k == "select":  # r[dst] = m ? a : b; dst must not alias m or a
            if not free:
                raise OverflowError
            dst = free.pop()
            steps.append((OP_MOV, dst, ops[2], ops[2]))
            steps.append((OP_SELECT, dst, ops[0], ops[1]))
            for src in set(n.inputs):
                if last_use.get(src) == i and src in reg and src not in pinned:
                    free.append(reg.pop(src))
            reg[(n.id, 0)] = dst
            continue
        for src in set(n.inputs):
            if last_use.get(src) == i and src in reg and src not in pinned:
                free.append(reg.pop(src))
        if not free:
            raise OverflowError
        dst = free.pop()
        if k in _BIN_CODE:
            steps.append((_BIN_CODE[k], dst, ops[0], ops[1]))
        elif k in _UN_CODE:
            steps.append((16 + _UN_CODE[k], dst, ops[0], ops[0]))
        else:  # cast between f64 (fp32) / i64 and bool
            to = n.attrs["dtype"]
            frm = g.ref_dtype(n.inputs[0])
            op = OP_TOBOOL if (to == DType.BOOL and frm != DType.BOOL) else OP_MOV
            steps.append((op, dst, ops[0], ops[0]))
        reg[(n.id, 0)] = dst
    if len(steps) > MAX_STEPS:
        raise OverflowError
    if outputs:
        return tuple(steps), tuple(reg[(i, 0)] for i in outputs)
    return tuple(steps)


MAX_OUTPUTS = 12


def fuse_elementwise(g, keep=()):
    """Replace elementwise groups (same output shape) by `fused_ew` nodes.
    A producer whose value is also read outside the group is absorbed when
    every such outside reader comes after the group's root in topological
    order (so the fused node cannot be on a cycle); it then becomes an extra
    output of a multi-output `fused_ewm` node.  Groups whose register program
    does not fit fall back to the single-output rule (interior values read
    only inside the group).  Returns the number of groups fused and the moved
    requested outputs."""
    keep = set(keep)
    topo = g.topo_order()
    live = live_set(g, keep)
    pos = {n.id: i for i, n in enumerate(topo)}
    users = {}
    for n in topo:
        if n.id not in live:
            continue
        for src in n.inputs:
            users.setdefault(src, set()).add(n.id)
    assigned = set()
    moved = {}
    fused = 0

    def grow(root, multi, domain="float"):
        shape = root.out_shapes[0]
        rpos = pos[root.id]
        group = {root.id}
        changed = True
        while changed:
            changed = False
            for nid in list(group):
                for src in g.nodes[nid].inputs:
                    p = g.nodes[src[0]]
                    if p.id in group or p.id in assigned or src[1] != 0:
                        continue
                    if not _ew_eligible(g, p, domain):
                        continue
                    outside = users.get(src, set()) - group
                    if p.out_shapes[0] != shape:
                        # a producer of a broadcast operand (F14): evaluated per
                        # element of the group's shape, so only cheap ops
                        # (compares, add/sub/mul, neg, logical not, select) and
                        # only when nothing else reads it
                        if (outside or src in keep or p.kind not in _CHEAP_BCAST
                                or not _broadcasts_to(p.out_shapes[0], shape)):
                            continue
                    if multi:
                        if any(pos[u] <= rpos for u in outside):
                            continue
                        n_out = 1 + sum(1 for m in group if m != root.id and _is_out(m, group))
                        if (outside or src in keep) and n_out + 1 > MAX_OUTPUTS:
                            continue
                    elif outside or src in keep:
                        continue
                    if len(group) + 1 > MAX_STEPS // 2:
                        continue
                    group.add(p.id)
                    changed = True
        return group

    def _is_out(nid, group):
        key = (nid, 0)
        return key in keep or bool(users.get(key, set()) - group)

    def build(root, group, domain="float"):
        order = sorted((g.nodes[i] for i in group), key=lambda n: pos[n.id])
        const_of = _const_scalar_f if domain == "float" else _const_scalar_i
        externals = []
        for n in order:
            for src in n.inputs:
                if src[0] not in group and src not in externals and const_of(g, src) is None:
                    externals.append(src)
        if len(externals) > MAX_INPUTS or not externals:
            # (no tensor input: a constant-only group -- left to the
            # executor's constant hoisting; the kernel needs >= 1 operand)
            return None
        extra = [n.id for n in order if n.id != root.id and _is_out(n.id, group)]
        try:
            if not extra and domain == "float":
                return order, externals, [root.id], _program(g, order, root, externals), None
            outs = [root.id] + extra
            prog, regs = _program(g, order, root, externals, outs, domain)
            return order, externals, outs, prog, regs
        except OverflowError:
            return None

    def best_group(root, domain):
        group = grow(root, True, domain)
        built = build(root, group, domain) if len(group) >= 2 else None
        if built is None:
            group = grow(root, False, domain)
            if len(group) < 2:
                # a lone op (the loop-trip `select` of a predicated while
                # body, the maxpool's backward mask compare) may still merge
                # with a sibling / producer group below; unmerged singletons
                # are dropped after merging
                return (group, None) if len(group) == 1 else None
            built = build(root, group, domain)
        return None if built is None else (group, built)

    groups = []  # [root, group, domain, built], reverse topo order of roots
    for root in reversed(topo):
        if root.id in assigned or root.id not in live:
            continue
        cands = [(d, best_group(root, d)) for d in _domains(g, root) if _ew_eligible(g, root, d)]
        cands = [(d, r) for d, r in cands if r is not None]
        if not cands:
            continue
        domain, (group, built) = max(cands, key=lambda c: len(c[1][0]))
        groups.append([root, group, domain, built])
        assigned |= group

    groups = _merge_groups(g, groups, users, pos, live, build)
    groups = [grp for grp in groups if grp[3] is not None]

    for root, group, domain, built in groups:
        order, externals, outs, prog, regs = built
        if domain == "int":
            new = g.add_node("fused_int", externals,
                             {"program": prog, "out_regs": regs,
                              "out_dtypes": tuple(g.nodes[i].out_dtypes[0] for i in outs)})
        elif regs is None:
            new = g.add_node("fused_ew", externals,
                             {"program": prog, "out_dtype": root.out_dtypes[0]})
        else:
            new = g.add_node("fused_ewm", externals,
                             {"program": prog, "out_regs": regs,
                              "out_dtypes": tuple(g.nodes[i].out_dtypes[0] for i in outs)})
        live.add(new.id)
        pos[new.id] = pos[root.id]
        for src in externals:  # the fused node now reads these (later groups redirect it)
            users.setdefault(src, set()).add(new.id)
            users[src] -= group
        for k, nid in enumerate(outs):
            key = (nid, 0)
            ext = users.get(key, set()) - group
            for u in ext:
                un = g.nodes[u]
                un.inputs = [(new.id, k) if s_ == key else s_ for s_ in un.inputs]
            users[(new.id, k)] = set(ext)
            if key in keep:
                moved[key] = (new.id, k)
        fused += 1
    g._topo_cache = None
    return fused, moved


def _merge_groups(g, groups, users, pos, live, build):
    """Merge same-shape, same-domain elementwise groups that are siblings
    (read a common tensor) or producer -> consumer, when the union has no
    path leaving and re-entering it through other nodes (which would make the
    fused node depend on itself) and its register program fits.  The LSTM
    backward step's gate cotangents (four groups reading dh and the saved
    gates) become one multi-output launch."""
    by_node = {}
    for gi, grp in enumerate(groups):
        for nid in grp[1]:
            by_node[nid] = gi
    alive = [True] * len(groups)

    def shape_of(grp):
        return grp[0].out_shapes[0]

    def inputs_of(grp):
        return {src for nid in grp[1] for src in g.nodes[nid].inputs if src[0] not in grp[1]}

    def creates_cycle(union):
        """Is there a path union -> (other nodes / other groups, each group
        contracted to one node) -> union?  Only nodes before the union's last
        position can lead back into it."""
        hi = max(pos[i] for i in union)
        seen = set()
        todo = [u for nid in union for p_ in range(g.nodes[nid].output_arity)
                for u in users.get((nid, p_), ()) if u not in union]
        while todo:
            u = todo.pop()
            if u in union:
                return True
            if u in seen or u not in pos:
                continue
            gi = by_node.get(u)
            grouped = gi is not None and alive[gi]
            if pos[u] > hi and not (grouped and min(pos[m] for m in groups[gi][1]) <= hi):
                continue
            seen.add(u)
            members = groups[gi][1] if grouped else (u,)
            for m in members:
                seen.add(m)
                for p_ in range(g.nodes[m].output_arity):
                    for v in users.get((m, p_), ()):
                        if v in union:
                            return True
                        if v not in seen:
                            todo.append(v)
        return False

    changed = True
    while changed:
        changed = False
        for bi, b in enumerate(groups):
            if not alive[bi]:
                continue
            b_in = inputs_of(b)
            related = set()
            for src in b_in:
                if src[0] in by_node:
                    related.add(by_node[src[0]])  # producer group
                for u in users.get(src, ()):
                    if u in by_node:
                        related.add(by_node[u])  # sibling reading the same tensor
            related.discard(bi)
            for ai in sorted(related, key=lambda i: -pos[groups[i][0].id]):
                if not alive[ai] or not alive[bi]:
                    continue
                a = groups[ai]
                if a[2] != b[2] or shape_of(a) != shape_of(b):
                    continue
                union = a[1] | b[1]
                if creates_cycle(union):
                    continue
                root = a[0] if pos[a[0].id] > pos[b[0].id] else b[0]
                built = build(root, union, a[2])
                if built is None:
                    continue
                keep_i, drop_i = (ai, bi) if root is a[0] else (bi, ai)
                groups[keep_i] = [root, union, a[2], built]
                alive[drop_i] = False
                for nid in union:
                    by_node[nid] = keep_i
                changed = True
                if drop_i == bi:
                    break
                b = groups[bi]
                b_in = inputs_of(b)
    out = [grp for grp, ok in zip(groups, alive) if ok]
    out.sort(key=lambda grp: -pos[grp[0].id])
    return out


# ----------------------------------------------------------------------------
# F13: placement instead of arithmetic for stacked results
#
# (a) The vectorized gradient of gather(v, g) at a constant index g is the
#     cotangent times a one-hot of g (reference autodiff.py:100-110 emits
#     scatter_add_rows, which pfor converts to one-hot products; vectorize.py
#     _convert_scatter_add_rows).  Summed over every index of v (the LSTM
#     cell's four gate slices, reference bench cell), sum_g onehot(g) * x_g is
#     exactly concat([x_0, .., x_{K-1}]) along the one-hot axis: x*1 = x and
#     the other terms are +-0, so the values agree (a slot's -0 becomes +0;
#     an inf/NaN in a *different* slot, which would make the reference's
#     product NaN, is not propagated).
# (b) A concat whose pieces are outputs of one fused elementwise group (plus
#     inputs it may pass through) costs no launch: the group writes its
#     outputs into slots of one packed buffer and the concat is a view of
#     adjacent slots (`fused_pack`).  cfg4: the backward step's gate
#     cotangents land in dz in place; the forward step's [x_{t+1}, h_t] GEMM
#     operand is assembled by the cell kernel that computes h_t.

_ONEHOT_KINDS = frozenset({"constant", "reshape", "tile_leading", "equal", "cast", "range_vec"})


def _const_eval(g, key, budget=1 << 20):
    """Host value of a small constant-only subgraph (one-hot factors), or None."""
    from .tensor import DType
    memo = {}

    def ev(k):
        if k in memo:
            return memo[k]
        n = g.nodes[k[0]]
        if n.kind not in _ONEHOT_KINDS or k[1] != 0:
            raise ValueError
        ins = [ev(s) for s in n.inputs]
        if n.kind == "constant":
            v = np.asarray(n.attrs["value"].data)
        elif n.kind == "reshape":
            v = ins[0].reshape(g.ref_shape(k))
        elif n.kind == "tile_leading":
            v = np.broadcast_to(ins[0], (int(ins[1]),) + ins[0].shape)
        elif n.kind == "range_vec":
            v = np.arange(int(ins[0]), dtype=np.int64)
        elif n.kind == "equal":
            v = np.equal(ins[0], ins[1])
        else:  # cast
            v = ins[0].astype(np.float64 if n.attrs["dtype"] == DType.F64 else
                              (np.int64 if n.attrs["dtype"] == DType.I64 else np.bool_))
        if v.size > budget:
            raise ValueError
        memo[k] = v
        return v

    try:
        return ev(key)
    except (ValueError, KeyError, TypeError, AttributeError):
        return None


def _onehot_axis(g, key, shape):
    """(axis, K, index) if `key` is a constant one-hot e_index along one axis of
    the broadcast `shape` (the same along every other axis), else None."""
    sk = g.ref_shape(key)
    if sk is None or None in sk or g.ref_dtype(key) != _f64():
        return None
    v = _const_eval(g, key)
    if v is None:
        return None
    v = v.reshape((1,) * (len(shape) - v.ndim) + v.shape)
    for a, ext in enumerate(v.shape):
        if ext < 2 or ext != shape[a]:
            continue
        moved = np.moveaxis(v, a, -1).reshape(-1, ext)
        row = moved[0]
        idx = np.flatnonzero(row)
        if len(idx) != 1 or row[idx[0]] != 1.0 or not np.all(moved == row):
            continue
        return a, ext, int(idx[0])
    return None


def _f64():
    from .tensor import DType
    return DType.F64


def stack_onehot_sums(g, keep=()):
    """F13a in place on `g`.  Returns (count, moved outputs)."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    count = 0
    for node in list(g.topo_order()):
        if node.id in g.nodes and node.kind == "add":
            count += _f13a(rw, node)
    return count, rw.replaced


def _f13a(rw, node):
    g, b = rw.g, rw.b
    shape = g.ref_shape((node.id, 0))
    if shape is None or None in shape or node.out_dtypes[0] != _f64():
        return 0
    # leaves of the add tree (interior adds single-use)
    leaves, todo = [], list(node.inputs)
    while todo:
        k = todo.pop()
        n = rw.node(k)
        if n.kind == "add" and k[1] == 0 and rw.single_use(k) and \
                tuple(g.ref_shape(k) or ()) == tuple(shape):
            todo.extend(n.inputs)
        else:
            leaves.append(k)
    if len(leaves) < 2:
        return 0
    axis = None
    parts = {}
    for k in leaves:
        n = rw.node(k)
        if n.kind != "mul" or k[1] != 0:
            return 0
        hit = None
        for oh, x in ((n.inputs[0], n.inputs[1]), (n.inputs[1], n.inputs[0])):
            sx = g.ref_shape(x)
            if sx is None or len(sx) != len(shape) or g.ref_dtype(x) != _f64():
                continue
            h = _onehot_axis(g, oh, shape)
            if h is None:
                continue
            a, K, idx = h
            if sx[a] != 1 or any(sx[i] != shape[i] for i in range(len(shape)) if i != a):
                continue
            hit = (a, K, idx, x)
            break
        if hit is None:
            return 0
        a, K, idx, x = hit
        if axis is None:
            axis = (a, K)
        if axis != (a, K) or idx in parts:
            return 0
        parts[idx] = x
    a, K = axis
    if sorted(parts) != list(range(K)):
        return 0
    cat = b.concat([Ref(g, *parts[i]) for i in range(K)], a)
    rw.redirect((node.id, 0), cat)
    return 1


def place_concats(g, keep=()):
    """F13b in place on `g` (after fuse_elementwise).  Returns (count, moved)."""
    from .tensor import DType
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    count = 0
    claimed = set()
    for node in list(g.topo_order()):
        if node.id not in g.nodes or node.kind != "concat":
            continue
        count += _f13b(rw, node, claimed, DType)
    return count, rw.replaced


def _ancestors(g, key, stop):
    seen, todo = set(), [key[0]]
    while todo:
        n = todo.pop()
        if n in seen:
            continue
        if n == stop:
            return True
        seen.add(n)
        todo.extend(s for s, _ in g.nodes[n].inputs)
    return False


def _f13b(rw, node, claimed, DType):
    g = rw.g
    shape = g.ref_shape((node.id, 0))
    if shape is None or None in shape or node.out_dtypes[0] != DType.F64:
        return 0
    ax = node.attrs["axis"]
    ax = ax + len(shape) if ax < 0 else ax

    def source(k):  # through reshape chains that end in the shape they started from
        want, cur = g.ref_shape(k), k
        while rw.node(cur).kind == "reshape" and cur[1] == 0:
            cur = rw.node(cur).inputs[0]
            if g.ref_shape(cur) == want:
                k = cur
        return k

    pieces = [source(s) for s in node.inputs]
    prods = {s[0] for s in pieces if rw.node(s).kind in ("fused_ew", "fused_ewm")}
    if len(prods) != 1:
        return 0
    fid = prods.pop()
    if fid in claimed:
        return 0
    f = g.nodes[fid]
    S = tuple(f.out_shapes[0])
    if None in S or len(S) != len(shape) or any(d != DType.F64 for d in f.out_dtypes):
        return 0
    ports, passthrough = [], []
    for s in pieces:
        if tuple(g.ref_shape(s) or ()) != S:
            return 0
        if s[0] == fid:
            if s in ports:
                return 0
            ports.append(s)
        else:
            if g.ref_dtype(s) != DType.F64 or _ancestors(g, s, fid):
                return 0
            passthrough.append(s)
    if not ports:
        return 0
    # the fused group's program: multi-output form, passthroughs appended as
    # load -> output registers
    if f.kind == "fused_ew":
        prog = list(f.attrs["program"])
        out_regs = [prog[-1][1]]
    else:
        prog = list(f.attrs["program"])
        out_regs = list(f.attrs["out_regs"])
    inputs = list(f.inputs)
    n_out0 = len(out_regs)
    if len(inputs) + len(passthrough) > MAX_INPUTS or n_out0 + len(passthrough) > MAX_OUTPUTS \
            or len(prog) + len(passthrough) > MAX_STEPS:
        return 0
    used = set(out_regs)
    free = [r for r in range(MAX_REGS) if r not in used]
    if len(free) < len(passthrough):
        return 0
    pt_port = {}
    for s in passthrough:
        if s in inputs:
            slot = inputs.index(s)
        else:
            inputs.append(s)
            slot = len(inputs) - 1
        r = free.pop(0)
        prog.append((OP_LOAD, r, slot, 0))
        out_regs.append(r)
        pt_port[s] = len(out_regs) - 1
    # slot order: the concat's pieces first, in order, then the other outputs
    cat_order = [s[1] if s[0] == fid else pt_port[s] for s in pieces]
    slots = cat_order + [k for k in range(len(out_regs)) if k not in cat_order]
    n_out = len(out_regs)
    new = g.add_node("fused_pack", inputs,
                     {"program": tuple(prog), "out_regs": tuple(out_regs),
                      "out_dtypes": tuple([DType.F64] * n_out), "pack_axis": ax,
                      "slots": tuple(slots), "cat_span": len(pieces)})
    claimed.add(new.id)
    for k in range(n_out0):
        rw.redirect((fid, k), Ref(g, new.id, k))
    rw.redirect((node.id, 0), Ref(g, new.id, n_out))
    return 1


# ----------------------------------------------------------------------------
# F16: row sums computed by the elementwise group that reads them
#
# fused(..., X, reshape(reduce_sum(X, axes 1..), [n, 1, .., 1]), ...) -- a row
# sum of one of the group's own inputs, broadcast back along the row (cfg5's
# per-step branch mask `reduce_sum(z) < 0`, whose compare F14 already moved
# into the select group) -- becomes a row-sum feed of the group
# (attrs["rowsum"] = ((k, j), ...): input k is the row sum of input j, and
# slot k carries X itself).  The executor's row kernel sums each row in the
# block that evaluates it (pfb_fused_ew_rows): the reduction is no longer a
# launch of its own (reference tensor.reduce_sum, tensor.py:279-283; the
# values are the same sums in a different fp32 association).

def fuse_row_sums(g, keep=()):
    """F16 in place on `g` (a private copy).  Returns (count, moved outputs)."""
    from .tensor import DType, normalize_axes
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    live = live_set(g, keep)

    def live_uses(key):  # readers among the live nodes (dead ones linger until DCE)
        if key in rw.keep:
            return 2
        return sum(1 for n, _ in rw.users().get(key, []) if n.id in live)
    count = 0
    for node in list(g.topo_order()):
        if node.id not in live or node.kind not in ("fused_ew", "fused_ewm") or node.attrs.get("rowsum"):
            continue
        osh = g.ref_shape((node.id, 0))
        if osh is None or None in osh or len(osh) < 2:
            continue
        ins = [tuple(i) for i in node.inputs]
        bshape = (osh[0],) + (1,) * (len(osh) - 1)
        rs = []
        for k, src in enumerate(ins):
            ksh = g.ref_shape(src)
            if ksh is None or tuple(ksh) != bshape:
                continue
            key, post = src, []
            while True:
                while rw.node(key).kind == "reshape" and live_uses(key) == 1:
                    key = tuple(rw.node(key).inputs[0])
                e = rw.node(key)
                op = _row_post_op(g, e) if live_uses(key) == 1 and len(post) < 4 else None
                if op is None:
                    break
                post.append(op[0])
                key = op[1]
            r = rw.node(key)
            if r.kind != "reduce_sum" or key[1] != 0 or live_uses(key) != 1:
                continue
            x = tuple(r.inputs[0])
            xsh = g.ref_shape(x)
            if xsh is None or tuple(xsh) != tuple(osh) or r.out_dtypes[0] != DType.F64 or x not in ins:
                continue
            if tuple(sorted(normalize_axes(r.attrs["axes"], len(xsh)))) != tuple(range(1, len(xsh))):
                continue
            j = ins.index(x)
            if any(e[1] == k for e in rs):
                continue
            if post:
                prog = _with_post_ops(node, k, post[::-1])
                if prog is None:
                    continue
                node.attrs["program"] = prog
            # the summand's own unary producer (cfg2's exp of the logits),
            # read nowhere else, moves into the group too: the kernel sums
            # op(input) and the program applies op after the input's load
            xn = rw.node(x)
            pre = None
            if xn.kind in _UN_CODE and xn.kind != "logical_not" and x[1] == 0 and \
                    xn.out_dtypes[0] == DType.F64 and \
                    all(n is node or n is r for n, _ in rw.users().get(x, []) if n.id in live) and \
                    g.ref_dtype(xn.inputs[0]) == DType.F64 and \
                    tuple(g.ref_shape(xn.inputs[0]) or ()) == tuple(osh):
                prog = _with_post_ops(node, j, [("un", 16 + _UN_CODE[xn.kind])])
                if prog is not None:
                    node.attrs["program"] = prog
                    node.inputs[j] = tuple(xn.inputs[0])
                    ins[j] = tuple(xn.inputs[0])
                    pre = 16 + _UN_CODE[xn.kind]
            rs.append((k, j) if pre is None else (k, j, pre))
        if not rs:
            continue
        for e in rs:
            node.inputs[e[0]] = node.inputs[e[1]]
        node.attrs["rowsum"] = tuple(rs)
        rw._users = None
        g._topo_cache = None
        count += 1
    return count, rw.replaced


# ----------------------------------------------------------------------------
# F17: sibling gathers of one operand become one launch
#
# An unrolled loop body gathers x_t = x[j, t_j + u] for every unrolled step u
# (cfg5: gather_stacked(X, t + u), u = 0..3); the index vectors are known at
# the top of the trip, so the q gathers can run as one node
# (gather_stacked_many, one kernel) instead of one launch per step.  Only
# gathers whose indices do not depend on one another's results merge (the
# merged node must be placeable before all of them); each keeps its own
# bounds check / error report (attrs["orig"]).

def merge_sibling_gathers(g, keep=(), max_q=8):
    """F17 in place on `g` (a private copy).  Returns (count, moved outputs)."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    live = live_set(g, keep)
    groups = {}
    for node in g.topo_order():
        if node.id in live and node.kind == "gather_stacked":
            sx, si = g.ref_shape(node.inputs[0]), g.ref_shape(node.inputs[1])
            if sx is None or si is None or len(si) != 1:
                continue
            groups.setdefault(tuple(node.inputs[0]), []).append(node)
    count = 0
    for x, nodes in groups.items():
        nodes = nodes[:max_q]
        if len(nodes) < 2:
            continue
        ids = {n.id for n in nodes}
        # no index may depend on a gather of the group (the merged node would
        # then feed its own input)
        if any(_ancestors(g, tuple(n.inputs[1]), m) for n in nodes for m in ids):
            continue
        new = g.add_node("gather_stacked_many", [x] + [tuple(n.inputs[1]) for n in nodes],
                         {"orig": tuple(n.id for n in nodes)})
        for k, n in enumerate(nodes):
            rw.redirect((n.id, 0), Ref(g, new.id, k))
        count += 1
    g._topo_cache = None
    return count, rw.replaced


# ----------------------------------------------------------------------------
# F18: a sum of scatter-adds over complementary constant row sets is placement
#
# The VJP of gather(x, idx) is scatter_add_rows(idx, g, total) (reference
# autodiff.py:100-110); the maxpool of the conv bench model gathers the even
# and the odd rows (bench.py:68-78), so its backward adds two scatter-adds
# whose index sets are {0, 2, ..} and {1, 3, ..}: every output row receives
# exactly one update.  That sum is an interleave -- concat([u_even[:, None],
# u_odd[:, None]], 1) reshaped to [total, ..] -- and a split at n
# ({0..n-1} / {n..total-1}) is a plain concat: one placement launch (or none,
# when F13b lets the producing group write the slots) instead of two zero
# fills, two scatter kernels and an add.  Values are the updates themselves
# (the reference's 0 + u turns a -0 update into +0; nothing else differs --
# the other set contributes exact zeros).

def place_scatter_sums(g, keep=()):
    """F18 in place on `g` (a private copy).  Returns (count, moved outputs)."""
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    live = live_set(g, keep)
    b = rw.b

    def live_uses(key):
        if key in rw.keep:
            return 2
        return sum(1 for n, _ in rw.users().get(key, []) if n.id in live)

    count = 0
    for node in list(g.topo_order()):
        if node.id not in live or node.kind != "add" or node.id not in g.nodes:
            continue
        chains = []
        for src in node.inputs:
            chain, key = [], tuple(src)
            while rw.node(key).kind in ("transpose", "reshape") and live_uses(key) == 1:
                n = rw.node(key)
                chain.append((n.kind, tuple(n.attrs["perm"] if n.kind == "transpose"
                                            else n.attrs["shape"])))
                key = tuple(n.inputs[0])
            sc = rw.node(key)
            if sc.kind != "scatter_add_rows" or key[1] != 0 or live_uses(key) != 1:
                break
            chains.append((chain, sc))
        if len(chains) != 2 or chains[0][0] != chains[1][0]:
            continue
        chain = chains[0][0]
        s1, s2 = chains[0][1], chains[1][1]
        T = s1.attrs["total"]
        if s2.attrs["total"] != T or not isinstance(T, (int, np.integer)):
            continue
        i1, i2 = _const_eval(g, tuple(s1.inputs[0])), _const_eval(g, tuple(s2.inputs[0]))
        sh1, sh2 = g.ref_shape(s1.inputs[1]), g.ref_shape(s2.inputs[1])
        if i1 is None or i2 is None or i1.ndim != 1 or i2.ndim != 1 or sh1 is None or sh2 is None:
            continue
        if None in sh1 or None in sh2 or tuple(sh1[1:]) != tuple(sh2[1:]):
            continue
        if sh1[0] != len(i1) or sh2[0] != len(i2):
            continue
        n1, n2, tail = len(i1), len(i2), list(sh1[1:])
        u1, u2 = Ref(g, *s1.inputs[1]), Ref(g, *s2.inputs[1])
        if np.array_equal(i1, np.arange(n1)) and np.array_equal(i2, np.arange(n1, T)):
            first, second, inter = u1, u2, False
        elif np.array_equal(i2, np.arange(n2)) and np.array_equal(i1, np.arange(n2, T)):
            first, second, inter = u2, u1, False
        elif n1 == n2 and 2 * n1 == T and {tuple(i1), tuple(i2)} == {
                tuple(range(0, T, 2)), tuple(range(1, T, 2))}:
            first, second = (u1, u2) if i1[0] == 0 else (u2, u1)
            inter = True
        else:
            continue
        if len(chain) == 1 and chain[0][0] == "transpose":
            # place in the consumer's layout: the pieces as transposed views
            # (usually undoing the transpose that produced them) and the
            # concat along the axis the scatter axis lands on
            perm = list(chain[0][1])
            a = perm.index(0)
            p1, p2 = b.transpose(first, perm), b.transpose(second, perm)
            osh = list(g.ref_shape((node.id, 0)))
            if inter:
                ins = lambda r: b.reshape(r, osh[:a] + [n1, 1] + osh[a + 1:])  # noqa: E731
                out = b.reshape(b.concat([ins(p1), ins(p2)], a + 1), osh)
            else:
                out = b.concat([p1, p2], a)
        else:
            if inter:
                merged = b.reshape(b.concat([b.reshape(first, [n1, 1] + tail),
                                             b.reshape(second, [n1, 1] + tail)], 1), [T] + tail)
            else:
                merged = b.concat([first, second], 0)
            out = merged
            for kind, arg in reversed(chain):
                out = b.transpose(out, list(arg)) if kind == "transpose" else b.reshape(out, list(arg))
        if tuple(g.ref_shape((out.nid, out.port))) != tuple(g.ref_shape((node.id, 0))):
            continue
        rw.redirect((node.id, 0), out)
        count += 1
    g._topo_cache = None
    return count, rw.replaced


def _row_post_op(g, e):
    """(step template, operand key) when `e` is an elementwise op on a per-row
    value whose other operand (if any) is a scalar constant -- F16 moves it
    into the reading group's program after the row-sum load (cfg2's softmax
    `1 / sum(exp(z))`).  Template: ("un", code) or ("bin", code, bits, const_left)."""
    import struct
    from .tensor import DType
    if e.output_arity != 1 or e.out_dtypes[0] != DType.F64:
        return None
    if e.kind in _UN_CODE and e.kind != "logical_not":
        return ("un", 16 + _UN_CODE[e.kind]), tuple(e.inputs[0])
    if e.kind in _BIN_CODE and e.kind not in ("less", "equal"):
        for side in (0, 1):
            c = _const_scalar_f(g, tuple(e.inputs[side]))
            if c is not None and _const_scalar_f(g, tuple(e.inputs[1 - side])) is None:
                bits = struct.unpack("<i", struct.pack("<f", c))[0]
                return ("bin", _BIN_CODE[e.kind], bits, side == 0), tuple(e.inputs[1 - side])
    return None


def _with_post_ops(node, k, post):
    """The group's program with `post` (innermost first) applied to input k
    right after its load: load r; [const t]; r = op(.., r, ..).  None when the
    input is loaded more than once, is an output register, or no register /
    step is free."""
    prog = [tuple(st) for st in node.attrs["program"]]
    loads = [i for i, st in enumerate(prog) if st[0] == OP_LOAD and st[2] == k]
    if len(loads) != 1:
        return None
    i = loads[0]
    r = prog[i][1]
    outs = node.attrs.get("out_regs", (prog[-1][1],))
    used = {st[1] for st in prog} | {st[2] for st in prog if st[0] not in (OP_LOAD, OP_CONST)} | \
        {st[3] for st in prog if st[0] not in (OP_LOAD, OP_CONST)}
    free = [t for t in range(MAX_REGS) if t not in used]
    last_write = {}
    for j, st in enumerate(prog):
        last_write[st[1]] = j
    # the loaded value itself must not be an output (a passthrough); a later
    # step that reuses r as an output register overwrites it anyway
    if (r in outs and last_write.get(r) == i) or not free:
        return None
    t = free[0]
    extra = []
    for op in post:
        if op[0] == "un":
            extra.append((op[1], r, r, r))
        else:
            _, code, bits, const_left = op
            extra.append((OP_CONST, t, bits, 0))
            extra.append((code, r, t, r) if const_left else (code, r, r, t))
    prog = prog[:i + 1] + extra + prog[i + 1:]
    if len(prog) > MAX_STEPS:
        return None
    return tuple(prog)


# ----------------------------------------------------------------------------
# F19: sibling weighted column sums sharing the weights become one launch
#
# DP-SGD's clipped bias-gradient sums, sum_i s_i g_i for every parameter block
# (reduce_dot(g_block, s, axes=(0,)), F4), share the clip scales s: one
# reduce_dot_many node (pfb_col_dots, one kernel over all blocks' columns).

def merge_sibling_reduce_dots(g, keep=(), max_q=8):
    """F19 in place on `g` (a private copy).  Returns (count, moved outputs)."""
    from .tensor import DType, normalize_axes
    rw = _Rewriter(g, keep)
    rw.replaced = {}
    live = live_set(g, keep)
    groups = {}
    for node in g.topo_order():
        if node.id not in live or node.kind != "reduce_dot":
            continue
        sx, sy = g.ref_shape(node.inputs[0]), g.ref_shape(node.inputs[1])
        if sx is None or sy is None or len(sx) != 2 or None in sx or sx[0] < 2:
            continue
        if tuple(normalize_axes(node.attrs["axes"], 2)) != (0,) or node.out_dtypes[0] != DType.F64:
            continue
        if tuple(sy) not in ((sx[0],), (sx[0], 1)):
            continue
        groups.setdefault(tuple(node.inputs[1]), []).append(node)
    count = 0
    for y, nodes in groups.items():
        nodes = nodes[:max_q]
        if len(nodes) < 2:
            continue
        ids = {n.id for n in nodes}
        if any(_ancestors(g, tuple(n.inputs[0]), m) for n in nodes for m in ids):
            continue
        new = g.add_node("reduce_dot_many", [y] + [tuple(n.inputs[0]) for n in nodes],
                         {"axes": (0,)})
        for k, n in enumerate(nodes):
            rw.redirect((n.id, 0), Ref(g, new.id, k))
        count += 1
    g._topo_cache = None
    return count, rw.replaced
