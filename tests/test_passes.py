"""CPU: the post-vectorization fusions (passes.py) preserve values.

The rewritten graphs run on the oracle here; on the GPU the same rewrites run
inside the executor (tests/test_gpu_parity.py compares against goldens)."""

import numpy as np
import pytest

from oracle import OracleExecutor
from paper_1903_04243_b200 import workloads as WL
from paper_1903_04243_b200.passes import optimize


def _run_both(w):
    g = w.graph
    keys = [tuple(o) for o in g.outputs]
    g2, m = optimize(g, keys)
    want = OracleExecutor(g).run(feeds=w.feeds)
    got = OracleExecutor(g2).run(feeds=w.feeds, outputs=[g2.out(*m[k]) for k in keys])
    for a, b in zip(got, want):
        np.testing.assert_allclose(a.data, b.data, rtol=1e-10, atol=1e-12)
    return g, g2, m


def _kinds(g, roots):
    from paper_1903_04243_b200.executor import _Plan  # noqa: F401  (torch import)
    live, todo = set(), [r[0] for r in roots]
    while todo:
        n = todo.pop()
        if n in live:
            continue
        live.add(n)
        todo.extend(s for s, _ in g.nodes[n].inputs)
    return [g.nodes[n] for n in sorted(live)]


def test_f1_norm_and_clipped_sum_without_stacked_grads():
    w = WL.cfg2(WL.this_api(), n=6, model="mlp", d_h=16)
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    big = [n for n in live if n.kind == "matmul" and len(n.out_shapes[0]) == 3
           and n.out_shapes[0][1] == 784]
    assert not big, "the [n,784,16] per-example outer product must not be computed"


def test_f1_conv_model():
    _run_both(WL.cfg2(WL.this_api(), n=3, model="conv"))


def test_f2_outer_product_sum_becomes_one_gemm():
    w = WL.cfg4(WL.this_api(), n=3, steps=5, units=4)
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    k1 = [n for n in live if n.kind == "matmul" and len(n.out_shapes[0]) == 3
          and n.out_shapes[0][1:] == (8, 16)]
    assert len(k1) == 1, [n.out_shapes for n in k1]


@pytest.mark.parametrize("cfg,kw", [("cfg1", dict(batch=4, d_in=12, d_h=8, d_out=3)),
                                    ("cfg3", dict(width=16, out_dim=8)),
                                    ("cfg5", dict(n=5, max_len=6, units=4))])
def test_passes_neutral_elsewhere(cfg, kw):
    _run_both(WL.BUILDERS[cfg](WL.this_api(), **kw))


def test_f5_matmul_epilogues_and_f6_row_dots():
    """cfg2 MLP: forward GEMMs carry bias(+tanh) epilogues, the clipped-sum
    GEMMs the clip-factor kscale, and the six per-block |g_i|^2 reductions
    run as one row_dots node -- values unchanged (oracle)."""
    w = WL.cfg2(WL.this_api(), n=6, model="mlp", d_h=16)
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    eps = [n for n in live if n.kind == "matmul_ep"]
    assert any(n.attrs["act"] == "tanh" and n.attrs["has_bias"] for n in eps)
    assert sum(n.attrs["has_kscale"] for n in eps) == 2
    rd = [n for n in live if n.kind == "row_dots"]
    assert len(rd) == 1 and rd[0].attrs["n"] == 6
    assert not [n for n in live if n.kind == "reduce_dot" and len(n.out_shapes[0]) == 1
                and n.out_shapes[0][0] == 6 and len(g2.ref_shape(n.inputs[0])) > 1
                and n.attrs["axes"] != (0,)]


def test_f5_respects_multi_use_preactivation():
    """z = xW + b used twice (tanh and an output): only the bias is fused."""
    from paper_1903_04243_b200 import GraphBuilder
    from oracle import OracleExecutor as OE
    r = np.random.default_rng(0)
    b = GraphBuilder()
    x = b.const(r.standard_normal((5, 7)))
    W = b.const(r.standard_normal((7, 3)))
    bias = b.const(r.standard_normal((3,)))
    z = b.add(b.matmul(x, W), bias)
    y = b.tanh(z)
    b.graph.set_outputs([y, b.mul(z, z)])
    keys = [tuple(o) for o in b.graph.outputs]
    g2, mp = optimize(b.graph, keys)
    want = OE(b.graph).run()
    got = OE(g2).run(outputs=[g2.out(*mp[k]) for k in keys])
    for a_, b_ in zip(got, want):
        np.testing.assert_allclose(a_.data, b_.data, rtol=1e-12)
    eps = [n for n in g2.nodes.values() if n.kind == "matmul_ep"]
    assert len(eps) == 1 and eps[0].attrs["act"] is None and eps[0].attrs["has_bias"]


def test_f7_dual_matmul_sum_and_concat():
    """F7: z = x Wx + h Wh (cfg5's cell, inside the while body) becomes one
    matmul2; matmul(concat([a1, a2], -1), W) becomes matmul2 over row-split W
    views -- values unchanged (oracle)."""
    from paper_1903_04243_b200 import GraphBuilder
    from oracle import OracleExecutor as OE
    w = WL.cfg5(WL.this_api(), n=6, max_len=5, units=8, masked=True)
    _, g2, _ = _run_both(w)

    def count(gr):
        c = 0
        for n in gr.nodes.values():
            c += n.kind == "matmul2"
            if n.block is not None:
                c += sum(count(sg) for sg in n.block.subgraphs.values())
        return c
    assert count(g2) >= 1
    r = np.random.default_rng(1)
    b = GraphBuilder()
    a1, a2 = b.const(r.standard_normal((5, 3))), b.const(r.standard_normal((5, 4)))
    W, bias = b.const(r.standard_normal((7, 6))), b.const(r.standard_normal((6,)))
    b.graph.set_outputs([b.tanh(b.add(b.matmul(b.concat([a1, a2], 1), W), bias))])
    keys = [tuple(o) for o in b.graph.outputs]
    g3, mp = optimize(b.graph, keys)
    live = _kinds(g3, [mp[k] for k in keys])
    m2 = [n for n in live if n.kind == "matmul2"]
    assert len(m2) == 1 and m2[0].attrs["act"] == "tanh" and m2[0].attrs["has_bias"]
    assert not [n for n in live if n.kind == "concat"]
    want = OE(b.graph).run()
    got = OE(g3).run(outputs=[g3.out(*mp[k]) for k in keys])
    np.testing.assert_allclose(got[0].data, want[0].data, rtol=1e-12)


@pytest.mark.parametrize("kw", [dict(masked=True, unroll=4), dict(masked=True, unroll=1), dict()])
def test_f8_loop_invariants_leave_the_while_body(kw):
    """F8: no per-trip iota is left in cfg5's while body (the B200 registry's
    stacked gather needs none; a range_vec of a captured size would move out
    as a new capture) -- values unchanged."""
    w = WL.cfg5(WL.this_api(), n=6, max_len=5, units=8, **kw)
    g, g2, _ = _run_both(w)

    def body_kinds(gr):
        (wn,) = [n for n in gr.nodes.values() if n.kind == "while"]
        body = wn.block.subgraphs["body"]
        return wn, [n.kind for n in body.nodes.values()
                    if n.id in __import__("paper_1903_04243_b200.passes", fromlist=["x"]).live_set(
                        body, [tuple(o) for o in body.outputs])]
    w0, k0 = body_kinds(g)
    w1, k1 = body_kinds(g2)
    assert "range_vec" not in k1
    if "range_vec" in k0:  # hoisted values arrive as new captures
        assert len(w1.inputs) > len(w0.inputs)


def test_f3_leaves_constant_only_groups_alone():
    """A chain whose only inputs are scalar constants (reference randgen
    corpus case 123) is not turned into an input-less fused kernel."""
    import gzip
    import json
    import pathlib
    from paper_1903_04243_b200 import pfg
    from oracle import OracleExecutor as OE
    c = json.load(gzip.open(pathlib.Path(__file__).parent / "golden" / "corpus.json.gz",
                            "rt"))["123_1"]
    g = pfg.loads(c["vec"])
    keys = [tuple(o) for o in g.outputs]
    g2, mp = optimize(g, keys)

    def walk(gr):
        for n in gr.nodes.values():
            if n.kind in ("fused_ew", "fused_ewm"):
                assert n.inputs, n
            if n.block is not None:
                for sg in n.block.subgraphs.values():
                    walk(sg)
    walk(g2)
    from oracle import RngState, VariableStore
    want = OE(g, store=VariableStore(g.variables), rng=RngState(123)).run()
    got = OE(g2, store=VariableStore(g2.variables), rng=RngState(123)).run(
        outputs=[g2.out(*mp[k]) for k in keys])
    for a, b in zip(got, want):
        if a.data.size and not c["tainted"][0]:
            np.testing.assert_allclose(a.data, b.data, rtol=1e-12)


def test_f3_integer_domain_groups():
    """cfg5's masked loop body: the per-example counter / index / mask
    arithmetic (i64 and bool) fuses into `fused_int` programs -- values
    unchanged (oracle), integer results exact."""
    w = WL.cfg5(WL.this_api(), n=7, max_len=6, units=4, masked=True, unroll=2)
    _, g2, _ = _run_both(w)

    def kinds(gr):
        out = []
        for n in gr.nodes.values():
            out.append(n.kind)
            if n.block is not None:
                for sg in n.block.subgraphs.values():
                    out.extend(kinds(sg))
        return out
    assert "fused_int" in kinds(g2)


def test_f5_derivative_epilogue():
    """The tanh VJP's cotangent multiply cot * (1 - y^2) rides on the GEMM
    that produces cot (cfg2's dlogits W2^T; cfg3's backprop chain)."""
    w = WL.cfg2(WL.this_api(), n=6, model="mlp", d_h=16)
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    assert any(n.kind == "matmul_ep" and n.attrs.get("dop") == "dtanh" for n in live)
    w3 = WL.cfg3(WL.this_api(), width=16, out_dim=8)
    g, g3, m3 = _run_both(w3)
    live3 = _kinds(g3, [m3[tuple(o)] for o in g.outputs])
    assert any(n.kind == "matmul_ep" and n.attrs.get("dop") == "dtanh" for n in live3)


def _gate_grads(n=3, u=4, gates=(1,)):
    """per-example gradient of sum(square(W[g] * x_i)) over the gate rows
    `gates` of a [4, u] weight: the gradient of each gather(W, g) is a one-hot
    product (reference autodiff.py:100-110 -> vectorized one-hot)."""
    api = WL.this_api()
    r = np.random.default_rng(1)
    X0 = r.standard_normal((n, u)).astype(np.float32).astype(np.float64)
    W0 = r.standard_normal((4, u)).astype(np.float32).astype(np.float64)
    b = api.GraphBuilder()
    X = b.placeholder("x", api.DType.F64, (n, u))
    W = b.const(W0)

    def body(bb, i):
        xi = bb.reshape(bb.gather(X, i), [1, u])
        terms = [bb.mul(bb.reshape(bb.gather(bb._imp(W), bb.i64(gi)), [1, u]), xi) for gi in gates]
        acc = terms[0]
        for t in terms[1:]:
            acc = bb.add(acc, bb.tanh(t))
        loss = bb.reduce_sum(bb.square(acc), [0, 1])
        return api.gradient(bb.graph, loss, [bb._imp(W)], emit=bb)

    outs = api.pfor(b, body, n)
    b.graph.set_outputs(outs)
    return WL.Workload("gates", b.graph, {"x": X0}, n, "grads", {})


def test_f3_integer_group_ending_in_float_cast():
    """a one-hot factor cast(equal(t, range), f64) that F13a cannot turn into
    placement (one gate row of four): the integer compare and the cast to f64
    are one `fused_int` launch with an f64 output (values unchanged, oracle)."""
    from paper_1903_04243_b200.tensor import DType
    w = _gate_grads(gates=(1,))
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    fi = [n for n in live if n.kind == "fused_int"]
    assert any(DType.F64 in n.attrs["out_dtypes"] for n in fi)
    assert not any(n.kind == "cast" and n.out_dtypes[0] == DType.F64 and
                   g2.ref_dtype(n.inputs[0]) in (DType.BOOL, DType.I64) for n in live)


def test_f13a_onehot_sum_over_every_index_is_a_concat():
    """all four gate rows used: sum_g onehot(g) * dW_g is placement -- the
    live program has no one-hot product and no fused_int left (oracle values
    unchanged)."""
    w = _gate_grads(gates=(0, 1, 2, 3))
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    assert not [n for n in live if n.kind in ("fused_int", "equal")]


def test_f13_cfg4_steps_are_one_gemm_and_one_fused_launch():
    """cfg4 after F13: every time step is one GEMM and one fused launch in
    each direction -- the forward cell writes [x_{t+1}, h_t] (the next GEMM's
    operand) into its packed outputs, the backward cell writes the gate
    cotangents into dz in place; no per-step concat or one-hot stack."""
    T = 5
    w = WL.cfg4(WL.this_api(), n=3, steps=T, units=4)
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    kinds = [n.kind for n in live]
    packs = [n for n in live if n.kind == "fused_pack"]
    assert len(packs) == 2 * T - 1, kinds  # (step 0's operand has no cell before it)
    ew = [n for n in live if n.kind in ("fused_ew", "fused_ewm", "fused_int")]
    assert len(ew) <= 2, [n.kind for n in ew]  # bias-gradient sum, first cell's tail
    step_cats = [n for n in live if n.kind == "concat" and len(n.inputs) in (2, 4)]
    assert len(step_cats) == 1, [(n.kind, n.out_shapes) for n in step_cats]


def test_f9_backward_gemm_computes_only_live_columns():
    """cfg4: the backward GEMM dz_t Wg^T yields d[x_t, h]; only dh is live,
    so after F9 every per-step backward GEMM has N = units, not 2*units."""
    w = WL.cfg4(WL.this_api(), n=3, steps=4, units=4)
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    bwd = [n for n in live if n.kind == "matmul" and len(n.out_shapes[0]) == 2]
    assert bwd and all(n.out_shapes[0] == (3, 4) for n in bwd), [n.out_shapes for n in bwd]


def test_f10_cse_shares_the_backward_chain_of_the_jacobians():
    """cfg3 builds jacobian(y, W_l) for l = 0..3, each re-deriving the
    backward chain from y; after CSE the chain GEMMs run once: 3 forward
    GEMMs + 3 chain GEMMs (the reference emits 3 + 6)."""
    w = WL.cfg3(WL.this_api(), width=16, out_dim=8)
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    gemms = [n for n in live if n.kind in ("matmul", "matmul_ep")
             and g2.ref_shape(n.inputs[0])[-1] != 1]  # (K=1 outer products excluded)
    assert len(gemms) == 6, [(n.kind, n.out_shapes) for n in gemms]


def test_f11_long_add_chain_becomes_one_reduction_sharing_f2_operand():
    """cfg4's bias gradient sum_t dz_t (T-1 adds) becomes one reduce_sum over
    F2's K-major dz concat (shared through CSE): no add nodes remain."""
    w = WL.cfg4(WL.this_api(), n=3, steps=12, units=4)
    g, g2, m = _run_both(w)
    live = _kinds(g2, [m[tuple(o)] for o in g.outputs])
    assert not [n for n in live if n.kind == "add"]
    red = [n for n in live if n.kind == "reduce_sum"]
    assert len(red) == 1
    cat = g2.nodes[red[0].inputs[0][0]]
    assert cat.kind == "concat" and len(cat.inputs) == 12
    # the same concat feeds the F2 GEMM (through its K-major transpose view)
    readers = [n for n in live if any(tuple(s) == (cat.id, 0) for s in n.inputs)]
    assert len(readers) == 2


def test_f14_mask_compare_is_absorbed_into_the_select_group():
    """cfg5 (masked, unrolled): reshape(less(reduce_sum(z), 0), [n, 1, 1])
    becomes less(reshape(.), 0), which F3 evaluates inside the select group
    per element of [n, 1, units] -- the loop body keeps no standalone compare
    (oracle values unchanged)."""
    from paper_1903_04243_b200 import passes
    w = WL.cfg5(WL.this_api(), n=6, max_len=5, units=8, masked=True, unroll=2)
    g, g2, m = _run_both(w)
    bodies = [n.block.subgraphs["body"] for n in g2.nodes.values() if n.kind == "while"]
    assert bodies
    for body in bodies:
        live = passes.live_set(body, [tuple(o) for o in body.outputs])
        kinds = [body.nodes[i].kind for i in live]
        assert "less" not in kinds and kinds.count("fused_ew") >= 2, sorted(kinds)


def test_f16_row_sum_is_computed_by_the_select_group():
    """cfg5 (masked, unrolled): the per-step `reduce_sum(z)` whose only reader
    is the select group becomes a row-sum feed of that group (attrs
    "rowsum"): no reduce_sum over the step's rows stays live in the loop body
    (oracle values unchanged)."""
    from paper_1903_04243_b200 import passes
    w = WL.cfg5(WL.this_api(), n=6, max_len=5, units=8, masked=True, unroll=2)
    g, g2, m = _run_both(w)
    bodies = [n.block.subgraphs["body"] for n in g2.nodes.values() if n.kind == "while"]
    assert bodies
    for body in bodies:
        live = passes.live_set(body, [tuple(o) for o in body.outputs])
        nodes = [body.nodes[i] for i in live]
        fused = [n for n in nodes if n.kind == "fused_ew" and n.attrs.get("rowsum")]
        assert len(fused) == 2, sorted(n.kind for n in nodes)
        for f in fused:
            for k, j in f.attrs["rowsum"]:
                assert tuple(f.inputs[k]) == tuple(f.inputs[j])
        rows = [n for n in nodes if n.kind == "reduce_sum" and len(body.ref_shape(n.inputs[0])) == 3]
        assert not rows, rows


def test_f17_sibling_gathers_of_one_operand_merge():
    """cfg5 (masked, unrolled x4): the four per-step x_t gathers of a trip
    (indices known at the top of the trip) become one gather_stacked_many
    node (one launch); values unchanged on the oracle."""
    from paper_1903_04243_b200 import passes
    w = WL.cfg5(WL.this_api(), n=6, max_len=9, units=8, masked=True, unroll=4)
    g, g2, m = _run_both(w)
    bodies = [n.block.subgraphs["body"] for n in g2.nodes.values() if n.kind == "while"]
    assert bodies
    for body in bodies:
        live = passes.live_set(body, [tuple(o) for o in body.outputs])
        kinds = [body.nodes[i].kind for i in live]
        assert "gather_stacked" not in kinds and kinds.count("gather_stacked_many") == 1, kinds
        (gm,) = [body.nodes[i] for i in live if body.nodes[i].kind == "gather_stacked_many"]
        assert len(gm.attrs["orig"]) == 4


def test_f17_keeps_dependent_gathers_apart():
    """A gather whose index is computed from another gather's result of the
    same operand cannot merge with it."""
    from paper_1903_04243_b200 import passes
    from paper_1903_04243_b200.builder import GraphBuilder
    from paper_1903_04243_b200.tensor import DType
    b = GraphBuilder()
    x = b.placeholder("x", DType.F64, (4, 3, 4))
    i0 = b.placeholder("i", DType.I64, (4,))
    g1 = b.graph.add_node("gather_stacked", [x, i0], {})
    j = b.cast(b.reduce_sum(b.graph.out(g1.id, 0), [1]), DType.I64)
    g2 = b.graph.add_node("gather_stacked", [x, j], {})
    keys = [(g2.id, 0)]
    b.graph.set_outputs(keys)
    dst, mp = passes.optimize(b.graph, keys)
    live = passes.live_set(dst, [mp[k] for k in keys])
    kinds = [dst.nodes[n].kind for n in live]
    assert kinds.count("gather_stacked") == 2 and "gather_stacked_many" not in kinds


def test_masked_while_test_is_recognised_as_any():
    """The predicated while's loop test (vectorize._convert_while_masked:
    less(0, reduce_sum(cast(active, i64)))) survives the passes in the shape
    the device loop turns into one pfb_set_condition_any launch per trip."""
    from paper_1903_04243_b200.executor import _any_mask_test
    w = WL.cfg5(WL.this_api(), n=6, max_len=5, units=8, masked=True, unroll=2)
    keys = [tuple(o) for o in w.graph.outputs]
    g2, _ = optimize(w.graph, keys)
    loops = [n for n in g2.nodes.values() if n.kind == "while"]
    assert loops
    for n in loops:
        assert _any_mask_test(n.block.subgraphs["cond"]) == 0
        # a body is not a loop test
        assert _any_mask_test(n.block.subgraphs["body"]) is None


def test_f18_maxpool_backward_scatter_sums_become_placement():
    """cfg2 conv: the maxpool VJP's even-row + odd-row scatter-add sums
    (complementary constant row sets) become interleaving concats -- no
    scatter_add_rows and no add of scatter results stays live; oracle values
    unchanged."""
    from paper_1903_04243_b200 import passes
    w = WL.cfg2(WL.this_api(), n=3, model="conv")
    g, g2, m = _run_both(w)
    live = passes.live_set(g2, [m[tuple(o)] for o in g.outputs])
    kinds = [g2.nodes[i].kind for i in live]
    assert "scatter_add_rows" not in kinds, kinds
    assert kinds.count("concat") >= 2


def test_f18_split_scatter_sum_is_a_concat():
    """scatter_add(0..n-1, a) + scatter_add(n..T-1, b) == concat([a, b])."""
    from paper_1903_04243_b200 import passes
    from paper_1903_04243_b200.builder import GraphBuilder
    from paper_1903_04243_b200.tensor import DType
    from oracle import OracleExecutor
    b = GraphBuilder()
    x = b.placeholder("x", DType.F64, (5, 3))
    a = b.mul(b.gather(x, b.const(np.array([0, 1], np.int64))), b.f64(2.0))
    c = b.gather(x, b.const(np.array([2, 3, 4], np.int64)))
    s1 = b.graph.add_node("scatter_add_rows", [b.const(np.array([3, 4], np.int64)), a], {"total": 5})
    s2 = b.graph.add_node("scatter_add_rows", [b.const(np.array([0, 1, 2], np.int64)), c], {"total": 5})
    y = b.add(b.graph.out(s1.id, 0), b.graph.out(s2.id, 0))
    b.graph.set_outputs([y])
    keys = [tuple(o) for o in b.graph.outputs]
    g2, mp = passes.optimize(b.graph, keys)
    live = passes.live_set(g2, [mp[k] for k in keys])
    assert "scatter_add_rows" not in [g2.nodes[i].kind for i in live]
    xv = np.arange(15.0).reshape(5, 3)
    want = OracleExecutor(b.graph).run(feeds={"x": xv})[0].data
    got = OracleExecutor(g2).run(feeds={"x": xv}, outputs=[g2.out(*mp[keys[0]])])[0].data
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(want, np.concatenate([xv[2:5], 2 * xv[0:2]]))


def test_f16_softmax_exp_and_division_move_into_the_group():
    """cfg2 (mlp): the softmax's exp producer, row sum and 1/sum all run in
    the group that reads them (rowsum entry (k, j, exp)); no exp, no division
    and no row reduction stays live; oracle values unchanged."""
    from paper_1903_04243_b200 import passes
    w = WL.cfg2(WL.this_api(), n=4, model="mlp")
    g, g2, m = _run_both(w)
    live = passes.live_set(g2, [m[tuple(o)] for o in g.outputs])
    nodes = [g2.nodes[i] for i in live]
    kinds = [n.kind for n in nodes]
    assert "exp" not in kinds and "div" not in kinds, kinds
    ents = [e for n in nodes if n.attrs.get("rowsum") for e in n.attrs["rowsum"]]
    assert any(len(e) == 3 and e[2] == 16 + passes._UN_CODE["exp"] for e in ents), ents


def test_f19_clipped_bias_sums_share_one_launch():
    """cfg2 (mlp): the two clipped bias-gradient sums (reduce_dot with the
    shared clip scales) become one reduce_dot_many node; values unchanged."""
    from paper_1903_04243_b200 import passes
    w = WL.cfg2(WL.this_api(), n=4, model="mlp")
    g, g2, m = _run_both(w)
    live = passes.live_set(g2, [m[tuple(o)] for o in g.outputs])
    kinds = [g2.nodes[i].kind for i in live]
    assert "reduce_dot" not in kinds and kinds.count("reduce_dot_many") == 1, kinds
