"""CPU: predicated (masked) cond/while conversion gives the reference's values.

Policy(masked_control=True) replaces the reference's active-set compaction
(where_true / gather / scatter_rows / complement, data-dependent sizes) with
fixed-shape predication (select), so loop bodies are CUDA-graph capturable.
Checked here against the reference's own outputs (goldens) on the oracle."""

import numpy as np
import pytest

from oracle import OracleExecutor
from paper_1903_04243_b200 import GraphBuilder, Policy, pfor, vectorize_graph
from paper_1903_04243_b200 import workloads as WL
from test_oracle_golden import PROGRAM_CASES

MASKED = Policy(masked_control=True)


def _kinds(g):
    out = set()
    for n in g.nodes.values():
        out.add(n.kind)
        if n.block is not None:
            for sg in n.block.subgraphs.values():
                out |= _kinds(sg)
    return out


@pytest.mark.parametrize("unroll", [1, 3])
@pytest.mark.parametrize("name", ["cfg5", "cfg5_mid"])
def test_masked_cfg5_matches_reference(name, unroll, golden):
    cfg, kw = PROGRAM_CASES[name]
    from paper_1903_04243_b200 import b200_registry
    reg = b200_registry()
    api = WL.this_api()
    policy = Policy(masked_control=True, unroll=unroll)
    orig = api.pfor
    api.pfor = lambda b, body, n, **k: orig(b, body, n, policy=policy, **k)
    w = WL.cfg5(api, registry=reg, **kw)
    kinds = _kinds(w.graph)
    assert not {"where_true", "complement", "scatter_rows"} & kinds
    outs = OracleExecutor(w.graph).run(feeds=w.feeds)
    for j, o in enumerate(outs):
        np.testing.assert_allclose(o.data, golden["programs"][f"{name}/out/{j}"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["cond_example", "while_example"])
def test_masked_worked_examples(name, golden):
    import worked_examples_local as WE
    g2, diags = vectorize_graph(getattr(WE, name)(), policy=MASKED)
    assert any(e[2] == "masked" for e in diags.entries)
    for j, o in enumerate(OracleExecutor(g2).run()):
        np.testing.assert_array_equal(o.data, golden["programs"][f"we_{name}/out/{j}"])


def _nested_program(policy):
    """while inside cond inside while, per-example data-dependent gathers."""
    r = np.random.default_rng(3)
    X = r.standard_normal((6, 5))
    L = np.array([0, 1, 5, 3, 2, 4])
    b = GraphBuilder()
    cX, cL = b.const(X), b.const(L)

    def body(bb, i):
        x = bb.gather(cX, i)
        li = bb.gather(cL, i)

        def wcond(cb, car):
            return cb.less(car[0], cb._imp(li))

        def wbody(wb, car):
            t, acc = car
            v = wb.gather(wb._imp(x), t)
            pos = wb.less(wb.f64(0.0), v)
            (inc,) = wb.cond(pos, lambda tb: [tb.mul(tb._imp(v), tb.f64(2.0))],
                             lambda eb: [eb.neg(eb._imp(v))])
            return [wb.add(t, wb.i64(1)), wb.add(acc, inc)]

        _, acc = bb.while_loop([bb.i64(0), bb.f64(0.0)], wcond, wbody)
        return [acc]

    outs = pfor(b, body, 6, policy=policy)
    b.graph.set_outputs(outs)
    return b.graph


def test_masked_nested_matches_compaction_and_loop():
    want = OracleExecutor(_nested_program(None)).run()[0].data
    got = OracleExecutor(_nested_program(MASKED)).run()[0].data
    np.testing.assert_array_equal(got, want)
    g = GraphBuilder()
    loop = _nested_program.__wrapped__ if hasattr(_nested_program, "__wrapped__") else None
    assert loop is None
    X = np.random.default_rng(3).standard_normal((6, 5))
    L = [0, 1, 5, 3, 2, 4]
    manual = [sum((2 * v if v > 0 else -v) for v in X[i, :L[i]]) for i in range(6)]
    np.testing.assert_allclose(got, manual, rtol=0, atol=1e-12)
    del g


def test_passes_inside_loop_bodies_preserve_values(golden):
    """optimize() also fuses inside cond / while sub-graphs (predicated cfg5 body)."""
    from paper_1903_04243_b200.passes import optimize
    _, kw = PROGRAM_CASES["cfg5_mid"]
    w = WL.cfg5(WL.this_api(), masked=True, unroll=2, **kw)
    keys = [tuple(o) for o in w.graph.outputs]
    g2, m = optimize(w.graph, keys)
    fused = [n for n in g2.nodes.values() if n.block is not None
             for sg in n.block.subgraphs.values() for x in sg.nodes.values()
             if x.kind == "fused_ew"]
    assert fused
    got = OracleExecutor(g2).run(feeds=w.feeds, outputs=[g2.out(*m[k]) for k in keys])
    np.testing.assert_allclose(got[0].data, golden["programs"]["cfg5_mid/out/0"], rtol=0,
                               atol=1e-12)
