"""Error and aliasing semantics the B200 additions must keep (advisor
findings, round 1): the stacked x stacked gather converter raises like the
reference on out-of-range per-iteration indices, loop-invariant code motion
never hoists an op that can raise out of a zero-trip loop, shard= refuses
bodies with random draws, and captured loop bodies whose results alias their
inputs (passthrough, permutation, transposed view) stay correct on replay."""

import numpy as np
import pytest

from oracle import OracleExecutor
from paper_1903_04243_b200 import GraphBuilder, pfor, reference_registry
from paper_1903_04243_b200 import errors as E
from paper_1903_04243_b200.passes import optimize


def _stacked_gather_graph(indices, registry=None):
    b = GraphBuilder()
    X = b.const(np.arange(12, dtype=np.float64).reshape(3, 2, 2))
    I = b.const(np.asarray(indices, dtype=np.int64))

    def body(bb, i):
        x = bb.gather(X, i)       # stacked [2, 2]
        k = bb.gather(I, i)       # stacked scalar index
        return [bb.gather(x, k)]  # x[i][I[i]]

    kw = {} if registry is None else {"registry": registry}
    (out,) = pfor(b, body, 3, **kw)
    b.graph.set_outputs([out])
    return b.graph


@pytest.mark.parametrize("registry", [None, "reference"])
def test_stacked_gather_out_of_range_raises(registry):
    reg = reference_registry() if registry else None
    g = _stacked_gather_graph([0, 2, 1], reg)
    with pytest.raises(E.ExecError) as ei:
        OracleExecutor(g).run()
    assert isinstance(ei.value.cause, E.IndexOutOfBounds)
    assert "out of range [0, 2)" in str(ei.value.cause)


def test_stacked_gather_in_range_matches_reference_registry():
    got = OracleExecutor(_stacked_gather_graph([0, 1, 1])).run()[0].data
    want = OracleExecutor(_stacked_gather_graph([0, 1, 1], reference_registry())).run()[0].data
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(got, [[0, 1], [6, 7], [10, 11]])


def _zero_trip_gather_graph(trips):
    """while t < trips: acc = acc + gather(X, [5]) -- X has 2 rows, so the
    body raises whenever it runs; with trips = 0 it never runs."""
    b = GraphBuilder()
    X = b.const(np.zeros((2, 2)))
    idx = b.const(np.asarray([5], dtype=np.int64))

    def cond(cb, car):
        return cb.less(car[0], cb.i64(trips))

    def step(wb, car):
        t, acc = car
        return [wb.add(t, wb.i64(1)), wb.add(acc, wb.gather(wb._imp(X), wb._imp(idx)))]

    _, acc = b.while_loop([b.i64(0), b.const(np.zeros((1, 2)))], cond, step)
    b.graph.set_outputs([acc])
    return b.graph


def test_licm_keeps_raising_ops_inside_zero_trip_loops():
    g = _zero_trip_gather_graph(0)
    keys = [tuple(o) for o in g.outputs]
    g2, m = optimize(g, keys)
    (want,) = OracleExecutor(g).run()
    (got,) = OracleExecutor(g2).run(outputs=[g2.out(*m[k]) for k in keys])
    np.testing.assert_array_equal(got.data, want.data)
    np.testing.assert_array_equal(got.data, np.zeros((1, 2)))


def test_licm_still_raises_when_the_loop_runs():
    g = _zero_trip_gather_graph(2)
    keys = [tuple(o) for o in g.outputs]
    g2, m = optimize(g, keys)
    with pytest.raises(E.ExecError):
        OracleExecutor(g2).run(outputs=[g2.out(*m[k]) for k in keys])


def test_licm_hoists_in_range_constant_gathers():
    from paper_1903_04243_b200.passes import hoist_loop_invariants
    b = GraphBuilder()
    X = b.const(np.arange(6, dtype=np.float64).reshape(3, 2))
    idx = b.const(np.asarray([2, 0], dtype=np.int64))

    def step(wb, car):
        t, acc = car
        return [wb.add(t, wb.i64(1)), wb.add(acc, wb.gather(wb._imp(X), wb._imp(idx)))]

    _, acc = b.while_loop([b.i64(0), b.const(np.zeros((2, 2)))],
                          lambda cb, car: cb.less(car[0], cb.i64(3)), step)
    b.graph.set_outputs([acc])
    (want,) = OracleExecutor(b.graph).run()
    assert hoist_loop_invariants(b.graph) >= 1
    (got,) = OracleExecutor(b.graph).run()
    np.testing.assert_array_equal(got.data, want.data)


def test_shard_rejects_random_draws():
    b = GraphBuilder()

    def body(bb, i):
        return [bb.random_uniform((2,))]

    with pytest.raises(E.VectorizeError):
        pfor(b, body, 4, shard=(0, 2))


# ---------------------------------------------------------------------------
# GPU: captured loop bodies whose results alias their inputs

def _swap_loop(trips, transpose=False):
    """(a, b) -> (b, a) [or (b, a^T)] for `trips` trips, plus a counter."""
    b = GraphBuilder()
    A = b.const(np.arange(4, dtype=np.float64).reshape(2, 2))
    B = b.const(10 + np.arange(4, dtype=np.float64).reshape(2, 2))

    def step(wb, car):
        t, x, y = car
        return [wb.add(t, wb.i64(1)), wb.transpose(y, [1, 0]) if transpose else y, x]

    _, x, y = b.while_loop([b.i64(0), A, B], lambda cb, car: cb.less(car[0], cb.i64(trips)),
                           step)
    b.graph.set_outputs([x, y])
    return b.graph


@pytest.mark.gpu
@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("trips", [1, 2, 3, 5])
def test_captured_loop_with_aliasing_results(trips, transpose):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1903_04243_b200.executor import Executor
    g = _swap_loop(trips, transpose)
    want = [o.data for o in OracleExecutor(g).run()]
    ex = Executor(g)
    for _ in range(4):  # eager, capture (sub-graph or device loop), replays
        got = ex.run()
        for a, w in zip(got, want):
            np.testing.assert_array_equal(np.asarray(a.data, np.float64), w)
