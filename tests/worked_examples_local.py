"""The reference's worked-example loop bodies (reference tests/worked_examples.py),
built with this package's API.  Seeds and shapes match, so outputs can be
compared against the goldens the reference produced."""

import numpy as np

from paper_1903_04243_b200 import GraphBuilder


def _graph(body, n, consts=()):
    b = GraphBuilder()
    refs = [b.const(c) for c in consts]
    b.graph.set_outputs(b.parfor(lambda bb, i: body(bb, i, *refs), n))
    return b.graph


def pairwise_sum_diff():
    def body(bb, i, a, c):
        x, y = bb.gather(a, i), bb.gather(c, i)
        return [bb.add(x, y), bb.sub(x, y)]
    return _graph(body, 4, [np.array([1.0, 2.0, 3.0, 4.0]), np.array([10.0, 20.0, 30.0, 40.0])])


def gather_identity():
    return _graph(lambda bb, i, X: [bb.gather(X, i)], 4, [np.arange(12.0).reshape(4, 3)])


def matmul_fold():
    r = np.random.default_rng(7)
    X, Y = r.standard_normal((4, 2, 3)), r.standard_normal((3, 5))
    return _graph(lambda bb, i, X, Y: [bb.matmul(bb.gather(X, i), bb._imp(Y))], 4, [X, Y])


def conv2d_fold():
    r = np.random.default_rng(8)
    X, F = r.standard_normal((3, 1, 4, 4, 1)), r.standard_normal((2, 2, 1, 2))
    return _graph(lambda bb, i, X, F: [bb.conv2d(bb.gather(X, i), bb._imp(F))], 3, [X, F])


def reduce_sum_renumber():
    X = np.random.default_rng(9).standard_normal((4, 2, 3, 2))
    return _graph(lambda bb, i, X: [bb.reduce_sum(bb.gather(X, i), [1, -1])], 4, [X])


def concat_shift():
    r = np.random.default_rng(10)
    A, B = r.standard_normal((3, 2, 4)), r.standard_normal((3, 3, 4))
    return _graph(lambda bb, i, A, B: [bb.concat([bb.gather(A, i), bb.gather(B, i)], 0)], 3,
                  [A, B])


def broadcast_reshape():
    r = np.random.default_rng(11)
    X, Y = r.standard_normal((3, 2)), r.standard_normal((4, 2))
    return _graph(lambda bb, i, X, Y: [bb.add(bb._imp(X), bb.gather(Y, i))], 4, [X, Y])


def cond_example():
    def body(bb, i):
        (r,) = bb.cond(bb.less(i, bb.i64(2)),
                       lambda tb: [tb.mul(tb._imp(i), tb.i64(2))],
                       lambda eb: [eb.add(eb._imp(i), eb.i64(10))])
        return [r]
    return _graph(body, 4)


def while_example():
    def body(bb, i):
        (r,) = bb.while_loop([bb.i64(0)], lambda cb, car: cb.less(car[0], cb._imp(i)),
                             lambda wb, car: [wb.add(car[0], wb.i64(1))])
        return [r]
    return _graph(body, 5)
