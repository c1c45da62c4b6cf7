"""The BASELINE.json configurations as pfor programs.

Every builder takes an `api` namespace -- this package, or the reference
`pforvec` (used by tests/golden/make_golden.py to produce reference outputs)
-- so the *same* user program is built against both.  Builders return
`Workload(graph, feeds, units, meta)`: the graph's outputs are set, `feeds`
maps placeholder names to host arrays (the per-step inputs), `units` is how
many metric units (jacobian rows / per-example gradients / examples) one run
produces.

Synthetic data: one numpy default_rng(0) per config, tensors
drawn in the listed order, standard normal, scaled, rounded to fp32.  The
B200 path consumes the fp32 values; the f64 reference/oracle gets the same
values upcast.
"""

from __future__ import annotations

import types
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    graph: object
    feeds: dict
    units: int
    unit: str
    meta: dict = field(default_factory=dict)


def this_api():
    from .apps import jacobian, per_example_gradients, pfor
    from .autodiff import gradient
    from .builder import GraphBuilder
    from .tensor import DType
    return types.SimpleNamespace(GraphBuilder=GraphBuilder, pfor=pfor, jacobian=jacobian,
                                 gradient=gradient, per_example_gradients=per_example_gradients,
                                 DType=DType, supports_shard=True)


def reference_api(pforvec):
    return types.SimpleNamespace(GraphBuilder=pforvec.GraphBuilder, pfor=pforvec.pfor,
                                 jacobian=pforvec.jacobian, gradient=pforvec.gradient,
                                 per_example_gradients=pforvec.per_example_gradients,
                                 DType=pforvec.DType, supports_shard=False)


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def _pfor(api, b, body, n, shard, mode="vectorize", **kw):
    """`mode`: the reference's pfor modes (apps.py:28-45) -- "vectorize" (the
    hot path), "parfor" (per-iteration SIMD interpreter) and "fallback"
    (every op through the sequential while loop); the latter two are the
    CPU loop baselines bench.py times beside the device."""
    if mode != "vectorize":
        kw["mode"] = mode
    if shard is not None:
        return api.pfor(b, body, n, shard=shard, **kw)
    return api.pfor(b, body, n, **kw)


def _jac(api, b, y, w, shard, mode):
    kw = {} if mode == "vectorize" else {"mode": mode}
    if shard is not None:
        kw["shard"] = shard
    return api.jacobian(b, y, w, **kw)


# ----------------------------------------------------------------------------
# cfg1: jacobian of a 2-layer tanh MLP 784-256-10 wrt the input, batch 32

def _mlp_params(r, d_in, d_h, d_out):
    W1 = _f32(r.standard_normal((d_in, d_h)) / np.sqrt(d_in))
    b1 = _f32(0.1 * r.standard_normal((d_h,)))
    W2 = _f32(r.standard_normal((d_h, d_out)) / np.sqrt(d_h))
    b2 = _f32(0.1 * r.standard_normal((d_out,)))
    return W1, b1, W2, b2


def cfg1(api, batch=32, d_in=784, d_h=256, d_out=10, variant="batch", shard=None, registry=None,
         mode="vectorize"):
    """variant "batch": batch_jacobian [B,10,784] (pfor over examples of
    jacobian(y_b, x_b)); variant "full": jacobian(y, x) [B,10,B,784]."""
    r = np.random.default_rng(0)
    x0 = _f32(r.standard_normal((batch, d_in)))
    W1, b1, W2, b2 = _mlp_params(r, d_in, d_h, d_out)
    b = api.GraphBuilder()
    x = b.placeholder("x", api.DType.F64, (batch, d_in))
    cW1, cb1, cW2, cb2 = (b.const(v) for v in (W1, b1, W2, b2))
    kw = {} if registry is None else {"registry": registry}

    def net(bb, xin, rows):
        h = bb.tanh(bb.add(bb.matmul(bb.reshape(xin, [rows, d_in]), bb._imp(cW1)), bb._imp(cb1)))
        return bb.add(bb.matmul(h, bb._imp(cW2)), bb._imp(cb2))

    if variant == "full":
        y = net(b, x, batch)
        J = _jac(api, b, y, x, shard, mode)
        units = batch * d_out if shard is None else shard[1] - shard[0]
        b.graph.set_outputs([J])
    else:
        def body(bb, i):
            xb = bb.gather(x, i)
            yb = bb.reshape(net(bb, xb, 1), [d_out])
            return [_jac(api, bb, yb, xb, None, mode)]
        (J,) = _pfor(api, b, body, batch, shard, mode, **kw)
        b.graph.set_outputs([J])
        units = (batch if shard is None else shard[1] - shard[0]) * d_out
    return Workload(f"cfg1_{variant}", b.graph, {"x": x0}, units, "jacobian rows",
                    {"batch": batch, "d_in": d_in, "d_h": d_h, "d_out": d_out})


# ----------------------------------------------------------------------------
# cfg2: per-example gradients with per-example norm + clip (DP-SGD style)

def _xent(bb, logits, onehot):
    """log sum exp(logits) - <logits, onehot>; composed (no softmax op exists)."""
    lse = bb.log(bb.reduce_sum(bb.exp(logits), [0, 1]))
    return bb.sub(lse, bb.reduce_sum(bb.mul(logits, onehot), [0, 1]))


def _norm_clip(bb, grads, clip):
    sq = None
    for g in grads:
        s = bb.reduce_sum(bb.square(g), list(range(len(bb.graph.ref_shape(g)))))
        sq = s if sq is None else bb.add(sq, s)
    norm = bb.exp(bb.mul(bb.f64(0.5), bb.log(sq)))
    scale = bb.min_(bb.f64(1.0), bb.div(bb.f64(clip), norm))
    return norm, [bb.mul(g, scale) for g in grads]


def _maxpool2x2(bb, x, h, w):
    """reference bench.py:68-78 (gather/max/transpose composition)."""
    i64 = np.int64
    eh, oh = bb.const(np.arange(0, h, 2, dtype=i64)), bb.const(np.arange(1, h, 2, dtype=i64))
    ew, ow = bb.const(np.arange(0, w, 2, dtype=i64)), bb.const(np.arange(1, w, 2, dtype=i64))
    t = bb.transpose(x, [1, 0, 2, 3])
    m = bb.max_(bb.gather(t, eh), bb.gather(t, oh))
    t = bb.transpose(m, [2, 1, 0, 3])
    m = bb.max_(bb.gather(t, ew), bb.gather(t, ow))
    return bb.transpose(m, [2, 1, 0, 3])


def cfg2(api, n=128, model="mlp", clip=1.0, materialize=False, shard=None, registry=None,
         d_h=256, mode="vectorize"):
    """model "mlp": 784-d_h-10 tanh; model "conv": reference bench mnist_like.
    Outputs: norms [n], per-parameter clipped sums (+ stacked clipped grads when
    `materialize`)."""
    r = np.random.default_rng(0)
    if model == "mlp":
        X0 = _f32(r.standard_normal((n, 784)))
    else:
        X0 = _f32(r.standard_normal((n, 28, 28, 1)))
    labels = r.integers(0, 10, n)
    Y0 = np.eye(10)[labels]
    b = api.GraphBuilder()
    X = b.placeholder("x", api.DType.F64, X0.shape)
    Y = b.placeholder("y", api.DType.F64, (n, 10))
    if model == "mlp":
        W1, b1, W2, b2 = _mlp_params(r, 784, d_h, 10)
        params = [b.const(v) for v in (W1, b1, W2, b2)]

        def logits_fn(bb, x):
            cW1, cb1, cW2, cb2 = (bb._imp(p) for p in params)
            h = bb.tanh(bb.add(bb.matmul(bb.reshape(x, [1, 784]), cW1), cb1))
            return bb.add(bb.matmul(h, cW2), cb2)
    else:
        F = _f32(r.standard_normal((3, 3, 1, 8)) / 3.0)
        D = _f32(r.standard_normal((14 * 14 * 8, 10)) / 40.0)
        params = [b.const(F), b.const(D)]

        def logits_fn(bb, x):
            cF, cD = (bb._imp(p) for p in params)
            hcv = bb.relu(bb.conv2d(bb.reshape(x, [1, 28, 28, 1]), cF))
            p = _maxpool2x2(bb, hcv, 28, 28)
            return bb.matmul(bb.reshape(p, [1, 14 * 14 * 8]), cD)

    def body(bb, i):
        x = bb.gather(X, i)
        yoh = bb.reshape(bb.gather(Y, i), [1, 10])
        loss = _xent(bb, logits_fn(bb, x), yoh)
        grads = api.gradient(bb.graph, loss, [bb._imp(p) for p in params], emit=bb)
        norm, clipped = _norm_clip(bb, grads, clip)
        return [norm] + clipped

    kw = {} if registry is None else {"registry": registry}
    outs = _pfor(api, b, body, n, shard, mode, **kw)
    norms, stacked = outs[0], outs[1:]
    sums = [b.reduce_sum(s, [0]) for s in stacked]
    b.graph.set_outputs([norms] + sums + (list(stacked) if materialize else []))
    units = n if shard is None else shard[1] - shard[0]
    P = sum(int(np.prod(b.graph.ref_shape(p))) for p in params)
    return Workload(f"cfg2_{model}", b.graph, {"x": X0, "y": Y0}, units, "per-example gradients",
                    {"n": n, "model": model, "params": P, "clip": clip,
                     "materialize": materialize})


# ----------------------------------------------------------------------------
# cfg3: full jacobian of a 4-layer FC net wrt all weights

def cfg3(api, width=4096, out_dim=1024, rows=None, shard=None, mode="vectorize"):
    """jacobian(y, W_l) for l = 0..3.  `shard=(lo, hi)` builds output rows
    lo..hi-1 only (the per-rank / per-chunk form); `rows` is a convenience for
    shard=(0, rows)."""
    r = np.random.default_rng(0)
    x0 = _f32(r.standard_normal((1, width)))
    Ws = [_f32(r.standard_normal((width, width)) / np.sqrt(width)) for _ in range(3)]
    Ws.append(_f32(r.standard_normal((width, out_dim)) / np.sqrt(width)))
    b = api.GraphBuilder()
    x = b.placeholder("x", api.DType.F64, (1, width))
    cW = [b.const(w) for w in Ws]
    h = x
    for l in range(3):
        h = b.tanh(b.matmul(h, cW[l]))
    y = b.reshape(b.matmul(h, cW[3]), [out_dim])
    if rows is not None and shard is None:
        shard = (0, rows)
    b.graph.set_outputs([_jac(api, b, y, cW[l], shard, mode) for l in range(4)])
    units = out_dim if shard is None else shard[1] - shard[0]
    return Workload("cfg3", b.graph, {"x": x0}, units, "jacobian rows",
                    {"width": width, "out_dim": out_dim, "shard": shard})


def cfg3_rows(api, width, out_dim, rows_idx, mode="vectorize"):
    """Reference-compatible row sampling (no shard= in the reference): the
    jacobian of gather(y, rows) -- SURVEY.md §8d."""
    r = np.random.default_rng(0)
    x0 = _f32(r.standard_normal((1, width)))
    Ws = [_f32(r.standard_normal((width, width)) / np.sqrt(width)) for _ in range(3)]
    Ws.append(_f32(r.standard_normal((width, out_dim)) / np.sqrt(width)))
    b = api.GraphBuilder()
    x = b.placeholder("x", api.DType.F64, (1, width))
    cW = [b.const(w) for w in Ws]
    h = x
    for l in range(3):
        h = b.tanh(b.matmul(h, cW[l]))
    y = b.reshape(b.matmul(h, cW[3]), [out_dim])
    ys = b.gather(y, b.const(np.asarray(rows_idx, dtype=np.int64)))
    b.graph.set_outputs([_jac(api, b, ys, cW[l], None, mode) for l in range(4)])
    return Workload("cfg3_rows", b.graph, {"x": x0}, len(rows_idx), "jacobian rows",
                    {"width": width, "out_dim": out_dim, "rows": list(rows_idx)})


# ----------------------------------------------------------------------------
# cfg4: per-example gradients of an unrolled 1-layer LSTM (reference bench cell)

def cfg4(api, n=256, steps=64, units=512, shard=None, registry=None, mode="vectorize"):
    r = np.random.default_rng(0)
    X0 = _f32(r.standard_normal((n, steps, units)))
    Wg0 = _f32(r.standard_normal((2 * units, 4 * units)) / 8.0)
    Bg0 = _f32(r.standard_normal((1, 4 * units)) / 8.0)
    b = api.GraphBuilder()
    X = b.placeholder("x", api.DType.F64, (n, steps, units))
    Wg, Bg = b.const(Wg0), b.const(Bg0)

    def loss_fn(bb, x):
        h = bb.const(np.zeros((1, units)))
        c = bb.const(np.zeros((1, units)))
        for t in range(steps):
            xt = bb.reshape(bb.gather(x, bb.i64(t)), [1, units])
            z = bb.add(bb.matmul(bb.concat([xt, h], 1), bb._imp(Wg)), bb._imp(Bg))
            gates = bb.reshape(z, [4, units])
            ig = bb.sigmoid(bb.reshape(bb.gather(gates, bb.i64(0)), [1, units]))
            fg = bb.sigmoid(bb.reshape(bb.gather(gates, bb.i64(1)), [1, units]))
            og = bb.sigmoid(bb.reshape(bb.gather(gates, bb.i64(2)), [1, units]))
            gg = bb.tanh(bb.reshape(bb.gather(gates, bb.i64(3)), [1, units]))
            c = bb.add(bb.mul(fg, c), bb.mul(ig, gg))
            h = bb.mul(og, bb.tanh(c))
        return bb.reduce_sum(bb.square(h), [0, 1])

    def body(bb, i):
        loss = loss_fn(bb, bb.gather(X, i))
        return api.gradient(bb.graph, loss, [bb._imp(Wg), bb._imp(Bg)], emit=bb)

    kw = {} if registry is None else {"registry": registry}
    outs = _pfor(api, b, body, n, shard, mode, **kw)
    b.graph.set_outputs(outs)
    units_n = n if shard is None else shard[1] - shard[0]
    return Workload("cfg4", b.graph, {"x": X0}, units_n, "per-example gradients",
                    {"n": n, "steps": steps, "units": units})


# ----------------------------------------------------------------------------
# cfg5: auto-batched variable-length RNN (per-example while + cond)

def cfg5(api, n=1024, max_len=100, units=256, shard=None, registry=None, masked=False,
         unroll=1, mode="vectorize"):
    """`masked=True` converts the per-example while/cond with predication
    (Policy(masked_control=True)) instead of the reference's compaction:
    same values, fixed shapes (CUDA-graph capturable loop body)."""
    r = np.random.default_rng(0)
    X0 = _f32(r.standard_normal((n, max_len, units)))
    L0 = r.integers(1, max_len + 1, n).astype(np.int64)
    Wx0 = _f32(r.standard_normal((units, units)) / np.sqrt(units))
    Wh0 = _f32(r.standard_normal((units, units)) / np.sqrt(units))
    b = api.GraphBuilder()
    X = b.placeholder("x", api.DType.F64, (n, max_len, units))
    L = b.placeholder("lengths", api.DType.I64, (n,))
    Wx, Wh = b.const(Wx0), b.const(Wh0)

    def body(bb, i):
        x = bb.gather(X, i)
        li = bb.gather(L, i)

        def cond_fn(cb, car):
            return cb.less(car[0], cb._imp(li))

        def step_fn(wb, car):
            t, h = car
            xt = wb.reshape(wb.gather(wb._imp(x), t), [1, units])
            z = wb.add(wb.matmul(xt, wb._imp(Wx)), wb.matmul(h, wb._imp(Wh)))
            neg = wb.less(wb.reduce_sum(z, [0, 1]), wb.f64(0.0))
            (hn,) = wb.cond(neg, lambda tb: [tb.tanh(tb._imp(z))],
                            lambda eb: [eb.relu(eb._imp(z))])
            return [wb.add(t, wb.i64(1)), hn]

        _, hf = bb.while_loop([bb.i64(0), bb.const(np.zeros((1, units)))], cond_fn, step_fn)
        return [bb.reshape(hf, [units])]

    kw = {} if registry is None else {"registry": registry}
    if masked:
        from .vectorize import Policy
        kw["policy"] = Policy(masked_control=True, unroll=unroll)
    (H,) = _pfor(api, b, body, n, shard, mode, **kw)
    b.graph.set_outputs([H])
    sel = slice(None) if shard is None else slice(shard[0], shard[1])
    units_n = n if shard is None else shard[1] - shard[0]
    return Workload("cfg5", b.graph, {"x": X0, "lengths": L0}, units_n, "examples",
                    {"n": n, "max_len": max_len, "units": units,
                     "tokens": int(L0[sel].sum())})


BUILDERS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


# ----------------------------------------------------------------------------
# bench configurations (bench.py lines and the bench-scale parity tests)

# name: (builder, kwargs at bench size, unit, oracle sample)
# The oracle sample is what the CPU checker can run in seconds at bench size:
# None = the whole program; a list of shards = those iterations only
# (sharded pfor is bit-identical to the unsharded one).
BENCH_CONFIGS = {
    "cfg4": ("cfg4", dict(n=256, steps=64, units=512), "per-example grads/s", [(0, 1), (255, 256)]),
    "cfg2_mlp": ("cfg2", dict(n=128, model="mlp"), "per-example grads/s", None),
    "cfg2_conv": ("cfg2", dict(n=128, model="conv"), "per-example grads/s", None),
    "cfg1_batch": ("cfg1", dict(batch=32, variant="batch"), "jacobian rows/s", None),
    "cfg1_full": ("cfg1", dict(batch=32, variant="full"), "jacobian rows/s", None),
    "cfg3": ("cfg3", dict(width=4096, out_dim=1024, rows=32), "jacobian rows/s", [(0, 1), (31, 32)]),
    "cfg5": ("cfg5", dict(n=1024, max_len=100, units=256, masked=True, unroll=4), "examples/s",
             None),
    "cfg5_compact": ("cfg5", dict(n=1024, max_len=100, units=256), "examples/s", None),
}


def bench_workload(name, world=1, rank=0, api=None, **over):
    """The bench program of config `name` for one rank of `world`.

    Weak scaling over the sharded iteration space: the global problem has
    `world` times the per-GPU iterations and rank r runs the block
    `dist.shard_range(total, world, r)` through `shard=(lo, hi)` -- distinct
    jacobian rows (cfg1_full, cfg3) or distinct examples (cfg1_batch, cfg2,
    cfg4, cfg5) per rank.  cfg5's examples are first dealt by length
    (`dist.balanced_order`) so every rank gets a similar trip-count mix."""
    from .dist import balanced_order, shard_range
    api = api or this_api()
    builder, kw, _, _ = BENCH_CONFIGS[name]
    kw = dict(kw, **over)
    if world == 1:
        return BUILDERS[builder](api, **kw)
    if name == "cfg3":
        rows = kw.pop("rows")
        lo, hi = shard_range(rows * world, world, rank)
        return cfg3(api, shard=(lo, hi), **kw)
    key = "batch" if builder == "cfg1" else "n"
    per = kw[key]
    total = per * world
    kw[key] = total
    if name == "cfg1_full":
        lo, hi = shard_range(total * kw.get("d_out", 10), world, rank)
    else:
        lo, hi = shard_range(total, world, rank)
    w = BUILDERS[builder](api, shard=(lo, hi), **kw)
    if builder == "cfg5":
        perm, _ = balanced_order(w.feeds["lengths"], world)
        w.feeds = {k: np.ascontiguousarray(v[perm]) for k, v in w.feeds.items()}
        w.meta["tokens"] = int(w.feeds["lengths"][lo:hi].sum())
        w.meta["order"] = "dist.balanced_order"
    w.meta["shard"] = (lo, hi)
    w.meta["global_units"] = total * (kw.get("d_out", 10) if name == "cfg1_full" else 1)
    return w
