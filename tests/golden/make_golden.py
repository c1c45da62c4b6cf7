"""Generate golden fixtures from the REAL reference implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference `pforvec` package read-only from
/root/reference/pkg/src and writes, next to this script:

* kernels.npz   -- inputs + outputs of every reference NumPy kernel on the
                   hot path (tensor.py / interp.py inline kernels), seeded;
* programs.npz  -- feeds + outputs of the BASELINE workloads (small scale)
                   and the reference's worked examples, executed by the
                   reference Executor;
* structure.json -- the op-kind sequence of each reference vectorized graph
                   (the drop-in frontend must emit the same kernels);
* pfg/*.pfg      -- the reference's `.pfg` text (its own serializer) of each
                   worked example's source graph (`src_*`) and vectorized
                   graph (`vec_*`), and of small BASELINE programs (`prog_*`):
                   the interchange-format fixtures (`--pfg-only` rewrites
                   just these);
* corpus.json.gz -- the reference's randomized differential-testing corpus
                   (randgen.generate_case, seeds 42..141 x n in {0,1,3,7}):
                   source + vectorized `.pfg`, reference outputs and variable
                   values (`--corpus-only`).

The GPU box has no /root/reference: tests there read only these files.
"""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg")
HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(HERE.parent.parent))

import pforvec  # noqa: E402
import worked_examples as W  # noqa: E402

from paper_1903_04243_b200 import workloads as WL  # noqa: E402

T = sys.modules["pforvec.tensor"]
interp = sys.modules["pforvec.interp"]

PROGRAM_CASES = {
    "cfg1_batch": ("cfg1", dict(batch=4, d_in=12, d_h=8, d_out=3, variant="batch")),
    "cfg1_full": ("cfg1", dict(batch=4, d_in=12, d_h=8, d_out=3, variant="full")),
    "cfg1_real": ("cfg1", dict(batch=32, variant="batch")),
    "cfg2_mlp": ("cfg2", dict(n=6, model="mlp", d_h=16)),
    "cfg2_mlp_real": ("cfg2", dict(n=16, model="mlp")),
    "cfg2_conv": ("cfg2", dict(n=4, model="conv")),
    "cfg3": ("cfg3", dict(width=16, out_dim=8)),
    "cfg4": ("cfg4", dict(n=3, steps=3, units=4)),
    "cfg4_mid": ("cfg4", dict(n=4, steps=8, units=16)),
    "cfg5": ("cfg5", dict(n=5, max_len=6, units=4)),
    "cfg5_mid": ("cfg5", dict(n=32, max_len=12, units=16)),
}


def tv(a, dt=None):
    return T.tensor(np.asarray(a), dt)


class _R:
    """default_rng whose float draws are rounded to fp32 (the parity rule:
    inputs drawn in fp32, upcast for the f64 reference)."""

    def __init__(self, seed):
        self._r = np.random.default_rng(seed)

    def standard_normal(self, shape):
        return np.asarray(self._r.standard_normal(shape), np.float32).astype(np.float64)

    def integers(self, lo, hi, shape):
        return self._r.integers(lo, hi, shape)


def kernel_cases(r):
    """(name, fn, inputs dict) triples; every fn is the reference kernel."""
    F, I, B = T.DType.F64, T.DType.I64, T.DType.BOOL
    cases = []
    shapes = [((3, 4), (4,)), ((2, 1, 5), (3, 1)), ((6,), ()), ((4, 3, 8), (4, 1, 8)),
              ((1,), (5, 1)), ((40, 32, 16), (32, 16))]
    for op in T.BINARY_OPS:
        for k, (sa, sb) in enumerate(shapes):
            a = r.standard_normal(sa)
            b = r.standard_normal(sb)
            if op == "div":
                b = np.where(np.abs(b) < 0.1, 0.5, b)
            if op in ("max", "min") and k == 0:
                a[0, 0] = np.nan
            cases.append((f"binary_{op}_{k}", lambda a, b, op=op: T.binary_elementwise(op, tv(a), tv(b)),
                          {"a": a, "b": b}))
        if op not in ("div",):
            ia = r.integers(-5, 5, (4, 6))
            ib = r.integers(-5, 5, (6,))
            cases.append((f"binary_{op}_i64", lambda a, b, op=op: T.binary_elementwise(op, tv(a), tv(b)),
                          {"a": ia, "b": ib}))
    for op in ("less", "equal"):
        ba = r.integers(0, 2, (5, 3)).astype(bool)
        bb = r.integers(0, 2, (3,)).astype(bool)
        cases.append((f"binary_{op}_bool", lambda a, b, op=op: T.binary_elementwise(op, tv(a), tv(b)),
                      {"a": ba, "b": bb}))
    for op in T.UNARY_OPS:
        if op == "logical_not":
            x = r.integers(0, 2, (7, 3)).astype(bool)
        elif op == "log":
            x = np.abs(r.standard_normal((5, 7))) + 0.1
        else:
            x = r.standard_normal((5, 7)) * 2
        cases.append((f"unary_{op}", lambda x, op=op: T.unary_elementwise(op, tv(x)), {"x": x}))
    for op in ("neg", "relu", "square"):
        cases.append((f"unary_{op}_i64", lambda x, op=op: T.unary_elementwise(op, tv(x)),
                      {"x": r.integers(-9, 9, (4, 5))}))
    x = np.array([1.5, -2.5, 0.0, 3.99, -0.7])
    cases.append(("cast_f_i", lambda x: T.cast(tv(x), I), {"x": x}))
    cases.append(("cast_f_b", lambda x: T.cast(tv(x), B), {"x": x}))
    cases.append(("cast_i_f", lambda x: T.cast(tv(x), F), {"x": r.integers(-100, 100, (6,))}))
    cases.append(("cast_b_f", lambda x: T.cast(tv(x), F), {"x": r.integers(0, 2, (6,)).astype(bool)}))
    for k, (sa, sb) in enumerate([((7, 5), (5, 3)), ((4, 6, 5), (4, 5, 2)), ((33, 70), (70, 65)),
                                  ((130, 1), (1, 77)), ((3, 9, 40), (3, 40, 8))]):
        cases.append((f"matmul_{k}", lambda a, b: T.matmul(tv(a), tv(b)),
                      {"a": r.standard_normal(sa), "b": r.standard_normal(sb)}))
    for k, (sx, sf) in enumerate([((2, 5, 6, 3), (3, 3, 3, 4)), ((3, 7, 7, 1), (3, 3, 1, 8)),
                                  ((1, 4, 5, 2), (2, 4, 2, 3))]):
        x, f = r.standard_normal(sx), r.standard_normal(sf)
        cases.append((f"conv2d_{k}", lambda x, f: T.conv2d(tv(x), tv(f)), {"x": x, "f": f}))
        gy = r.standard_normal(sx[:3] + (sf[3],))
        cases.append((f"conv2d_input_grad_{k}", lambda gy, f: T.conv2d_input_grad(tv(gy), tv(f)),
                      {"gy": gy, "f": f}))
        cases.append((f"im2col_{k}", lambda x, k1=sf[0], k2=sf[1]: T.im2col(tv(x), k1, k2), {"x": x}))
    for k, (shape, axes) in enumerate([((3, 4, 5), (1,)), ((3, 4, 5), (0, 2)), ((3, 4, 5), (-1,)),
                                       ((6, 7), (0, 1)), ((9, 2000), (1,)), ((3000, 5), (0,)),
                                       ((4, 3, 5, 2), (1, 3))]):
        cases.append((f"reduce_sum_{k}", lambda x, axes=axes: T.reduce_sum(tv(x), axes),
                      {"x": r.standard_normal(shape)}))
    cases.append(("reduce_sum_i64", lambda x: T.reduce_sum(tv(x), (0,)),
                  {"x": r.integers(-50, 50, (8, 3))}))
    cases.append(("concat_ax1", lambda a, b: T.concat([tv(a), tv(b)], 1),
                  {"a": r.standard_normal((3, 2, 4)), "b": r.standard_normal((3, 5, 4))}))
    cases.append(("concat_ax0", lambda a, b: T.concat([tv(a), tv(b)], 0),
                  {"a": r.standard_normal((2, 4)), "b": r.standard_normal((3, 4))}))
    X = r.standard_normal((9, 3, 2))
    cases.append(("gather_vec", lambda x, i: T.gather_rows(tv(x), tv(i)),
                  {"x": X, "i": np.array([4, 0, 8, 4, 2])}))
    cases.append(("gather_scalar", lambda x, i: T.gather_rows(tv(x), tv(i)),
                  {"x": X, "i": np.int64(7)}))
    cases.append(("gather_i64", lambda x, i: T.gather_rows(tv(x), tv(i)),
                  {"x": r.integers(0, 100, (6, 4)), "i": np.array([5, 1, 1])}))
    cases.append(("scatter_rows", lambda i0, i1, p0, p1: T.scatter_rows([tv(i0), tv(i1)],
                                                                         [tv(p0), tv(p1)], 6),
                  {"i0": np.array([4, 0, 2]), "i1": np.array([1, 5, 3]),
                   "p0": r.standard_normal((3, 2)), "p1": r.standard_normal((3, 2))}))
    cases.append(("scatter_add_dup", lambda i, u: T.scatter_add_rows(tv(i), tv(u), 5),
                  {"i": np.array([1, 3, 1, 1, 0]), "u": r.standard_normal((5, 4))}))
    cases.append(("scatter_add_scalar", lambda i, u: T.scatter_add_rows(tv(i), tv(u), 4),
                  {"i": np.int64(2), "u": r.standard_normal((3,))}))
    cases.append(("transpose", lambda x: T.transpose(tv(x), (2, 0, 1)),
                  {"x": r.standard_normal((3, 4, 5))}))
    cases.append(("stack", lambda a, b: T.stack([tv(a), tv(b)]),
                  {"a": r.standard_normal((2, 3)), "b": r.standard_normal((2, 3))}))
    cases.append(("tile_leading", lambda x: T.tile_leading(tv(x), 3),
                  {"x": r.standard_normal((2, 3))}))
    cases.append(("slice_leading", lambda x: T.slice_leading(tv(x), 2),
                  {"x": r.standard_normal((5, 3))}))
    m = r.integers(0, 2, (50,)).astype(bool)
    cases.append(("where_true", lambda m: T.TensorValue(I, np.nonzero(m)[0].astype(np.int64)), {"m": m}))
    return cases


def ref_complement(idx, total):
    return np.setdiff1d(np.arange(total, dtype=np.int64), np.atleast_1d(idx))


def main():
    r = _R(1234)
    kern = {}
    for name, fn, ins in kernel_cases(r):
        ins = {k: (np.asarray(v, np.float32).astype(np.float64)
                   if np.asarray(v).dtype == np.float64 else v) for k, v in ins.items()}
        out = fn(**ins)
        for k, v in ins.items():
            v = np.asarray(v)
            kern[f"{name}/in/{k}"] = v.astype(np.float32) if v.dtype == np.float64 else v
        kern[f"{name}/out"] = out.data
    # interp.py inline kernels
    idx = np.array([7, 2, 2, 9])
    kern["complement/in/idx"], kern["complement/in/total"] = idx, np.int64(12)
    kern["complement/out"] = ref_complement(idx, 12)
    rng = interp.RngState(seed=42, counter=3)
    kern["rng/in/seed"], kern["rng/in/counter"] = np.int64(42), np.int64(3)
    kern["rng/out"] = rng.draw((4, 5)).data
    np.savez_compressed(HERE / "kernels.npz", **kern)

    ref_api = WL.reference_api(pforvec)
    progs, structure = {}, {}
    for name, (cfg, kw) in PROGRAM_CASES.items():
        w = WL.BUILDERS[cfg](ref_api, **kw)
        outs = pforvec.Executor(w.graph).run(feeds=w.feeds)
        for k, v in w.feeds.items():
            v = np.asarray(v)
            progs[f"{name}/feed/{k}"] = v.astype(np.float32) if v.dtype == np.float64 else v
        for j, o in enumerate(outs):
            progs[f"{name}/out/{j}"] = o.data
        structure[name] = [n.kind for n in w.graph.topo_order()]
    for name, fn in list(W.GOLDEN_EXAMPLES.items()) + [("cond_example", W.cond_example),
                                                       ("while_example", W.while_example)]:
        g2, _ = pforvec.vectorize_graph(fn())
        outs = pforvec.Executor(g2).run()
        for j, o in enumerate(outs):
            progs[f"we_{name}/out/{j}"] = o.data
        structure[f"we_{name}"] = [n.kind for n in g2.topo_order()]
    np.savez_compressed(HERE / "programs.npz", **progs)
    (HERE / "structure.json").write_text(json.dumps(structure, indent=0))
    print(f"kernels: {len([k for k in kern if k.endswith('/out')])} cases; "
          f"programs: {len(PROGRAM_CASES)} + worked examples")


def write_corpus(seeds=range(42, 142), ns=(0, 1, 3, 7)):
    """Differential-testing corpus (reference randgen.py / test_acceptance.py
    criterion 1): random parfor bodies from the reference's own generator; per
    case the source graph and the reference's vectorized graph as `.pfg`
    text, the reference Executor's outputs / final variable values on the
    source graph (RngState(seed)), and which of them depend on random draws
    (compared by shape/dtype only, as the reference does)."""
    import gzip
    rg = sys.modules.get("pforvec.randgen") or __import__("pforvec.randgen", fromlist=["x"])
    ser = sys.modules.get("pforvec.serialize") or __import__("pforvec.serialize", fromlist=["x"])
    cases = {}
    for seed in seeds:
        for n in ns:
            case = rg.generate_case(seed, max_depth=8, n=n)
            g = case.graph
            ex = interp.Executor(g, store=interp.VariableStore(g.variables),
                                 rng=interp.RngState(seed))
            try:
                outs = ex.run()
            except pforvec.PforVecError as e:  # noqa: F841  (not in the corpus)
                continue
            g2, _ = pforvec.vectorize_graph(g, policy=pforvec.Policy(stateful_assign_fallback=True))
            enc = lambda v: {"dtype": v.dtype.value, "shape": list(v.shape),  # noqa: E731
                             "data": np.asarray(v.data, np.float64).reshape(-1).tolist()}
            cases[f"{seed}_{n}"] = {
                "seed": seed, "n": n, "src": ser.dumps(g), "vec": ser.dumps(g2),
                "outs": [enc(o) for o in outs], "tainted": list(map(bool, case.tainted)),
                "vars": {k: enc(v) for k, v in ex.store.values.items()},
                "var_tainted": {k: bool(t) for k, t in case.var_tainted.items()}}
    with gzip.open(HERE / "corpus.json.gz", "wt") as fh:
        json.dump(cases, fh)
    print(f"corpus: {len(cases)} cases")


def write_pfg():
    ser = sys.modules["pforvec.serialize"] if "pforvec.serialize" in sys.modules else None
    if ser is None:
        import pforvec.serialize as ser  # noqa: F811
    out = HERE / "pfg"
    out.mkdir(exist_ok=True)
    for name, fn in list(W.GOLDEN_EXAMPLES.items()) + [("cond_example", W.cond_example),
                                                       ("while_example", W.while_example)]:
        g = fn()
        (out / f"src_{name}.pfg").write_text(ser.dumps(g))
        g2, _ = pforvec.vectorize_graph(g)
        (out / f"vec_{name}.pfg").write_text(ser.dumps(g2))
    ref_api = WL.reference_api(pforvec)
    for name in ("cfg1_full", "cfg2_mlp", "cfg5"):
        cfg, kw = PROGRAM_CASES[name]
        w = WL.BUILDERS[cfg](ref_api, **kw)
        (out / f"prog_{name}.pfg").write_text(ser.dumps(w.graph))
    print(f"pfg fixtures: {len(list(out.glob('*.pfg')))}")


if __name__ == "__main__":
    if "--pfg-only" not in sys.argv and "--corpus-only" not in sys.argv:
        main()
    if "--corpus-only" not in sys.argv:
        write_pfg()
    write_corpus()
