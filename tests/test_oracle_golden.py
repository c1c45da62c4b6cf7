"""CPU: pin the oracle (and the host frontend) to the real reference.

Golden fixtures were produced by the reference itself (tests/golden/
make_golden.py).  Here the oracle restatement must reproduce them exactly
(f64, same NumPy ops), and the frontend must emit the reference's op
sequence -- the kernels the B200 executor will run.
"""

import json
import pathlib

import numpy as np
import pytest

import kernel_graphs as KG
from oracle import OracleExecutor, RngState
from oracle import kernels as OK
from paper_1903_04243_b200 import workloads as WL
from paper_1903_04243_b200 import vectorize_graph

GOLD = pathlib.Path(__file__).parent / "golden"
STRUCT = json.loads((GOLD / "structure.json").read_text())


def _names():
    return KG.case_names(np.load(GOLD / "kernels.npz").files)


@pytest.mark.parametrize("name", [n for n in _names() if n not in ("rng",)])
def test_oracle_kernel_matches_reference(name, golden):
    K = golden["kernels"]
    g = KG.build_case(name, KG.inputs(K, name))
    (got,) = OracleExecutor(g).run()
    want = K[f"{name}/out"]
    assert got.shape == tuple(want.shape)
    if want.dtype.kind == "f":
        np.testing.assert_allclose(got.data, want, rtol=0, atol=1e-12, equal_nan=True)
    else:
        np.testing.assert_array_equal(got.data, want)


def test_oracle_rng_bit_exact(golden):
    K = golden["kernels"]
    got = OK.rng_uniform(int(K["rng/in/seed"]), int(K["rng/in/counter"]), (4, 5))
    np.testing.assert_array_equal(got.data, K["rng/out"])


def _program_cases():
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden_cases", GOLD / "make_golden.py")
    src = (GOLD / "make_golden.py").read_text()
    start = src.index("PROGRAM_CASES = {")
    end = src.index("}\n", start) + 2
    ns = {}
    exec(src[start:end], ns)
    return ns["PROGRAM_CASES"]


PROGRAM_CASES = _program_cases()


def build_program(name, **over):
    cfg, kw = PROGRAM_CASES[name]
    kw = dict(kw, **over)
    return WL.BUILDERS[cfg](WL.this_api(), **kw)


@pytest.mark.parametrize("name", sorted(PROGRAM_CASES))
def test_oracle_program_matches_reference(name, golden):
    P = golden["programs"]
    w = build_program(name, registry=__import__("paper_1903_04243_b200").reference_registry()) \
        if PROGRAM_CASES[name][0] != "cfg3" else build_program(name)
    for k, v in w.feeds.items():
        np.testing.assert_array_equal(np.asarray(v, np.float32 if np.asarray(v).dtype == np.float64
                                                  else np.asarray(v).dtype), P[f"{name}/feed/{k}"])
    outs = OracleExecutor(w.graph).run(feeds=w.feeds)
    for j, o in enumerate(outs):
        np.testing.assert_allclose(o.data, P[f"{name}/out/{j}"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", sorted(PROGRAM_CASES))
def test_frontend_emits_reference_op_sequence(name):
    from paper_1903_04243_b200 import reference_registry
    cfg, _ = PROGRAM_CASES[name]
    w = build_program(name) if cfg == "cfg3" else build_program(name, registry=reference_registry())
    assert [n.kind for n in w.graph.topo_order()] == STRUCT[name]


def test_b200_registry_removes_fallback_loops_with_same_values(golden):
    """§8f-1: conv maxpool backward and the cfg5 x[t] gather no longer fall back."""
    P = golden["programs"]
    for name in ("cfg2_conv", "cfg5"):
        w = build_program(name)
        kinds = [n.kind for n in w.graph.topo_order()]
        assert kinds.count("while") <= STRUCT[name].count("while")
        outs = OracleExecutor(w.graph).run(feeds=w.feeds)
        for j, o in enumerate(outs):
            np.testing.assert_allclose(o.data, P[f"{name}/out/{j}"], rtol=0, atol=1e-12)
    conv = build_program("cfg2_conv")
    assert [n.kind for n in conv.graph.topo_order()].count("while") == 0


def _worked():
    import worked_examples_local as WE
    return WE


@pytest.mark.parametrize("name", ["pairwise_sum_diff", "gather_identity", "matmul_fold",
                                  "conv2d_fold", "reduce_sum_renumber", "concat_shift",
                                  "broadcast_reshape", "cond_example", "while_example"])
def test_worked_examples(name, golden):
    WE = _worked()
    g = getattr(WE, name)()
    g2, _ = vectorize_graph(g, registry=__import__("paper_1903_04243_b200").reference_registry())
    assert [n.kind for n in g2.topo_order()] == STRUCT[f"we_{name}"]
    P = golden["programs"]
    for j, o in enumerate(OracleExecutor(g2).run()):
        np.testing.assert_array_equal(o.data, P[f"we_{name}/out/{j}"])
    # and the un-vectorized graph under the SIMD interpreter (the loop baseline)
    for j, o in enumerate(OracleExecutor(g).run()):
        np.testing.assert_array_equal(o.data, P[f"we_{name}/out/{j}"])
