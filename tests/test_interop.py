"""CPU: graphs built by the REFERENCE package itself import into this IR and
run to the same values (oracle here; the B200 Executor accepts them the same
way).  Skipped where /root/reference is absent (the GPU box)."""

import pathlib
import sys

import numpy as np
import pytest

REF = pathlib.Path("/root/reference/pkg")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not mounted")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF / "src"))
    sys.path.insert(0, str(REF / "tests"))
    import pforvec
    import worked_examples
    return pforvec, worked_examples


def test_import_reference_worked_examples(ref):
    pforvec, W = ref
    from oracle import OracleExecutor
    from paper_1903_04243_b200.interop import import_graph
    for name in list(W.GOLDEN_EXAMPLES) + ["cond_example", "while_example"]:
        fn = W.GOLDEN_EXAMPLES.get(name) or getattr(W, name)
        g = fn()
        want = pforvec.Executor(g).run()
        got = OracleExecutor(import_graph(g)).run()
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a.data, b.data)


def test_import_reference_jacobian_and_per_example(ref):
    pforvec, _ = ref
    from oracle import OracleExecutor
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.interop import import_graph
    for cfg, kw in (("cfg1", dict(batch=3, d_in=6, d_h=4, d_out=2, variant="full")),
                    ("cfg2", dict(n=4, model="mlp", d_h=8)),
                    ("cfg5", dict(n=4, max_len=5, units=3))):
        w = WL.BUILDERS[cfg](WL.reference_api(pforvec), **kw)
        want = pforvec.Executor(w.graph).run(feeds=w.feeds)
        got = OracleExecutor(import_graph(w.graph)).run(feeds=w.feeds)
        for a, b in zip(got, want):
            np.testing.assert_allclose(a.data, b.data, rtol=0, atol=1e-12)
