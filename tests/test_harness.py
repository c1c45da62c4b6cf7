"""The reference bench harness restated (paper_1903_04243_b200.harness):
same models, seeds, modes and CSV columns.  CPU: each model's graph, built by
this package, computes what the reference's own bench graph computes (oracle
vs the reference Executor; skipped where /root/reference is absent).  GPU:
run_bench on the device produces the reference CSV format."""

import csv
import pathlib
import sys

import numpy as np
import pytest

from paper_1903_04243_b200 import harness as H

REF = pathlib.Path("/root/reference/pkg")
SMALL = {"linear": 3, "mnist_like": 2, "lstm_unrolled": 2, "per_example_grad": 3, "jacobian": 4}


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
@pytest.mark.parametrize("model", sorted(H.MODELS))
@pytest.mark.parametrize("mode", ["vectorize", "parfor"])
def test_models_match_reference_bench(model, mode):
    sys.path.insert(0, str(REF / "src"))
    import pforvec
    rb = sys.modules["pforvec.bench"] if "pforvec.bench" in sys.modules else __import__(
        "pforvec.bench", fromlist=["x"])
    from oracle import OracleExecutor
    n = SMALL[model]
    want = pforvec.Executor(rb.MODELS[model](n, mode)).run()
    g = H.MODELS[model](n, mode)
    got = OracleExecutor(g).run()
    assert len(got) == len(want)
    for a, b in zip(got, want):
        np.testing.assert_allclose(np.asarray(a.data, np.float64), np.asarray(b.data, np.float64),
                                   rtol=1e-10, atol=1e-12)


def test_csv_format(tmp_path):
    rec = [H.BenchRecord("linear", "vectorize", 4, 0.0012345678, 7, 3240.1234)]
    p = tmp_path / "b.csv"
    H.write_csv(rec, p)
    rows = list(csv.reader(open(p)))
    assert rows[0] == H.CSV_HEADER
    assert rows[1] == ["linear", "vectorize", "4", "0.001235", "7", "3240.12"]
    assert H.format_table(rec).splitlines()[0] == ",".join(H.CSV_HEADER)


def test_unknown_model():
    with pytest.raises(H.UnknownModel):
        H.run_bench("resnet", 2, "vectorize")


@pytest.mark.gpu
@pytest.mark.parametrize("model", sorted(H.MODELS))
def test_run_bench_on_device(model):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    recs = [H.run_bench(model, SMALL[model], mode, repeats=2) for mode in ("vectorize", "parfor")]
    for r in recs:
        assert r.wall_time_s > 0 and r.dispatch_count > 0 and r.throughput > 0
    # vectorized dispatch count is independent of the batch (the paper's claim)
    big = H.run_bench(model, 2 * SMALL[model], "vectorize", repeats=1)
    assert big.dispatch_count == recs[0].dispatch_count
