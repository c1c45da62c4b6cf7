"""GPU: every bench configuration at the size bench.py measures, checked
against the oracle (the pinned CPU restatement of the reference executor).

The programs are built exactly as bench.py builds them
(`workloads.BENCH_CONFIGS`), executed the way the bench executes them -- an
eager warm-up run (which also autotunes the GEMM shapes), a CUDA-graph capture
and replays -- and the replayed outputs are compared with the reference
formulation (reference converter registry) run by the oracle in f64.  Where
the whole program is too large for the CPU checker (cfg3 at width 4096: 7 GB
per 32 rows; cfg4 at U=512: 2.15 GB of per-example gradients) the oracle runs
sampled iterations through `shard=(lo, hi)`, which builds exactly those
iterations of the same program (bit-identical to the unsharded pfor, §8e).

Mirrors the reference's acceptance check of per-example gradients
(`/root/reference/pkg/tests/test_acceptance.py:221-296`): per-example
results of the vectorized program equal the independently computed ones.
Bar: rtol 1e-4 / atol 1e-5 (fp32 vs the f64 reference); integer outputs exact.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _oracle_outputs(builder, kw, shard):
    from oracle import OracleExecutor
    from paper_1903_04243_b200 import reference_registry
    from paper_1903_04243_b200 import workloads as WL
    kw = dict(kw)
    if builder != "cfg3":
        kw["registry"] = reference_registry()
    if shard is not None:
        kw.pop("rows", None)
        kw["shard"] = shard
    if builder == "cfg5":  # the reference formulation: compaction, no predication
        kw.pop("masked", None)
        kw.pop("unroll", None)
    w = WL.BUILDERS[builder](WL.this_api(), **kw)
    return [np.asarray(o.data) for o in OracleExecutor(w.graph, budget=10 ** 9).run(feeds=w.feeds)]


def _close(got, want, what):
    got = np.asarray(got)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    if want.dtype.kind == "f":
        err = np.abs(got.astype(np.float64) - want)
        bad = err > ATOL + RTOL * np.abs(want)
        assert not bad.any(), (f"{what}: {int(bad.sum())} of {bad.size} elements outside "
                               f"rtol {RTOL} / atol {ATOL}; max abs err {float(err.max()):.3g}")
    else:
        np.testing.assert_array_equal(got.astype(want.dtype), want, err_msg=what)


def _run_bench_style(w, dev, runs=3):
    """eager (autotune) -> capture -> replay, as bench.py's warm-up does."""
    from paper_1903_04243_b200.executor import Executor
    ex = Executor(w.graph, device=dev)
    for _ in range(runs - 1):
        ex.run_device(w.feeds)
    return ex, ex.run_device(w.feeds)


@pytest.mark.parametrize("name", ["cfg2_mlp", "cfg2_conv", "cfg1_batch", "cfg1_full", "cfg5",
                                  "cfg5_compact", "cfg4", "cfg3"])
def test_bench_config_at_bench_size(name, dev):
    import torch
    from paper_1903_04243_b200 import workloads as WL
    builder, kw, _, sample = WL.BENCH_CONFIGS[name]
    w = WL.bench_workload(name)
    ex, outs = _run_bench_style(w, dev)
    if sample is None:
        want = _oracle_outputs(builder, kw, None)
        assert len(want) == len(outs)
        for j, (o, r) in enumerate(zip(outs, want)):
            _close(o.to_numpy() if hasattr(o, "to_numpy") else o.value, r, f"{name} out {j}")
    else:
        for lo, hi in sample:
            want = _oracle_outputs(builder, kw, (lo, hi))
            for j, (o, r) in enumerate(zip(outs, want)):
                got = o.torch_view()[lo:hi].cpu().numpy()
                _close(got, r, f"{name} out {j} iterations [{lo},{hi})")
    torch.cuda.synchronize(dev)
    assert ex.launch_count > 0


def test_cfg4_replay_is_deterministic(dev):
    """Two replays of the captured cfg4 step give bit-identical results (no
    races in the split-K / pair GEMMs or the fused gate kernels)."""
    from paper_1903_04243_b200 import workloads as WL
    w = WL.bench_workload("cfg4", n=32)
    ex, outs = _run_bench_style(w, dev)
    a = [o.torch_view().clone() for o in outs]
    outs = ex.run_device(w.feeds)
    for x, o in zip(a, outs):
        assert bool((x == o.torch_view()).all())
