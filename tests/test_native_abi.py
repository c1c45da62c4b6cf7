"""CPU: the C-ABI library loads and exports exactly what include/pfb.h declares."""

import ctypes
import pathlib
import re

import pytest

from paper_1903_04243_b200 import _native as N

ROOT = pathlib.Path(__file__).resolve().parent.parent


def declared():
    src = (ROOT / "include" / "pfb.h").read_text()
    return sorted(set(re.findall(r"^(?:int|int64_t) (pfb_\w+)\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("pfb_binary", "pfb_unary", "pfb_cast", "pfb_matmul", "pfb_reduce_sum",
                 "pfb_gather_rows", "pfb_scatter_rows", "pfb_scatter_add_rows",
                 "pfb_where_true", "pfb_complement", "pfb_conv2d", "pfb_conv2d_input_grad",
                 "pfb_im2col", "pfb_rng_uniform", "pfb_copy", "pfb_iota"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not N.LIB_PATH.exists():
        pytest.skip("libpfb.so not built (run __graft_entry__.build())")
    lib = N.load()
    for name in declared():
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert set(declared()) == set(N.EXPORTED)
    assert lib.pfb_version() >= 100


def test_library_is_sm100a():
    import subprocess
    if not N.LIB_PATH.exists():
        pytest.skip("libpfb.so not built")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(N.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_executor_fails_loudly_without_device(monkeypatch):
    import torch
    from paper_1903_04243_b200 import GraphBuilder, errors
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    from paper_1903_04243_b200.executor import Executor
    b = GraphBuilder()
    b.graph.set_outputs([b.add(b.f64(1.0), b.f64(2.0))])
    with pytest.raises(errors.NativeUnavailable):
        Executor(b.graph)
