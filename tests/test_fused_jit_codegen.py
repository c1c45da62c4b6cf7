"""CPU (no device): the fused-program specialiser (csrc/fused_jit.cu) emits
CUDA that NVRTC compiles for sm_100a, for every fused group the passes form
on the bench programs and the reference's randomized corpus, in each feed
mode (vector / broadcast / strided) and both domains.  The device-side
equality with the interpreter is tests/test_gpu_jit.py."""

import ctypes
import gzip
import json
import pathlib

import pytest

from test_oracle_golden import PROGRAM_CASES, build_program

GOLD = pathlib.Path(__file__).parent / "golden"
F32, I64, BOOL = 0, 1, 2


@pytest.fixture(scope="module")
def lib():
    from paper_1903_04243_b200 import _native
    L = _native.load()
    probe = _check(L, False, 4, 0, 1, [F32], [[67, 1, 0, 0]], [1], [F32])
    if probe == 5:  # PFB_E_UNSUPPORTED: no NVRTC in this process
        pytest.skip("NVRTC unavailable here")
    assert probe == 0
    return L


def _check(L, integer, v, modes, n_in, in_dt, program, out_regs, out_dt):
    flat = [int(x) for step in program for x in step]
    arr = lambda xs: (ctypes.c_int32 * max(len(xs), 1))(*xs)  # noqa: E731
    return L.pfb_fused_jit_check(int(integer), v, modes, n_in, arr(in_dt), len(program), arr(flat),
                                 len(out_regs), arr(out_regs), arr(out_dt))


def _dt(d):
    return BOOL if getattr(d, "value", d) == "bool" else (I64 if getattr(d, "value", d) == "i64"
                                                          else F32)


def _groups(g, acc):
    """(integer, n_in, program, out_regs, out_dtypes) of every fused node,
    nested block subgraphs included"""
    for n in g.nodes.values():
        if n.kind in ("fused_ew", "fused_ewm", "fused_int", "fused_pack"):
            prog = tuple(tuple(int(x) for x in s) for s in n.attrs["program"])
            if n.kind == "fused_ew":
                regs, dts = (prog[-1][1],), (_dt(n.attrs["out_dtype"]),)
            else:
                regs = tuple(int(r) for r in n.attrs["out_regs"])
                dts = tuple(_dt(d) for d in n.attrs["out_dtypes"])
            acc.add((n.kind == "fused_int", len(n.inputs), prog, regs, dts))
        if n.block is not None:
            for sg in n.block.subgraphs.values():
                _groups(sg, acc)
    return acc


def _optimized(g):
    from paper_1903_04243_b200.passes import optimize
    keys = [tuple(o) for o in g.outputs]
    return optimize(g, keys)[0]


def _compile_all(lib, groups, variants):
    bad = []
    for integer, n_in, prog, regs, dts in sorted(groups):
        for v, mode in ([(1, 2)] if integer else variants):
            modes = 0
            for o in range(1, n_in + 1):
                modes |= mode << (2 * o)
            in_dt = [I64 if integer else F32] * n_in
            rc = _check(lib, integer, v, modes, n_in, in_dt, prog, list(regs), list(dts))
            if rc != 0:
                bad.append((rc, integer, v, mode, prog))
    return bad


def test_bench_program_groups_compile(lib):
    groups = set()
    for name in sorted(PROGRAM_CASES):
        _groups(_optimized(build_program(name).graph), groups)
    assert groups, "no fused groups formed on the bench programs"
    bad = _compile_all(lib, groups, [(4, 0), (4, 1), (4, 2), (1, 2)])
    assert not bad, bad[:3]


def test_corpus_groups_compile(lib):
    from paper_1903_04243_b200 import pfg
    corpus = json.load(gzip.open(GOLD / "corpus.json.gz", "rt"))
    groups = set()
    for key in sorted(corpus):
        _groups(_optimized(pfg.loads(corpus[key]["vec"])), groups)
    assert groups
    bad = _compile_all(lib, groups, [(4, 0)])
    assert not bad, bad[:3]


def test_bool_inputs_and_outputs_compile(lib):
    # less(x, y) -> bool, select(mask, a, b), logical_not of a bool input
    prog = [[64, 0, 0, 0], [64, 1, 1, 0], [64, 2, 2, 0], [6, 3, 0, 1],
            [68, 1, 2, 0], [16 + 7, 4, 2, 0]]
    for v, mode in [(4, 0), (4, 1), (1, 2)]:
        modes = sum(mode << (2 * o) for o in range(1, 4))
        assert _check(lib, False, v, modes, 3, [F32, F32, BOOL], prog, [3, 1, 4],
                      [BOOL, F32, BOOL]) == 0


def test_bad_program_rejected(lib):
    assert _check(lib, False, 4, 0, 1, [F32], [[67, 99, 0, 0]], [1], [F32]) == 4  # PFB_E_ARG
    assert _check(lib, False, 3, 0, 1, [F32], [[67, 1, 0, 0]], [1], [F32]) == 4
