"""CPU: the reference's randomized differential-testing corpus (randgen.py;
reference tests/test_acceptance.py criterion 1), 400 random parfor bodies
(seeds 42..141 x n in {0,1,3,7}: elementwise, linalg, nested cond/while,
variables, random draws) generated and run BY THE REFERENCE
(tests/golden/make_golden.py -> corpus.json.gz).

* the frontend's pfor conversion of each source graph is byte-identical to
  the reference's vectorized graph (`.pfg` text);
* the oracle run of the source graph reproduces the reference's outputs and
  final variable values (random-draw-dependent ones by shape/dtype only, as
  the reference compares them)."""

import gzip
import json
import pathlib

import numpy as np
import pytest

from oracle import OracleExecutor, RngState, VariableStore
from paper_1903_04243_b200 import Policy, pfg
from paper_1903_04243_b200.vectorize import vectorize_graph

CORPUS = json.load(gzip.open(pathlib.Path(__file__).parent / "golden" / "corpus.json.gz", "rt"))


def decode(e):
    return np.asarray(e["data"], np.float64).reshape(e["shape"])


def compare(got, want, tainted, tol):
    if tuple(got.shape) != tuple(want["shape"]) or got.dtype.value != want["dtype"]:
        return f"{got.dtype.value}{list(got.shape)} vs {want['dtype']}{want['shape']}"
    if tainted:
        return None
    g = np.asarray(got.data, np.float64)
    w = decode(want)
    if g.size and not np.allclose(g, w, rtol=tol[0], atol=tol[1], equal_nan=True):
        return f"max abs delta {np.max(np.abs(g - w)):.3e}"
    return None


def test_corpus_vectorized_graphs_are_byte_identical():
    bad = []
    for key, c in CORPUS.items():
        g2, _ = vectorize_graph(pfg.loads(c["src"]), policy=Policy(stateful_assign_fallback=True))
        if pfg.dumps(g2) != c["vec"]:
            bad.append(key)
    assert not bad, f"{len(bad)}/{len(CORPUS)} differ, e.g. {bad[:5]}"


def test_corpus_oracle_matches_reference_outputs():
    bad = []
    for key, c in CORPUS.items():
        g = pfg.loads(c["src"])
        ex = OracleExecutor(g, store=VariableStore(g.variables), rng=RngState(c["seed"]))
        outs = ex.run()
        for j, (o, w) in enumerate(zip(outs, c["outs"])):
            msg = compare(o, w, c["tainted"][j], (0, 1e-9))
            if msg:
                bad.append(f"{key} out {j}: {msg}")
        for name, w in c["vars"].items():
            msg = compare(ex.store.values[name], w, c["var_tainted"].get(name, False), (0, 1e-9))
            if msg:
                bad.append(f"{key} var {name}: {msg}")
    assert not bad, bad[:5]
