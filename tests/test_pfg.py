"""CPU: the `.pfg` interchange format (reference serialize.py; SURVEY §8f
row 4).  Fixtures in tests/golden/pfg/ were written by the reference's own
serializer (tests/golden/make_golden.py): src_* = worked-example source
graphs, vec_* = the reference's vectorized graphs (byte-identical to its
tests/golden/*.pfg), prog_* = BASELINE programs at small scale."""

import pathlib

import numpy as np
import pytest

from oracle import OracleExecutor
from paper_1903_04243_b200 import pfg
from paper_1903_04243_b200.errors import ParseError
from paper_1903_04243_b200.vectorize import vectorize_graph

PFG = pathlib.Path(__file__).parent / "golden" / "pfg"
FILES = sorted(p.name for p in PFG.glob("*.pfg"))
SRC = sorted(p.name[4:-4] for p in PFG.glob("src_*.pfg"))
PROGS = {"prog_cfg1_full.pfg": "cfg1_full", "prog_cfg2_mlp.pfg": "cfg2_mlp",
         "prog_cfg5.pfg": "cfg5"}


@pytest.mark.parametrize("name", FILES)
def test_roundtrip_is_byte_identical(name):
    text = (PFG / name).read_text()
    assert pfg.dumps(pfg.loads(text)) == text


@pytest.mark.parametrize("name", SRC)
def test_vectorizer_emits_the_reference_graph(name):
    """pfor conversion of the reference's source graph reproduces the
    reference's vectorized graph text exactly (ids, attrs, constants)."""
    g2, _ = vectorize_graph(pfg.load(PFG / f"src_{name}.pfg"))
    assert pfg.dumps(g2) == (PFG / f"vec_{name}.pfg").read_text()


@pytest.mark.parametrize("name", SRC)
def test_loaded_vectorized_graph_runs_to_reference_outputs(name, golden):
    P = golden["programs"]
    got = OracleExecutor(pfg.load(PFG / f"vec_{name}.pfg")).run()
    for j, o in enumerate(got):
        np.testing.assert_allclose(np.asarray(o.data, np.float64), P[f"we_{name}/out/{j}"],
                                   rtol=0, atol=1e-12)


@pytest.mark.parametrize("fname", sorted(PROGS))
def test_loaded_program_runs_to_reference_outputs(fname, golden):
    P = golden["programs"]
    case = PROGS[fname]
    g = pfg.load(PFG / fname)
    feeds = {k.split("/")[-1]: P[k] for k in P if k.startswith(f"{case}/feed/")}
    feeds = {k: (v.astype(np.float64) if v.dtype == np.float32 else v) for k, v in feeds.items()}
    got = OracleExecutor(g).run(feeds=feeds)
    for j, o in enumerate(got):
        np.testing.assert_allclose(np.asarray(o.data, np.float64), P[f"{case}/out/{j}"],
                                   rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("text", ["%0 = constant[value=f64[2]{1.0,2.0}](\n",
                                  "%0 = add(%1, %2)\noutputs(%0)\n",
                                  "%0 = constant[value=f64[]{1.0}]()\noutputs(%0) junk\n",
                                  "%0 = constant[value=f64[]{1.0}]() $\n"])
def test_malformed_text_raises_parse_error(text):
    with pytest.raises(ParseError):
        pfg.loads(text)
