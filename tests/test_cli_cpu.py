"""CLI harness host side against fixtures made by the
reference `tcg` CLI (tests/golden/make_golden_cli.py): `gen` writes the same
files byte for byte, the edge-list / Matrix Market loaders build the same
CSR, and the error paths print the same messages with the same exit codes."""

from __future__ import annotations

import contextlib
import io
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2112_02052_b200 import cli
from paper_2112_02052_b200 import io as gio

GOLD = Path(__file__).resolve().parent / "golden" / "cli"
META = json.loads((GOLD / "cli.json").read_text())
ARR = np.load(GOLD / "cli_graphs.npz")


def _run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


@pytest.mark.parametrize("name", sorted(META["gen"]))
def test_gen_matches_reference_bytes(tmp_path, name):
    path = tmp_path / f"{name}.txt"
    rc, out, _ = _run(["gen", *META["gen"][name]["argv"], "--out", str(path)])
    assert rc == 0
    assert out.strip().replace(str(path), "<path>") == META["gen"][name]["stdout"]
    assert path.read_bytes() == (GOLD / f"{name}.txt").read_bytes()


@pytest.mark.parametrize("f", ["uniform300.txt", "powerlaw500.txt", "blockdense64.txt",
                               "sym5.mtx", "pattern40.mtx"])
def test_loaders_match_reference(f):
    g = gio.load_graph(GOLD / f)
    key = Path(f).stem
    np.testing.assert_array_equal(g.node_pointer, ARR[f"{key}_ptr"])
    np.testing.assert_array_equal(g.edge_list, ARR[f"{key}_cols"])
    if f"{key}_vals" in ARR:
        np.testing.assert_array_equal(g.edge_values, ARR[f"{key}_vals"])
    else:
        assert g.edge_values is None


def test_error_paths_match_reference():
    rc, _, err = _run(["stats", "--input", str(GOLD / "bad.txt")])
    ref = META["errors"]["bad.txt"]
    assert rc == ref["rc"] and err.strip().replace(str(GOLD), "<dir>") == ref["stderr"]
    rc, _, err = _run(["run", "spmm", "--input", str(GOLD / "uniform300.tcgt")])
    ref = META["errors"]["run_tcgt"]
    assert rc == ref["rc"] and err.strip().replace(str(GOLD), "<dir>") == ref["stderr"]


@pytest.mark.parametrize("text,msg", [
    ("%%MatrixMarket matrix array real general\n2 2\n", "unsupported object/format"),
    ("%%MatrixMarket matrix coordinate complex general\n", "unsupported field"),
    ("%%MatrixMarket matrix coordinate real general\n2 3 0\n", "must be square"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "declared 2 entries"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n", "out of declared bounds"),
    ("0 1 2\n", "expected 'src dst'"),
    ("-1 2\n", "negative node id"),
])
def test_loader_errors(tmp_path, text, msg):
    p = tmp_path / ("g.mtx" if text.startswith("%%") else "g.txt")
    p.write_text(text)
    with pytest.raises(gio.GraphFormatError, match=msg):
        gio.load_graph(p)
