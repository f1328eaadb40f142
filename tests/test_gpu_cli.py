"""CLI harness on the GPU: `stats`, `translate` and
`run --engine b200` print what the reference `tcg` printed on the same files
(tests/golden/make_golden_cli.py). Timings and the error column (measured
against a different exact path) are the only fields not compared."""

from __future__ import annotations

import contextlib
import io
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "cli"
META = json.loads((GOLD / "cli.json").read_text())
FILES = ["uniform300.txt", "powerlaw500.txt", "blockdense64.txt", "sym5.mtx", "pattern40.mtx"]


def _run(argv):
    from paper_2112_02052_b200 import cli

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


@pytest.mark.parametrize("f", FILES)
@pytest.mark.parametrize("bh,bw", [(16, 8), (8, 4)])
def test_stats(f, bh, bw):
    rc, out, _ = _run(["stats", "--input", str(GOLD / f), "--blk-h", str(bh), "--blk-w", str(bw)])
    ref = META["stats"][f"{Path(f).stem}:{bh}x{bw}"]
    assert rc == ref["rc"] and out == ref["stdout"]


def test_stats_from_tcgt():
    rc, out, _ = _run(["stats", "--input", str(GOLD / "uniform300.tcgt")])
    ref = META["stats"]["uniform300.tcgt"]
    assert rc == ref["rc"] and out == ref["stdout"]


@pytest.mark.parametrize("f", FILES)
def test_translate(f, tmp_path):
    out_t = tmp_path / "t.tcgt"
    rc, out, _ = _run(["translate", "--input", str(GOLD / f), "--out", str(out_t)])
    ref = META["translate"][Path(f).stem]
    assert rc == ref["rc"] and out.split(" sgt_ms=")[0] == ref["stdout"]
    if f == "uniform300.txt":
        assert out_t.read_bytes() == (GOLD / "uniform300.tcgt").read_bytes()


@pytest.mark.parametrize("f", FILES)
@pytest.mark.parametrize("kernel", ["spmm", "sddmm", "gcn", "agnn"])
@pytest.mark.parametrize("prec", ["f32", "tf32"])
def test_run(f, kernel, prec):
    rc, out, err = _run(["run", kernel, "--input", str(GOLD / f), "--dim", "16",
                         "--precision", prec, "--repeat", "2", "--engine", "b200"])
    ref = META["run"][f"{Path(f).stem}:{kernel}:{prec}"]
    header, row = out.strip().splitlines()
    cols = dict(zip(header.split(","), row.split(",")))
    assert rc == ref["rc"] == 0, err
    cols.pop("avg_ms")
    err_col = cols.pop("max_rel_err_vs_oracle")
    want = dict(ref["fields"])
    want.pop("max_rel_err_vs_oracle")
    assert cols == want
    if prec == "f32" and kernel in ("spmm", "sddmm"):
        assert float(err_col) == 0.0  # the f32 engine is the bitwise reference fold
