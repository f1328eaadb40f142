#!/usr/bin/env python3
"""Golden fixtures for the command-line harness,
produced by running the REFERENCE `tcg` CLI itself:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cli.py

Writes tests/golden/cli/: input graphs made by the reference `tcg gen`
(edge lists) plus two hand-written Matrix Market files, and cli.json with the
reference's stdout for `stats`, `translate` and `run` on them and the CSR
arrays its loaders produce (cli_graphs.npz). Run in the build container only.
"""

from __future__ import annotations

import contextlib
import io
import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from tcgraph import cli as rcli  # noqa: E402  (reference, read-only)
from tcgraph import io as rio  # noqa: E402

OUT = Path(__file__).resolve().parent / "cli"

MTX_SYM = """%%MatrixMarket matrix coordinate real symmetric
% hand-written: symmetric, duplicate entry, diagonal
5 5 6
1 2 0.5
2 3 1.5
3 3 2.0
4 1 -1.0
5 4 0.25
1 2 0.5
"""
MTX_PAT = """%%MatrixMarket matrix coordinate pattern general
% hand-written pattern matrix with an isolated node
40 40 7
1 2
2 1
3 30
30 3
17 17
40 1
1 40
"""


def run(argv):
    buf, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
        rc = rcli.main(argv)
    return rc, buf.getvalue(), err.getvalue()


def main():
    OUT.mkdir(exist_ok=True)
    gens = [("uniform300", ["--model", "uniform", "--n", "300", "--avg-degree", "6", "--seed", "7"]),
            ("powerlaw500", ["--model", "powerlaw", "--n", "500", "--avg-degree", "5", "--seed", "3"]),
            ("blockdense64", ["--model", "blockdense", "--n", "64", "--blocks-per-window", "3",
                              "--seed", "1"])]
    meta = {"gen": {}, "stats": {}, "translate": {}, "run": {}}
    for name, args in gens:
        path = OUT / f"{name}.txt"
        rc, out, _ = run(["gen", *args, "--out", str(path)])
        assert rc == 0, out
        meta["gen"][name] = {"argv": args, "stdout": out.strip().replace(str(path), "<path>")}
    (OUT / "sym5.mtx").write_text(MTX_SYM)
    (OUT / "pattern40.mtx").write_text(MTX_PAT)
    files = ["uniform300.txt", "powerlaw500.txt", "blockdense64.txt", "sym5.mtx", "pattern40.mtx"]
    arrays = {}
    for f in files:
        g = rio.load_graph(OUT / f)
        key = Path(f).stem
        arrays[f"{key}_ptr"] = g.node_pointer
        arrays[f"{key}_cols"] = g.edge_list
        if g.edge_values is not None:
            arrays[f"{key}_vals"] = g.edge_values
        for blk in (["--blk-h", "16", "--blk-w", "8"], ["--blk-h", "8", "--blk-w", "4"]):
            rc, out, _ = run(["stats", "--input", str(OUT / f), *blk])
            meta["stats"][f"{key}:{blk[1]}x{blk[3]}"] = {"rc": rc, "stdout": out}
        rc, out, _ = run(["translate", "--input", str(OUT / f)])
        meta["translate"][key] = {"rc": rc, "stdout": out.split(" sgt_ms=")[0]}
        for kernel in ("spmm", "sddmm", "gcn", "agnn"):
            for prec in ("f32", "tf32"):
                rc, out, _ = run(["run", kernel, "--input", str(OUT / f), "--dim", "16",
                                  "--precision", prec, "--repeat", "1"])
                header, row = out.strip().splitlines()
                cols = dict(zip(header.split(","), row.split(",")))
                cols.pop("avg_ms")
                meta["run"][f"{key}:{kernel}:{prec}"] = {"rc": rc, "fields": cols}
    # TCGT input to stats (structure-only tiling)
    tpath = OUT / "uniform300.tcgt"
    run(["translate", "--input", str(OUT / "uniform300.txt"), "--out", str(tpath)])
    rc, out, _ = run(["stats", "--input", str(tpath)])
    meta["stats"]["uniform300.tcgt"] = {"rc": rc, "stdout": out}
    # error paths
    (OUT / "bad.txt").write_text("0 1\n1 x\n")
    rc, out, err = run(["stats", "--input", str(OUT / "bad.txt")])
    meta["errors"] = {"bad.txt": {"rc": rc, "stderr": err.strip().replace(str(OUT), "<dir>")}}
    rc, out, err = run(["run", "spmm", "--input", str(tpath)])
    meta["errors"]["run_tcgt"] = {"rc": rc, "stderr": err.strip().replace(str(OUT), "<dir>")}
    np.savez_compressed(OUT / "cli_graphs.npz", **arrays)
    (OUT / "cli.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
