#!/usr/bin/env python3
"""Golden fixtures for the 8(f) rows (graph normalisation, invariants, tile
accounting), produced by calling the REFERENCE package itself:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_graphops.py

Writes tests/golden/graphops.npz (from_edges inputs/outputs, count_blocks_before
per-window counts) and graphops.json (validate() messages on corrupted graphs,
structure_blocks_before totals). Run in the build container only: the GPU box
has no /root/reference, it reads the committed outputs.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import tcgraph as tg  # noqa: E402  (reference, read-only)
from tcgraph import graph as rgraph  # noqa: E402
from tcgraph import sgt as rsgt  # noqa: E402
from tcgraph import synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"from_edges": [], "validate": [], "blocks": []}
    rng = np.random.default_rng(2024)
    # from_edges: duplicates, values, isolated rows, empty
    cases = [("dup_vals", 500, 4000, True), ("dup_novals", 300, 5000, False),
             ("sparse", 5000, 800, True), ("empty", 10, 0, True), ("one", 1, 3, True)]
    for name, n, m, with_vals in cases:
        src = rng.integers(0, n, m)
        dst = rng.integers(0, max(n // 3, 1), m)  # many duplicate pairs
        vals = rng.standard_normal(m).astype(np.float32) if with_vals else None
        g = rgraph.CsrGraph.from_edges(src, dst, n, values=vals)
        arrays[f"fe_{name}_src"] = src
        arrays[f"fe_{name}_dst"] = dst
        if vals is not None:
            arrays[f"fe_{name}_vals"] = vals
            arrays[f"fe_{name}_out_vals"] = g.edge_values
        arrays[f"fe_{name}_ptr"] = g.node_pointer
        arrays[f"fe_{name}_cols"] = g.edge_list
        meta["from_edges"].append({"name": name, "n": n, "values": with_vals})
    # validate(): corrupted graphs
    base = synth.gen_uniform(200, 5, 3)

    def msgs(ptr, cols, n=200, vals=None):
        g = rgraph.CsrGraph(n, ptr, cols, vals)
        return rgraph.validate(g)

    corruptions = {}
    p, c = base.node_pointer.copy(), base.edge_list.copy()
    corruptions["ok"] = (p, c)
    c2 = c.copy(); c2[7] = 500; c2[90] = 999; corruptions["oob"] = (p, c2)
    c3 = c.copy(); s = int(p[10]); c3[s], c3[s + 1] = c3[s + 1], c3[s]; corruptions["unsorted"] = (p, c3)
    c4 = c.copy(); s = int(p[20]); c4[s + 1] = c4[s]; c4[s + 2] = c4[s]; corruptions["dup"] = (p, c4)
    p5 = p.copy(); p5[50] = p5[52] + 3; corruptions["nonmono"] = (p5, c)
    p6 = p.copy(); p6[-1] -= 2; corruptions["bad_end"] = (p6, c)
    for k, (pp, cc) in corruptions.items():
        arrays[f"va_{k}_ptr"] = pp
        arrays[f"va_{k}_cols"] = cc
        meta["validate"].append({"name": k, "messages": msgs(pp, cc)})
    # tile accounting
    for (gn, n, deg, seed) in (("u1", 700, 6, 1), ("u2", 2000, 3, 5), ("pl", 1500, 8, 2)):
        g = synth.gen_uniform(n, deg, seed) if gn != "pl" else synth.gen_powerlaw(n, deg, seed)
        arrays[f"tb_{gn}_ptr"] = g.node_pointer
        arrays[f"tb_{gn}_cols"] = g.edge_list
        for bh, bw in ((16, 8), (8, 4), (32, 16)):
            cfg = rsgt.BlockConfig(blk_h=bh, blk_w=bw)
            tot, per = rsgt.count_blocks_before(g, cfg)
            t = rsgt.translate(g, cfg)
            arrays[f"tb_{gn}_{bh}x{bw}_per"] = per
            meta["blocks"].append({"graph": gn, "n": n, "blk_h": bh, "blk_w": bw, "total": tot,
                                   "structure": {str(w): rsgt.structure_blocks_before(t, w)
                                                 for w in (1, 8, 16, 64)},
                                   "after": rsgt.count_blocks_after(t)})
    np.savez_compressed(OUT / "graphops.npz", **arrays)
    (OUT / "graphops.json").write_text(json.dumps(meta, indent=1))
    print("wrote", OUT / "graphops.npz", OUT / "graphops.json")


if __name__ == "__main__":
    main()
