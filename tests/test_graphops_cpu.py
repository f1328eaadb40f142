"""8(f) rows on the host side: the package's host paths and the TCGT/TCEM
files against fixtures produced by the reference itself
(tests/golden/make_golden_graphops.py, make_golden.py)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import io
from paper_2112_02052_b200.sgt import TiledGraph

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def ops():
    return np.load(GOLD / "graphops.npz"), json.loads((GOLD / "graphops.json").read_text())


def test_from_edges_host_matches_reference(ops):
    arr, meta = ops
    for c in meta["from_edges"]:
        k = c["name"]
        vals = arr[f"fe_{k}_vals"] if c["values"] else None
        g = tcg.CsrGraph.from_edges(arr[f"fe_{k}_src"], arr[f"fe_{k}_dst"], c["n"], values=vals)
        assert np.array_equal(g.node_pointer, arr[f"fe_{k}_ptr"]), k
        assert np.array_equal(g.edge_list, arr[f"fe_{k}_cols"]), k
        if c["values"]:
            assert np.array_equal(g.edge_values, arr[f"fe_{k}_out_vals"]), k


def test_validate_host_messages(ops):
    arr, meta = ops
    for c in meta["validate"]:
        k = c["name"]
        g = tcg.CsrGraph(200, arr[f"va_{k}_ptr"], arr[f"va_{k}_cols"])
        assert tcg.validate(g) == c["messages"], k


def test_block_counts_host(ops, oracle):
    arr, meta = ops
    for c in meta["blocks"]:
        gn = c["graph"]
        g = tcg.CsrGraph(c["n"], arr[f"tb_{gn}_ptr"], arr[f"tb_{gn}_cols"])
        cfg = tcg.BlockConfig(blk_h=c["blk_h"], blk_w=c["blk_w"])
        tot, per = tcg.count_blocks_before(g, cfg)
        assert tot == c["total"]
        assert np.array_equal(per, arr[f"tb_{gn}_{c['blk_h']}x{c['blk_w']}_per"])
        # structure-only tiling (host arrays from the oracle SGT)
        wp, e2c, co, c2n = oracle.translate(g.node_pointer, g.edge_list, c["n"], c["blk_h"],
                                            c["blk_w"])
        t = TiledGraph(None, cfg, c["n"], g.num_edges, len(wp))
        t._host.update(win_partition=wp, edge_to_col=e2c, col_offsets=co, col_to_node=c2n)
        for w, want in c["structure"].items():
            assert tcg.structure_blocks_before(t, int(w)) == want
        assert tcg.count_blocks_after(t) == c["after"]


@pytest.mark.parametrize("name", ["tiny.tcgt", "uniform100.tcgt"])
def test_tcgt_golden_round_trip(name, tmp_path):
    raw = (GOLD / name).read_bytes()
    t = io.read_tcgt(GOLD / name)
    assert t.graph is None
    assert io.tcgt_bytes(t) == raw
    io.write_tcgt(t, tmp_path / name)
    assert (tmp_path / name).read_bytes() == raw


def test_tcgt_from_oracle_sgt_matches_golden(oracle):
    # uniform100.tcgt = translate(gen_uniform(100, 4, 42), BlockConfig()) (test_io.py:194-199)
    g = tcg.synth.gen_uniform(100, 4, 42)
    wp, e2c, co, c2n = oracle.translate(g.node_pointer, g.edge_list, 100, 16, 8)
    t = TiledGraph(None, tcg.BlockConfig(), 100, g.num_edges, len(wp))
    t._host.update(win_partition=wp, edge_to_col=e2c, col_offsets=co, col_to_node=c2n)
    assert io.tcgt_bytes(t) == (GOLD / "uniform100.tcgt").read_bytes()


def test_tcem_golden_round_trip(tmp_path):
    raw = (GOLD / "tiny.tcem").read_bytes()
    x = io.read_tcem(GOLD / "tiny.tcem")
    io.write_tcem(x, tmp_path / "x.tcem")
    assert (tmp_path / "x.tcem").read_bytes() == raw


def test_format_errors(tmp_path):
    raw = (GOLD / "uniform100.tcgt").read_bytes()
    cases = {"magic": b"XXXX" + raw[4:], "trunc": raw[:-3], "trail": raw + b"\0",
             "version": raw[:4] + (7).to_bytes(4, "little") + raw[8:]}
    msgs = {"magic": "bad magic", "trunc": "truncated file", "trail": "trailing bytes",
            "version": "unsupported format version 7"}
    for k, b in cases.items():
        p = tmp_path / f"{k}.tcgt"
        p.write_bytes(b)
        with pytest.raises(io.GraphFormatError, match=msgs[k]):
            io.read_tcgt(p)
    p = tmp_path / "bad.tcem"
    p.write_bytes((GOLD / "tiny.tcem").read_bytes()[:-1])
    with pytest.raises(io.GraphFormatError, match="truncated"):
        io.read_tcem(p)
    with pytest.raises(ValueError, match="2-D"):
        io.write_tcem(np.zeros(3, np.float32), tmp_path / "v.tcem")
