"""8(f) rows on the GPU: device graph normalisation (tcg_from_edges), device
invariant checks (tcg_validate), device tile accounting
(tcg_structure_blocks) and TCGT from a GPU SGT — against fixtures produced by
the reference itself (tests/golden/make_golden_graphops.py)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2112_02052_b200 as tcg

    return tcg, torch


@pytest.fixture(scope="module")
def ops():
    return np.load(GOLD / "graphops.npz"), json.loads((GOLD / "graphops.json").read_text())


def test_from_edges_device_bit_exact(env, ops):
    tcg, torch = env
    arr, meta = ops
    for c in meta["from_edges"]:
        k = c["name"]
        vals = arr[f"fe_{k}_vals"] if c["values"] else None
        g = tcg.CsrGraph.from_edges(arr[f"fe_{k}_src"], arr[f"fe_{k}_dst"], c["n"], values=vals,
                                    device="cuda")
        assert isinstance(g, tcg.DeviceCsrGraph)
        assert np.array_equal(g.node_pointer, arr[f"fe_{k}_ptr"]), k
        assert np.array_equal(g.edge_list, arr[f"fe_{k}_cols"]), k
        if c["values"]:
            assert np.array_equal(g.edge_values, arr[f"fe_{k}_out_vals"]), k


def test_from_edges_device_tensor_inputs_and_errors(env):
    tcg, torch = env
    src = torch.randint(0, 1000, (20000,), device="cuda")
    dst = torch.randint(0, 1000, (20000,), device="cuda")
    g = tcg.CsrGraph.from_edges(src, dst, 1000)
    h = tcg.CsrGraph.from_edges(src.cpu().numpy(), dst.cpu().numpy(), 1000)
    assert np.array_equal(g.node_pointer, h.node_pointer)
    assert np.array_equal(g.edge_list, h.edge_list)
    assert tcg.validate(g) == []
    with pytest.raises(ValueError, match="outside"):
        tcg.CsrGraph.from_edges(np.array([0, 5]), np.array([1, 1]), 3, device="cuda")
    with pytest.raises(ValueError, match="same length"):
        tcg.CsrGraph.from_edges(np.array([0, 1]), np.array([1]), 3, device="cuda")


def test_from_edges_products_scale(env):
    """Products-shaped edge list (2.45M nodes, 61.9M pairs) normalised on the
    GPU; sortedness and counts checked by the device validator and against
    the SGT digests' input (same generator, same dedup)."""
    tcg, torch = env
    n = 2449029
    gen = torch.Generator(device="cuda").manual_seed(1)
    src = torch.randint(0, n, (61859140,), device="cuda", generator=gen)
    dst = torch.randint(0, n, (61859140,), device="cuda", generator=gen)
    g = tcg.CsrGraph.from_edges(src, dst, n)
    assert tcg.validate(g, device="cuda") == []
    m = g.num_edges
    assert 61_000_000 < m <= 61859140
    # unique-pair count cross-check with torch.unique on the packed keys
    key = src * n + dst
    assert int(torch.unique(key).numel()) == m


def test_validate_device_messages(env, ops):
    tcg, torch = env
    arr, meta = ops
    for c in meta["validate"]:
        k = c["name"]
        g = tcg.CsrGraph(200, arr[f"va_{k}_ptr"], arr[f"va_{k}_cols"])
        assert tcg.validate(g, device="cuda") == c["messages"], k


def test_block_counts_device(env, ops):
    tcg, torch = env
    arr, meta = ops
    for c in meta["blocks"]:
        gn = c["graph"]
        g = tcg.CsrGraph(c["n"], arr[f"tb_{gn}_ptr"], arr[f"tb_{gn}_cols"])
        cfg = tcg.BlockConfig(blk_h=c["blk_h"], blk_w=c["blk_w"])
        tot, per = tcg.count_blocks_before(g, cfg, device="cuda")
        assert tot == c["total"]
        assert np.array_equal(per, arr[f"tb_{gn}_{c['blk_h']}x{c['blk_w']}_per"])
        t = tcg.translate(g, cfg)
        for w, want in c["structure"].items():
            assert tcg.structure_blocks_before(t, int(w)) == want
        assert tcg.count_blocks_after(t) == c["after"]


def test_tcgt_from_gpu_sgt(env, tmp_path):
    tcg, torch = env
    from paper_2112_02052_b200 import io

    g = tcg.synth.gen_uniform(100, 4, 42)
    t = tcg.translate(g, tcg.BlockConfig())
    assert io.tcgt_bytes(t) == (GOLD / "uniform100.tcgt").read_bytes()
    io.write_tcgt(t, tmp_path / "u.tcgt")
    t2 = io.read_tcgt(tmp_path / "u.tcgt", device="cuda")
    assert tcg.structure_blocks_before(t2, 8) == tcg.count_blocks_before(g, tcg.BlockConfig())[0]
    for k in ("win_partition", "edge_to_col", "col_offsets", "col_to_node"):
        assert np.array_equal(getattr(t2, k), getattr(t, k))


def test_edge_to_row_device(env):
    tcg, torch = env
    for n, deg, bh in ((1000, 5, 16), (777, 9, 8), (50, 2, 32)):
        g = tcg.synth.gen_uniform(n, deg, 3)
        t = tcg.translate(g, tcg.BlockConfig(blk_h=bh, blk_w=8))
        want = np.concatenate([t.window_edge_rows(w) for w in range(t.num_row_windows)])
        assert np.array_equal(t.edge_to_row.astype(np.int64), want)
