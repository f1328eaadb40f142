#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container only (it imports the read-only reference package
from /root/reference/pkg/src); the outputs are committed so the GPU box, which
has no /root/reference, can check against them:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

Fixtures written (all produced by calling the reference's public API):
  small_cases.npz   hand traces, the reference's structural test corpus and
                    seeded random small graphs x block configs: translate()
                    arrays, spmm/sddmm f32 + tf32 outputs, segment_softmax,
                    agnn_layer, gcn_layer (tcgraph/kernels.py, sgt.py).
  cora.npz          Cora-shaped uniform graph (2,708 / 10,858) at 16x8:
                    SGT arrays, spmm/sddmm f32+tf32 D=16, agnn_layer D=16.
  tf32_vectors.npz  quantize_tf32 (tiles.py:67-82) on specials, ties and
                    4,096 wide-range values.
  digests.json      sha256 of translate() arrays and of f32 spmm/sddmm
                    outputs at the full BASELINE shapes (arxiv, amazon0601;
                    products SGT with --big) -> size-independent bit-exact
                    checks on the GPU box.
  tiny.tcgt / uniform100.tcgt / tiny.tcem   reference io.write_tcgt/tcem
                    bytes (pkg/scripts/regen_goldens.py:18-31).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import tcgraph as tg  # noqa: E402  (reference, read-only)
from tcgraph import synth  # noqa: E402

OUT = Path(__file__).resolve().parent

# Dataset shapes (BASELINE.json configs).
SHAPES = {
    "cora": (2708, 10858),
    "pubmed": (19717, 88676),
    "arxiv": (169343, 1166243),
    "amazon0601": (403394, 3387388),
    "products": (2449029, 61859140),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def emb(n, d, seed):
    return np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)


def small_graphs():
    """(name, graph) list: hand trace + reference corpus (tests/conftest.py:38-57)
    + determinism corpus (tests/test_acceptance.py:62-72) + random small."""
    g = [
        ("four_node", tg.CsrGraph.from_edges([0, 0, 1, 2], [0, 3, 3, 1], 4)),
        ("empty_3", tg.CsrGraph.from_edges([], [], 3)),
        ("empty_48", tg.CsrGraph.from_edges([], [], 48)),
        ("single_self_loop", tg.CsrGraph.from_edges([0], [0], 1)),
        ("identity_37", tg.CsrGraph.from_edges(np.arange(37), np.arange(37), 37)),
        ("complete_2", tg.CsrGraph.from_edges([0, 0, 1, 1], [0, 1, 0, 1], 2)),
        ("uniform_300", synth.gen_uniform(300, 4, 11)),
        ("uniform_1000", synth.gen_uniform(1000, 8, 12)),
        ("powerlaw_500", synth.gen_powerlaw(500, 6, 13)),
        ("blockdense_8w", synth.gen_blockdense(8, 3, 16, 14)),
        ("ragged_45", synth.gen_uniform(45, 3, 15)),
        ("uniform_600", synth.gen_uniform(600, 8, 31)),
        ("powerlaw_400", synth.gen_powerlaw(400, 6, 32)),
        ("blockdense_33", synth.gen_blockdense(8, 3, 16, 33)),
        ("orth_pair", tg.CsrGraph.from_edges([0], [1], 2)),
        ("star_in_200", tg.CsrGraph.from_edges(np.arange(200), np.zeros(200, int), 200)),
        ("star_out_200", tg.CsrGraph.from_edges(np.zeros(200, int), np.arange(200), 200)),
        ("dense_row_window_64", tg.CsrGraph.from_edges(
            np.repeat(np.arange(16), 600), np.tile(np.arange(600), 16) * 3 % 1999, 2000)),
    ]
    rng = np.random.default_rng(2112)
    for i in range(24):
        n = int(rng.integers(1, 41))
        m = int(rng.integers(0, 121))
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        g.append((f"rand_{i}", tg.CsrGraph.from_edges(src, dst, n)))
    return g


def gen_small_cases() -> None:
    cfgs = [(16, 8), (7, 3), (5, 3), (2, 2), (1, 1), (9, 4)]
    arrays: dict[str, np.ndarray] = {}
    meta = []
    k = 0
    for name, g in small_graphs():
        n = g.num_nodes
        for bh, bw in cfgs:
            if n >= 300 and (bh, bw) not in ((16, 8), (7, 3)):
                continue  # keep the committed fixture small
            t = tg.translate(g, tg.BlockConfig(bh, bw))
            p = f"c{k}_"
            arrays[p + "ptr"] = g.node_pointer
            arrays[p + "cols"] = g.edge_list
            arrays[p + "win_partition"] = t.win_partition
            arrays[p + "edge_to_col"] = t.edge_to_col
            arrays[p + "col_offsets"] = t.col_offsets
            arrays[p + "col_to_node"] = t.col_to_node
            arrays[p + "paired"] = tg.paired_block_counts(t)
            d_spmm = 1 + (k % 19)
            d_sddmm = 1 + ((k * 7) % 23)
            x = emb(n, d_spmm, 100 + k)
            xs = emb(n, d_sddmm, 200 + k)
            f = np.random.default_rng(300 + k).standard_normal(g.num_edges).astype(np.float32)
            # inputs are regenerated from their seeds by the tests (emb() /
            # default_rng(300+k)); only outputs are stored
            arrays[p + "spmm_f32"] = tg.spmm(t, x)
            arrays[p + "spmm_w_f32"] = tg.spmm(t, x, f=f)
            arrays[p + "sddmm_f32"] = tg.sddmm(t, xs)
            scores = tg.sddmm(t, xs)
            arrays[p + "softmax"] = tg.segment_softmax(scores, g.node_pointer)
            arrays[p + "agnn_f32"] = tg.agnn_layer(t, x)
            if (bh, bw) == (16, 8):
                arrays[p + "spmm_tf32"] = tg.spmm(t, x, mode="tf32")
                arrays[p + "spmm_w_tf32"] = tg.spmm(t, x, f=f, mode="tf32")
                arrays[p + "sddmm_tf32"] = tg.sddmm(t, xs, mode="tf32")
                arrays[p + "agnn_tf32"] = tg.agnn_layer(t, x, mode="tf32")
                w = emb(d_spmm, 3, 400 + k)
                b = emb(1, 3, 500 + k)[0]
                arrays[p + "gcn_f32"] = tg.gcn_layer(t, x, w, b)
            c_sp, c_sd, c_ag = tg.Counters(), tg.Counters(), tg.Counters()
            tg.spmm(t, x, counters=c_sp)
            tg.sddmm(t, xs, counters=c_sd)
            tg.agnn_layer(t, x, counters=c_ag)
            meta.append(
                dict(
                    key=p, name=name, n=n, m=g.num_edges, blk_h=bh, blk_w=bw,
                    d_spmm=d_spmm, d_sddmm=d_sddmm, seed_x=100 + k, seed_xs=200 + k,
                    seed_f=300 + k, seed_w=400 + k, seed_b=500 + k,
                    counters_spmm=[c_sp.tiles_visited, c_sp.mma_calls, c_sp.bytes_gathered],
                    counters_sddmm=[c_sd.tiles_visited, c_sd.mma_calls, c_sd.bytes_gathered],
                    counters_agnn=[c_ag.tiles_visited, c_ag.mma_calls, c_ag.bytes_gathered],
                    warps_per_block=tg.make_plan(t, d_spmm).warps_per_block,
                    blocks_before=tg.count_blocks_before(g, tg.BlockConfig(bh, bw))[0],
                )
            )
            k += 1
    np.savez_compressed(OUT / "small_cases.npz", **arrays)
    (OUT / "small_cases.json").write_text(json.dumps(meta, indent=1))
    print(f"small_cases: {k} cases")


def gen_cora() -> None:
    n, m = SHAPES["cora"]
    g = synth.gen_uniform(n, m / n, seed=1)
    t = tg.translate(g, tg.BlockConfig())
    x = synth.random_embeddings(n, 16, seed=2)
    f = np.random.default_rng(3).random(g.num_edges).astype(np.float32)
    a = dict(
        ptr=g.node_pointer, cols=g.edge_list,
        win_partition=t.win_partition, edge_to_col=t.edge_to_col,
        col_offsets=t.col_offsets, col_to_node=t.col_to_node,
        x=x, f=f,
        spmm_f32=tg.spmm(t, x), spmm_tf32=tg.spmm(t, x, mode="tf32"),
        spmm_w_f32=tg.spmm(t, x, f=f), spmm_w_tf32=tg.spmm(t, x, f=f, mode="tf32"),
        sddmm_f32=tg.sddmm(t, x), sddmm_tf32=tg.sddmm(t, x, mode="tf32"),
        agnn_f32=tg.agnn_layer(t, x), agnn_tf32=tg.agnn_layer(t, x, mode="tf32"),
    )
    np.savez_compressed(OUT / "cora.npz", **a)
    print("cora: M =", g.num_edges)


def gen_tf32() -> None:
    special = np.array(
        [0.0, -0.0, 1.0, -2.5, 0.1, np.inf, -np.inf, np.nan, 3.4028235e38, -3.4028235e38,
         1e-45, -1e-45, 1.1754944e-38, 65504.0, 1.0000001, 1.00012207, 1.00036621],
        dtype=np.float32,
    )
    # exact ties at the 13-bit boundary, both parities of the kept lsb
    base = np.arange(64, dtype=np.uint32) << np.uint32(13)
    ties = ((np.uint32(0x3F800000) + base) | np.uint32(0x1000)).view(np.float32)
    rng = np.random.default_rng(0)
    wide = (rng.standard_normal(4096) * 10.0 ** rng.integers(-20, 20, 4096)).astype(np.float32)
    bits = (
        rng.integers(0, 2, 8192, dtype=np.uint32) << np.uint32(31)
        | rng.integers(0, 256, 8192, dtype=np.uint32) << np.uint32(23)
        | rng.integers(0, 1 << 23, 8192, dtype=np.uint32)
    )
    allexp = bits.view(np.float32)
    x = np.concatenate([special, ties, wide, allexp])
    np.savez_compressed(OUT / "tf32_vectors.npz", x=x, q=tg.quantize_tf32(x))
    print("tf32 vectors:", x.size)


def gen_digests(big: bool) -> None:
    out = {}
    names = ["pubmed", "arxiv", "amazon0601"] + (["products"] if big else [])
    for name in names:
        n, m = SHAPES[name]
        t0 = time.time()
        g = synth.gen_uniform(n, m / n, seed=1)
        t1 = time.time()
        t = tg.translate(g, tg.BlockConfig())
        t2 = time.time()
        rec = dict(
            n=n, m=g.num_edges,
            ptr=sha(g.node_pointer), cols=sha(g.edge_list),
            win_partition=sha(t.win_partition), edge_to_col=sha(t.edge_to_col),
            col_offsets=sha(t.col_offsets), col_to_node=sha(t.col_to_node),
            num_unique=int(t.col_offsets[-1]), sum_wp=int(t.win_partition.sum()),
            sum_paired=int(tg.paired_block_counts(t).sum()),
            gen_s=round(t1 - t0, 2), sgt_s=round(t2 - t1, 2),
        )
        if name != "products":
            for d in (16, 32):
                x = synth.random_embeddings(n, d, seed=2)
                rec[f"spmm_f32_d{d}"] = sha(tg.spmm(t, x, workers=8))
                rec[f"sddmm_f32_d{d}"] = sha(tg.sddmm(t, x, workers=8))
        out[name] = rec
        print(name, rec["m"], rec["gen_s"], rec["sgt_s"], flush=True)
    (OUT / "digests.json").write_text(json.dumps(out, indent=1))


def gen_formats() -> None:
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        four = tg.CsrGraph.from_edges([0, 0, 1, 2], [0, 3, 3, 1], 4)
        tg.write_tcgt(tg.translate(four, tg.BlockConfig(2, 2)), d / "tiny.tcgt")
        x = np.array([[1, 0], [0, 1], [2, 2], [5, 5]], dtype=np.float32)
        tg.write_tcem(x, d / "tiny.tcem")
        tg.write_tcgt(tg.translate(synth.gen_uniform(100, 4, 42), tg.BlockConfig()),
                      d / "uniform100.tcgt")
        for f in ("tiny.tcgt", "tiny.tcem", "uniform100.tcgt"):
            (OUT / f).write_bytes((d / f).read_bytes())
            print(f, hashlib.sha256((OUT / f).read_bytes()).hexdigest()[:12])


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    gen_formats()
    gen_tf32()
    gen_small_cases()
    gen_cora()
    gen_digests("--big" in sys.argv)
