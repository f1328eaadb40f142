"""Row-window shards of SGT ("SGT runs per shard"): every
shard translated on its own (tcg_sgt_count_range / tcg_sgt_fill_range) with
base = the exclusive scan of the lower shards' totals must reproduce the
whole-graph GPU SGT -- and so the reference translate (sgt.py:101-137) --
bit for bit on its windows and edges, for ragged shard boundaries, empty
shards, hub windows (> 512 edges: the CTA path) and every tile shape. Also
pins the warp-level ranking path against the round-1 CTA path
(TCG_SGT_CTA=1) through the golden digests' shapes."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _hub_graph(tcg, n, deg, seed):
    rng = np.random.default_rng(seed)
    src = np.concatenate([rng.integers(0, n, n * deg), np.repeat(np.arange(4), 700)])
    dst = np.concatenate([rng.integers(0, n, n * deg), rng.integers(0, n, 2800)])
    return tcg.CsrGraph.from_edges(src, dst, n)


@pytest.mark.parametrize("kind,parts,bh,bw", [
    ("uniform", 2, 16, 8), ("uniform", 3, 16, 8), ("uniform", 8, 16, 8),
    ("hub", 3, 16, 8), ("powerlaw", 4, 16, 8), ("uniform", 3, 8, 4), ("hub", 2, 32, 16),
])
def test_sharded_sgt_equals_whole_graph(oracle, kind, parts, bh, bw):
    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200.sgt import ShardSgt

    n = 4099
    g = (tcg.synth.gen_uniform(n, 9, 5) if kind == "uniform"
         else tcg.synth.gen_powerlaw(n, 9, 5) if kind == "powerlaw" else _hub_graph(tcg, n, 9, 5))
    cfg = tcg.BlockConfig(bh, bw)
    whole = tcg.translate(g, cfg)
    W = whole.num_row_windows
    cuts = np.linspace(0, W, parts + 1).astype(int)
    cuts[1] = cuts[1] // 2  # a ragged, small first shard
    base = 0
    for wb, we in zip(cuts[:-1], cuts[1:]):
        sh = ShardSgt(g, cfg, (int(wb), int(we))).count()
        total = int(sh.total.item())
        t = sh.fill(base)
        co, wco = t.col_offsets, whole.col_offsets
        assert np.array_equal(co[wb:we + 1], wco[wb:we + 1])
        assert np.array_equal(t.win_partition[wb:we], whole.win_partition[wb:we])
        e0, e1 = g.node_pointer[min(wb * bh, n)], g.node_pointer[min(we * bh, n)]
        assert np.array_equal(t.edge_to_col[e0:e1], whole.edge_to_col[e0:e1])
        u0, u1 = int(wco[wb]), int(wco[we])
        c2n = t.dev["col_to_node"][u0:u1].cpu().numpy().view(np.uint32)
        assert np.array_equal(c2n, whole.col_to_node[u0:u1])
        assert total == u1 - u0
        base += total
    assert base == whole.num_unique
    ref = oracle.translate(g.node_pointer, g.edge_list, n, bh, bw)
    assert np.array_equal(whole.edge_to_col, ref[1]) and np.array_equal(whole.col_to_node, ref[3])


def test_empty_shard_and_bad_range():
    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200.sgt import ShardSgt

    g = tcg.synth.gen_uniform(500, 4, 1)
    cfg = tcg.BlockConfig()
    sh = ShardSgt(g, cfg, (10, 10)).count()
    assert int(sh.total.item()) == 0
    with pytest.raises(IndexError):
        ShardSgt(g, cfg, (5, 40))


_CTA_SCRIPT = r"""
import sys, hashlib, json
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2112_02052_b200 as tcg
out = {}
for name, (n, deg) in {"a": (20000, 7), "b": (3000, 40), "c": (1000, 300)}.items():
    g = tcg.synth.gen_uniform(n, deg, 3)
    t = tcg.translate(g, tcg.BlockConfig())
    out[name] = [hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
                 for a in (t.win_partition, t.edge_to_col, t.col_offsets, t.col_to_node)]
print(json.dumps(out))
"""


def test_warp_path_equals_cta_path():
    """Windows of 7 / 40 / 300 edges per row (K = 8, 16 and the CTA fallback)
    through the warp ranking path and the round-1 CTA path: same bytes."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    res = []
    for env in ({}, {"TCG_SGT_CTA": "1"}):
        r = subprocess.run([sys.executable, "-c", _CTA_SCRIPT, str(ROOT)],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert res[0] == res[1]
