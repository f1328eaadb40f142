"""Row-window sharded training step on the GPU (world size 2, both ranks on
cuda:0, gloo collectives staged through the host): every sparse kernel runs
on its window range / row slab / edge range exactly as under NCCL on 8 GPUs.
The sharded AGNN and GCN forward + backward must match the unsharded run
(same weights) within the TF32 tolerance, and the sharded bench runs."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200 import dist as tdist, layers

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    torch.backends.cuda.matmul.allow_tf32 = False
    g = tcg.synth.gen_uniform(6000, 7, 4)
    cfg = tcg.BlockConfig()
    t = tcg.translate(g, cfg)
    plan = tdist.make_shard_plan(g.node_pointer, g.num_nodes, 16, rank=rank, world=world)
    shard = tdist.Shard.build(g, cfg, plan)
    # the rank's SGT shards are the whole-graph SGT restricted to its windows
    (w0, w1), (e0, e1) = plan.my_windows, plan.my_edges
    sgt_ok = (np.array_equal(shard.t.col_offsets[w0:w1 + 1], t.col_offsets[w0:w1 + 1])
              and np.array_equal(shard.t.edge_to_col[e0:e1], t.edge_to_col[e0:e1])
              and shard.t.num_unique == t.num_unique)
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((6000, 48)).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.integers(0, 5, 6000)).cuda()
    y47 = torch.from_numpy(rng.integers(0, 47, 6000)).cuda()
    res = {"sgt_ok": bool(sgt_ok)}
    # gcn47: an odd class count (padded-stride rows through the sharded path)
    for kind in ("agnn", "gcn", "gcn47"):
        grads = []
        for sh in (None, shard):
            torch.manual_seed(0)
            net = (layers.AGNN(48, 32, 5, layers=2) if kind == "agnn"
                   else layers.GCN(48, 16, 47 if kind == "gcn47" else 5)).cuda()
            lab = y47 if kind == "gcn47" else y
            if sh is None:
                loss = layers.cross_entropy(net(x, t), lab)
                loss.backward()
                lv = float(loss)
            else:
                # logits + sharded loss, and the output layer fused into the loss
                loss = (layers.cross_entropy_sharded(net(x, t, sh), lab, sh) if kind == "gcn"
                        else net.loss(x, t, lab, sh))
                loss.backward()
                sh.allreduce_grads(net.parameters())
                lt = loss.detach().cpu().reshape(1)
                dist.all_reduce(lt)
                lv = float(lt)
            grads.append([lv] + [p.grad.detach().cpu().numpy() for p in net.parameters()])
        ref, got = grads
        res[kind] = {
            "loss": [ref[0], got[0]],
            "rel": max(float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))
                       for a, b in zip(ref[1:], got[1:])),
        }
    (Path(out_dir) / f"rank{rank}.json").write_text(json.dumps(res))
    dist.destroy_process_group()


def test_sharded_train_step_matches_unsharded(tmp_path):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        res = json.loads((tmp_path / f"rank{r}.json").read_text())
        assert res.pop("sgt_ok") is True
        for kind, v in res.items():
            assert abs(v["loss"][0] - v["loss"][1]) <= 1e-4 * max(1.0, abs(v["loss"][0])), kind
            assert v["rel"] <= 5e-3, (kind, v)


def test_sharded_bench_runs():
    """bench.py --gpus 2 under torchrun with two ranks sharing cuda:0 (gloo):
    a functional check of the sharded bench path; the number is not a bench value."""
    env = dict(os.environ, TCG_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline", "--no-extras", "--workload", "pubmed-gcn"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["parallelism"] == "row-window shards x2"


_NCCL_SCRIPT = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch
import torch.distributed as dist
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import dist as tdist, layers
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=sys.argv[2])
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
torch.backends.cuda.matmul.allow_tf32 = False
g = tcg.synth.gen_uniform(5000, 8, 6)
cfg = tcg.BlockConfig()
t = tcg.translate(g, cfg)
plan = tdist.make_shard_plan(g.node_pointer, g.num_nodes, 16, rank=0, world=1)
shard = tdist.Shard.build(g, cfg, plan)
rng = np.random.default_rng(1)
x = torch.from_numpy(rng.standard_normal((5000, 40)).astype(np.float32)).cuda()
y = torch.from_numpy(rng.integers(0, 6, 5000)).cuda()
out = {}
for kind in ("agnn", "gcn"):
    nets = []
    for sh in (None, shard):
        torch.manual_seed(0)
        nets.append((layers.AGNN(40, 32, 6, layers=2) if kind == "agnn" else layers.GCN(40, 16, 6)).cuda())
    ref, net = nets
    loss = layers.cross_entropy(ref(x, t), y)
    loss.backward()
    opt = torch.optim.Adam(net.parameters(), lr=0.0, capturable=True, fused=True)

    def step():
        opt.zero_grad(set_to_none=False)
        lo = net.loss(x, t, y, shard)
        lo.backward()
        shard.allreduce_grads(net.parameters())
        opt.step()
        return lo.detach()

    for p in net.parameters():
        p.grad = torch.zeros_like(p)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            step()
    torch.cuda.current_stream().wait_stream(side)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        ls = step()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    rel = max(float((a.grad - b.grad).norm() / b.grad.norm().clamp_min(1e-30))
              for a, b in zip(net.parameters(), ref.parameters()))
    out[kind] = [float(loss), float(ls), rel]
print(json.dumps(out))
dist.destroy_process_group()
"""


def test_nccl_world1_captured_sharded_step():
    """The sharded step under a real NCCL communicator (world size 1 on the
    1-GPU lease): in-place all-gathers, the edge exchange and the gradient
    all-reduce captured in one CUDA graph and replayed; loss and gradients
    equal the unsharded eager step (lr 0, so replays keep the weights)."""
    r = subprocess.run([sys.executable, "-c", _NCCL_SCRIPT, str(ROOT), str(_free_port())],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for kind, (l_ref, l_got, rel) in res.items():
        assert abs(l_ref - l_got) <= 1e-4 * max(1.0, abs(l_ref)), (kind, l_ref, l_got)
        assert rel <= 5e-3, (kind, rel)


def test_sharded_bench_runs_with_extras():
    """bench.py --gpus 2 (gloo, both ranks on cuda:0) with the per-shard
    roofline / SGT extras: a functional check, not a bench value."""
    env = dict(os.environ, TCG_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline", "--workload", "pubmed-gcn"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["roofline"]["achieved"] > 0 and line["extras"]["sgt_ms"] > 0
