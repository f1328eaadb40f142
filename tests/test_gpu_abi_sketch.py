"""The SURVEY.md Appendix D entry points (tcg_sgt_count / tcg_sgt_fill,
tcg_softmax_fwd / tcg_softmax_bwd, tcg_agnn_fused_fwd), called through the C
ABI directly and checked against the oracle / the primary entry points."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest


pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200 import _lib

    return tcg, torch, _lib, _lib.load()


@pytest.fixture(scope="module")
def O():
    from oracle import tcg_oracle

    return tcg_oracle


def _s(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("bh,bw", [(16, 8), (1, 1), (3, 5), (32, 16)])
def test_sgt_two_phase_matches_oracle(env, O, bh, bw):
    tcg, torch, _lib, lib = env
    g = tcg.synth.gen_uniform(3000, 7.0, seed=11)
    ptr = torch.from_numpy(g.node_pointer.astype(np.int64)).cuda()
    cols = torch.from_numpy(g.edge_list.astype(np.int32)).cuda()
    n, m = g.num_nodes, g.num_edges
    W = -(-n // bh)
    e2c = torch.empty(m, dtype=torch.int32, device="cuda")
    offs = torch.empty(W + 1, dtype=torch.int64, device="cuda")
    wsb = int(lib.tcg_sgt_workspace_bytes(n, m, bh))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.tcg_sgt_count(ptr.data_ptr(), cols.data_ptr(), n, m, bh, bw, e2c.data_ptr(),
                                 offs.data_ptr(), ws.data_ptr(), wsb, _s(torch)), "count")
    u = int(offs[-1].item())
    c2n = torch.empty(u, dtype=torch.int32, device="cuda")
    wp = torch.empty(W, dtype=torch.int32, device="cuda")
    _lib.check(lib.tcg_sgt_fill(ptr.data_ptr(), cols.data_ptr(), n, m, bh, bw, e2c.data_ptr(),
                                offs.data_ptr(), wp.data_ptr(), c2n.data_ptr(), _s(torch)), "fill")
    r_wp, r_e2c, r_offs, r_c2n = O.translate(g.node_pointer, g.edge_list, n, bh, bw)
    np.testing.assert_array_equal(wp.cpu().numpy().view(np.uint32), r_wp)
    np.testing.assert_array_equal(e2c.cpu().numpy().view(np.uint32), r_e2c)
    np.testing.assert_array_equal(offs.cpu().numpy(), r_offs)
    np.testing.assert_array_equal(c2n.cpu().numpy().view(np.uint32), r_c2n)


def test_softmax_aliases(env, O):
    tcg, torch, _lib, lib = env
    g = tcg.synth.gen_uniform(2000, 6.0, seed=5)
    ptr = torch.from_numpy(g.node_pointer.astype(np.int64)).cuda()
    gen = torch.Generator(device="cuda").manual_seed(1)
    v = torch.randn(g.num_edges, device="cuda", generator=gen)
    dp = torch.randn(g.num_edges, device="cuda", generator=gen)
    a, b = torch.empty_like(v), torch.empty_like(v)
    n = g.num_nodes
    _lib.check(lib.tcg_segment_softmax(ptr.data_ptr(), n, v.data_ptr(), a.data_ptr(), _s(torch)),
               "")
    _lib.check(lib.tcg_softmax_fwd(ptr.data_ptr(), n, v.data_ptr(), b.data_ptr(), _s(torch)), "")
    assert torch.equal(a, b)
    ref = O.segment_softmax(v.cpu().numpy(), g.node_pointer)
    np.testing.assert_allclose(b.cpu().numpy(), ref, rtol=1e-5, atol=1e-7)
    _lib.check(lib.tcg_segment_softmax_backward(ptr.data_ptr(), n, b.data_ptr(), dp.data_ptr(),
                                                a.data_ptr(), _s(torch)), "")
    d2 = torch.empty_like(v)
    _lib.check(lib.tcg_softmax_bwd(ptr.data_ptr(), n, b.data_ptr(), dp.data_ptr(), d2.data_ptr(),
                                   _s(torch)), "")
    assert torch.equal(a, d2)


def test_agnn_fused_fwd_alias(env):
    tcg, torch, _lib, lib = env
    from paper_2112_02052_b200.kernels import agnn_forward_device

    g = tcg.synth.gen_uniform(5000, 8.0, seed=9)
    t = tcg.translate(g, tcg.BlockConfig())
    gen = torch.Generator(device="cuda").manual_seed(2)
    z = torch.randn(g.num_nodes, 32, device="cuda", generator=gen)
    y_ref, p_ref = agnn_forward_device(t, z)
    p = torch.empty(g.num_edges, device="cuda")
    y = torch.empty_like(z)
    _lib.check(lib.tcg_agnn_fused_fwd(C.byref(t.abi()), z.data_ptr(), 32, p.data_ptr(),
                                      y.data_ptr(), 32, _s(torch)), "tcg_agnn_fused_fwd")
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref) and torch.equal(p, p_ref[: g.num_edges])
