#!/usr/bin/env python3
"""Launch the hot kernels on the arxiv-shaped graph for ncu captures.

    ncu --set full --clock-control none --import-source on -k regex:spmm_tc \
        -s 2 -c 1 -o gpurun_out/prof python profiles/prof_kernels.py

Each kernel is launched 4 times (2 warm-up, then the captured ones).
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2112_02052_b200 as tcg  # noqa: E402
from paper_2112_02052_b200 import _lib  # noqa: E402
from paper_2112_02052_b200.kernels import (  # noqa: E402
    agnn_backward_device,
    agnn_forward_device,
    sddmm_device,
    spmm_device,
)


def main():
    shape = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    g = tcg.synth.shaped_graph(shape)
    t = tcg.translate(g, tcg.BlockConfig())
    tt = t.transpose()
    z = torch.randn(g.num_nodes, d, device="cuda")
    gy = torch.randn(g.num_nodes, d, device="cuda")
    p = sddmm_device(t, z, epilogue=_lib.EPI_SOFTMAX)
    out = torch.empty_like(z)
    ds = torch.empty_like(p)
    for _ in range(4):
        spmm_device(t, z, p, out=out)
        sddmm_device(t, z, epilogue=_lib.EPI_SOFTMAX, out=p)
        sddmm_device(t, gy, z, epilogue=_lib.EPI_SOFTMAX_BWD, aux=p, out=ds)
        spmm_device(tt.tiled, gy, p, weight_idx=tt.perm, x2=z, weights2=ds, weight_idx2=tt.perm,
                    out=out, accumulate=True)
        spmm_device(t, z, p, mode="f32", out=out)
        agnn_forward_device(t, z, p=p, out=out)
        agnn_backward_device(t, z, gy, p, ds=ds, out=out, y_fwd=out)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
