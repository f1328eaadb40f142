"""Host-side layout helpers and layer configuration (no GPU needed)."""

from __future__ import annotations

import pytest
import torch

from paper_2112_02052_b200 import dense, layers


@pytest.mark.parametrize("d,ld", [(47, 48), (22, 24), (16, 16), (40, 40), (7, 7), (3, 3)])
def test_rows_empty_padding(d, ld):
    x = dense.rows_empty(5, d, "cpu")
    assert x.shape == (5, d) and x.stride() == (ld, 1)
    assert dense.rows_ok(x) is x
    y = torch.zeros(d, 5).t()  # column-major view: copied into unit-stride rows
    z = dense.rows_ok(y)
    assert z is not y and z.stride(1) == 1 and torch.equal(z, y)


@pytest.mark.parametrize("fin,fout,order,agg_first", [
    (16, 47, "auto", True), (128, 16, "auto", False), (16, 16, "auto", False),
    (16, 7, "auto", False), (128, 16, "aggregate_first", True), (16, 47, "transform_first", False),
])
def test_gcnconv_order(fin, fout, order, agg_first):
    conv = layers.GCNConv(fin, fout, order=order)
    assert conv.aggregate_first is agg_first


def test_gcnconv_order_rejects_unknown():
    with pytest.raises(ValueError):
        layers.GCNConv(4, 4, order="sideways")
