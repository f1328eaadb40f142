"""Shared fixtures: golden fixtures from the reference, oracle import, markers.

`-m "not gpu"` tests run here (no GPU); `-m gpu` tests run on a B200 and call
the CUDA path through the C ABI (libtcg_b200.so).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

try:
    from hypothesis import settings

    settings.register_profile("no_deadline", deadline=None)
    settings.load_profile("no_deadline")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtcg_b200.so")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle import tcg_oracle

    return tcg_oracle


class SmallCases:
    """tests/golden/small_cases.{npz,json}: reference outputs per case; the
    inputs are regenerated from the recorded seeds."""

    def __init__(self):
        self.z = np.load(GOLDEN / "small_cases.npz")
        self.meta = json.loads((GOLDEN / "small_cases.json").read_text())

    def __iter__(self):
        return iter(self.meta)

    def arr(self, case, name):
        return self.z[case["key"] + name]

    def has(self, case, name):
        return (case["key"] + name) in self.z.files

    @staticmethod
    def emb(n, d, seed):
        return np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)

    def inputs(self, case):
        n, m = case["n"], case["m"]
        x = self.emb(n, case["d_spmm"], case["seed_x"])
        xs = self.emb(n, case["d_sddmm"], case["seed_xs"])
        f = np.random.default_rng(case["seed_f"]).standard_normal(m).astype(np.float32)
        return x, xs, f

    def gcn_params(self, case):
        w = self.emb(case["d_spmm"], 3, case["seed_w"])
        b = self.emb(1, 3, case["seed_b"])[0]
        return w, b


@pytest.fixture(scope="session")
def small_cases():
    return SmallCases()


@pytest.fixture(scope="session")
def cora_golden():
    return dict(np.load(GOLDEN / "cora.npz"))


@pytest.fixture(scope="session")
def digests():
    return json.loads((GOLDEN / "digests.json").read_text())


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a - b))


# North-star tolerance for TF32 outputs (10-bit-mantissa operands, fp32
# accumulate): relative L2 <= 5e-3 (BASELINE.json north_star).
TF32_REL_L2 = 5e-3
