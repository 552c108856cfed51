import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    lib = ROOT / "paper_2303_01778_b200" / "libparrot_b200.so"
    if not lib.exists():
        from paper_2303_01778_b200.build import build
        build()


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden_trainer():
    return dict(np.load(GOLDEN / "trainer.npz", allow_pickle=False))


@pytest.fixture(scope="session")
def golden_engine():
    return dict(np.load(GOLDEN / "engine.npz", allow_pickle=False))


@pytest.fixture(scope="session")
def golden_configs():
    return dict(np.load(GOLDEN / "configs.npz", allow_pickle=False))


@pytest.fixture(scope="session")
def golden_host():
    return json.loads((GOLDEN / "host.json").read_text())


def rel_gap(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(float(np.abs(want).max()), 1e-30)
    return float(np.abs(got - want).max()) / scale
