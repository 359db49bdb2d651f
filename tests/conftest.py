from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libdist_b200.so")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def golden_weights(g: dict):
    return [(g[f"W{i}"], g[f"b{i}"]) for i in range(int(g["n_layers"]))]


def cfg_from(arr, **over):
    """TraceConfig kwargs from the fixture's packed config array."""
    kw = dict(alpha=float(arr[0]), epsilon=float(arr[1]), max_steps=int(arr[2]),
              k_samples=int(arr[3]), coarse_start_scale=int(arr[4]),
              split_interval=int(arr[5]), normal_delta=float(arr[6]),
              use_dynamic_mask=bool(arr[7]))
    kw.update(over)
    return kw


@pytest.fixture(scope="session")
def golden():
    return load_golden
