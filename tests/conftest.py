"""Shared fixtures.  `gpu`-marked tests need a B200 (run via gpurun); the rest
run on CPU and cover the oracle, the host logic and the C-ABI surface."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size (BASELINE config) case")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def renderer():
    import paper_2406_12080_b200 as hs
    r = hs.Renderer(0, exact=True, debug=True, stats=True)
    yield r
    r.close()


@pytest.fixture(scope="session")
def c2():
    """BASELINE config[1]: the 10M-leaf hierarchy, shared by the full-size tests."""
    from paper_2406_12080_b200 import scenes
    cfg = scenes.CONFIGS["c2"]
    return cfg, scenes.hierarchy(cfg)


@pytest.fixture(scope="session")
def c2_oracle(c2):
    """The oracle's copy of the C2 hierarchy (304 B/node AoS, ~6 GB of host memory)."""
    from oracle import oracle as orc
    return orc.OracleHierarchy(c2[1])


@pytest.fixture(scope="session")
def c2_device(renderer, c2):
    return renderer.upload(c2[1], validate=True)
