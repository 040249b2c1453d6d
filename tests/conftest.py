import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle comparison")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref/libmscref.so)."""
    import refpy
    if not os.path.exists(refpy.LIB_PATH) and not os.path.isdir(refpy.REF_SRC):
        pytest.skip("reference library not built and /root/reference absent")
    refpy.lib()
    return refpy


@pytest.fixture(scope="session")
def rs():
    """The plain-C oracle restatement (oracle/_build/liborestate.so)."""
    import restatepy
    restatepy.lib()
    return restatepy


@pytest.fixture(scope="session")
def msc():
    import paper_1104_3349_b200 as m
    from paper_1104_3349_b200 import build
    if not os.path.exists(os.path.join(ROOT, "paper_1104_3349_b200", "libmscg.so")):
        build.build()
    return m


@pytest.fixture(scope="session")
def ctx(msc):
    return msc.Context(0)
