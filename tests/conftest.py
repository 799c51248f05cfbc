import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, GOLDEN_DIR)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _gpu_available() -> bool:
    from paper_2305_07238_b200 import Context, NoDeviceError, CudaError
    try:
        Context(0).close()
        return True
    except (NoDeviceError, CudaError):
        return False


@pytest.fixture(scope="session")
def built():
    """libmcg.so and the oracle builds (incremental; no-ops when current)."""
    from paper_2305_07238_b200 import build as B
    import _oracle
    B.build()
    _oracle.build_oracle(ref=os.path.isdir("/root/reference"))
    return True


@pytest.fixture(scope="session")
def oracle(built):
    import _oracle
    return _oracle.Oracle()


@pytest.fixture(scope="session")
def ref(built):
    import _oracle
    if not _oracle.Ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return _oracle.Ref()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        G = json.load(f)
    G["npz"] = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
    return G


@pytest.fixture(scope="session")
def scene_dir(tmp_path_factory):
    return str(tmp_path_factory.mktemp("scenes"))


@pytest.fixture(scope="session")
def ctx(built):
    if not _gpu_available():
        pytest.skip("no CUDA device")
    from paper_2305_07238_b200 import Context
    return Context(0)
