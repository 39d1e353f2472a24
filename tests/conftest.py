import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libdgx_cuda.so")


def _ensure_oracle():
    """Build oracle/_ref from /root/reference when it is missing (this container);
    on the GPU box the prebuilt files travel with the snapshot."""
    lib = os.path.join(ROOT, "oracle", "_ref", "libdgref_sm.so")
    if not os.path.exists(lib) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True)
    return os.path.exists(lib)


@pytest.fixture(scope="session")
def oracle():
    if not _ensure_oracle():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    from oracle import ref
    return ref


@pytest.fixture(scope="session")
def ctx():
    from paper_2306_08132_b200 import api
    return api.Context(0)
