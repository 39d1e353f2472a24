"""GPU: the drop-in C++ API (include/dgx/diffgrasp.hpp) used with the reference's
own types, checked in-process against the reference (oracle/test_dropin.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_api(oracle):
    exe = os.path.join(ROOT, "oracle", "_ref", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_dropin not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "DROPIN OK" in r.stdout, r.stdout + r.stderr


def test_cpp_dropin_reference_mesh_object(oracle):
    """dgx::Object built from the reference's own dg::GraspObject (icosphere
    mesh) vs dg::loss_gradient / evaluate_losses / MeshSdf queries, the
    unmodified reference linked in-process (oracle/test_dropin_mesh.cpp)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "test_dropin_mesh")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_dropin_mesh not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "DROPIN MESH OK" in r.stdout, r.stdout + r.stderr
