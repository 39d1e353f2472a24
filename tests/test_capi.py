"""CPU: the C-ABI library loads and exports exactly what include/dgx.h declares;
without a GPU it fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dgx.h")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dgx_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    for n in ("dgx_ctx_create", "dgx_loss_gradient_batch", "dgx_evaluate_losses_batch", "dgx_optimize_batch",
              "dgx_apply_gradient_step_batch", "dgx_forward_batch", "dgx_hand_upload", "dgx_object_upload"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2306_08132_b200 import capi
    lib = capi.load()
    for n in declared():
        assert hasattr(lib, n), n
    assert set(capi.EXPORTS) == set(declared())
    assert lib.dgx_abi_version() == 2
    nm = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (dgx_\w+)", nm))
    assert exported == set(declared()), exported ^ set(declared())


def test_sm100a_code_present():
    from paper_2306_08132_b200 import capi
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2306_08132_b200 import api, capi
    with pytest.raises(capi.DgxError):
        api.Context(0)
    L = capi.load()
    h = C.c_void_p()
    assert L.dgx_ctx_create(0, C.byref(h)) == 101  # DGX_E_CUDA
    assert b"cuda" in L.dgx_last_error().lower() or len(L.dgx_last_error()) > 0
