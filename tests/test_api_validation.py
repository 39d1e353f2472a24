"""Host-side argument validation of the Python API (no GPU needed): every
caller-supplied array is checked for shape / dtype / order before its pointer
crosses the C ABI, which trusts the sizes."""
import numpy as np
import pytest

from paper_2306_08132_b200 import api


def test_check_arr_numpy():
    api._check_arr(np.zeros((4, 3)), (4, 3), "f64", "q")
    api._check_arr(None, (4, 3), "f64", "q")
    with pytest.raises(ValueError, match="shape"):
        api._check_arr(np.zeros((4, 2)), (4, 3), "f64", "q")
    with pytest.raises(ValueError, match="dtype"):
        api._check_arr(np.zeros((4, 3), np.float32), (4, 3), "f64", "q")
    with pytest.raises(ValueError, match="dtype"):
        api._check_arr(np.zeros(4, np.int64), (4,), "i32", "status")
    with pytest.raises(ValueError, match="contiguous"):
        api._check_arr(np.zeros((3, 4)).T, (4, 3), "f64", "q")


def test_check_arr_torch():
    torch = pytest.importorskip("torch")
    api._check_arr(torch.zeros(4, 3, dtype=torch.float64), (4, 3), "f64", "q")
    with pytest.raises(ValueError, match="shape"):
        api._check_arr(torch.zeros(5, 3, dtype=torch.float64), (4, 3), "f64", "q")
    with pytest.raises(ValueError, match="dtype"):
        api._check_arr(torch.zeros(4, dtype=torch.int64), (4,), "i32", "status")


class _FakeObj:
    def __init__(self):
        import ctypes
        self.h = ctypes.c_void_p(1)


class _FakeHand:
    J, N = 9, 10
    h = None


def test_optimize_multi_validates_before_the_abi():
    """Wrong counts length, wrong adam shape or a wrong status dtype raise
    ValueError before anything reaches the library."""
    hand, objs = _FakeHand(), [_FakeObj(), _FakeObj()]
    B, D = 6, 15
    q = np.zeros((B, 16))
    m, v = np.zeros((B, D)), np.zeros((B, D))
    args = (api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(), api.OptConfig(10))
    with pytest.raises(ValueError, match="one entry per object"):
        api.optimize_multi(None, objs, hand, q, [6], *args, adam_m=m, adam_v=v, inplace=True)
    with pytest.raises(ValueError, match="adam_m"):
        api.optimize_multi(None, objs, hand, q, [3, 3], *args, adam_m=np.zeros((B, D - 1)), adam_v=v, inplace=True)
    with pytest.raises(ValueError, match="status"):
        api.optimize_multi(None, objs, hand, q, [3, 3], *args, adam_m=m, adam_v=v, inplace=True,
                           status=np.zeros(B, np.int64))
    with pytest.raises(ValueError, match="traj"):
        api.optimize_multi(None, objs, hand, q, [3, 3], *args, adam_m=m, adam_v=v, inplace=True, record=True,
                           traj=np.zeros((B, 2, 3 + D)), k_begin=0, k_end=1)
    with pytest.raises(ValueError, match="sum"):
        api.optimize_multi(None, objs, hand, q, [3, 2], *args, adam_m=m, adam_v=v, inplace=True)
