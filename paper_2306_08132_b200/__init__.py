"""paper_2306_08132_b200 — B200-native batched gradient-based grasp search
(the Fast-Grasp'D hot path, arXiv 2306.08132) behind the reference
diffgrasp API. Compute lives in libdgx_cuda.so (hand-written sm_100a CUDA,
include/dgx.h); this package is the host-side mirror."""
from .model import HandDesc, ObjectDesc  # noqa: F401

__all__ = ["HandDesc", "ObjectDesc"]
