"""B200-native cubic-spline build + eval (arXiv 2001.09253 hot path).

The compute path is the C-ABI library ``csrc/libfastspline.so`` (hand-written
sm_100a CUDA).  ``api`` marshals torch tensors into it; there is no CPU fallback:
calling any op without the built library raises.
"""
from .workloads import CONFIGS, generate  # noqa: F401

__all__ = ["CONFIGS", "generate", "api"]


def __getattr__(name):
    if name == "api":
        from . import api
        return api
    raise AttributeError(name)
