"""B200-native cubic-spline build + eval (arXiv 2001.09253 hot path).

The compute path is the C-ABI library ``csrc/libfastspline.so`` (hand-written
sm_100a CUDA).  ``api`` marshals torch tensors into it; there is no CPU fallback:
calling any op without the built library raises.
"""
from .workloads import CONFIGS, generate  # noqa: F401

__all__ = ["CONFIGS", "generate", "api", "dist"]


def __getattr__(name):
    if name in ("api", "dist"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
