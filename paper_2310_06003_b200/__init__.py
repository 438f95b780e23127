"""paper_2310_06003_b200 — B200-native PaRO sync + update step.

The product is libparo.so (C ABI in include/paro.h): planner, step engine and
sm_100a kernels.  `paro` is its ctypes binding; `torch_glue` allocates the
caller-owned optimizer state with torch (PyTorch is plumbing only: device
memory, streams, process groups).
"""
from . import paro  # noqa: F401  (raises ImportError if libparo.so is missing)

__all__ = ["paro"]
