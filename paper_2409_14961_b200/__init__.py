"""B200-native UELLM batch scheduler (arXiv 2409.14961, Sec. 4.2): sort by (SLO, predicted
length), exact SEG-DP segmentation under a KV cap, per-batch stats -- sm_100a kernels behind
the C ABI of include/uellm.h.  Importing the package loads libuellm.so and fails if it is
missing (no CPU fallback)."""
from . import uellm  # noqa: F401  (loads libuellm.so)

__all__ = ["uellm"]
