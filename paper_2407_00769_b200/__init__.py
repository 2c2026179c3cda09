"""B200-native stem-path contraction of sliced RQC tensor networks (arXiv 2407.00769).

The product is libtn.so (include/tn.h, sources in csrc/); ``tn`` is its ctypes binding."""
from . import tn  # noqa: F401
