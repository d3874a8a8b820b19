"""B200-native RAS-PML hot path (arXiv 2602.00735): libhelm (sm_100a CUDA, C ABI in include/helm.h) and its
thin Python binding."""
from .helm import Context, HelmError, load  # noqa: F401
