"""paper_2111_05188_b200 — B200-native (sm_100a) vectorised rollout hot path of
FinRL-Podracer (arXiv 2111.05188): libpod.so (CUDA kernels + C ABI in
include/pod.h) and a thin ctypes binding.  See DESIGN.md."""
from ._lib import PodError, load  # noqa: F401

__all__ = ["PodError", "load"]
