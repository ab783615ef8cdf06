"""B200-native left-balanced k-d tree builder (arXiv 2211.00120).

Drop-in for the build entry points of the reference package ``lbkd``
(/root/reference/pkg/src/lbkd/__init__.py:9-11): ``build_round_robin``,
``build_widest``, ``KdTree``, ``BuildRecorder``.  Device-resident variants
``build_round_robin_cuda`` / ``build_widest_cuda`` work on torch CUDA
tensors without host copies.  All building runs in hand-written sm_100a
CUDA behind the C-ABI library in ``_lib/`` (include/lbkd_b200.h).
"""

from .builder import BuildRecorder, KdTree, build_round_robin, build_round_robin_cuda
from .widest import build_widest, build_widest_cuda, build_widest_host
from .queries import Neighbor, knn, knn_cuda, radius_cuda, radius_query

__all__ = [
    "BuildRecorder",
    "KdTree",
    "build_round_robin",
    "build_round_robin_cuda",
    "build_widest",
    "build_widest_cuda",
    "build_widest_host",
    "Neighbor",
    "knn",
    "knn_cuda",
    "radius_cuda",
    "radius_query",
]

__version__ = "0.1.0"
