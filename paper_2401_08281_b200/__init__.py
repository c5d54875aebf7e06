"""B200-native exact flat k-NN search (IndexFlatL2 / IndexFlatIP).

Drop-in for the hot path of the reference ``annkit`` package (arXiv
2401.08281 reference): ``FlatIndex(d, metric)`` with ``add``,
``add_with_ids``, ``search -> SearchResult``, ``ntotal`` plus ``reset``.
The compute runs in hand-written sm_100a kernels (tcgen05 GEMM + fused
top-k) behind the C ABI declared in ``include/flatknn.h``.
"""

from . import config
from .core import (METRIC_IP, METRIC_L2, Index, Metric, MetricKind, RangeResult, SearchResult, as_vectors,
                   knn_recall)
from .flat import FlatIndex, IndexFlatIP, IndexFlatL2, refine_search
from .kmeans import assign_vectors, coarse_quantizer, kmeans_assign, probe_lists
from .sharded import ShardedFlatIndex

__version__ = "0.1.0"

__all__ = [
    "FlatIndex",
    "IndexFlatIP",
    "IndexFlatL2",
    "Index",
    "Metric",
    "MetricKind",
    "METRIC_IP",
    "METRIC_L2",
    "RangeResult",
    "SearchResult",
    "ShardedFlatIndex",
    "as_vectors",
    "config",
    "assign_vectors",
    "coarse_quantizer",
    "kmeans_assign",
    "knn_recall",
    "probe_lists",
    "refine_search",
]
