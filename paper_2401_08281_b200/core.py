"""Index contract and result types of the drop-in, mirroring the reference.

Same names, argument meanings, validation order and exception types as the
reference's ``annkit.core`` for the flat k-NN path:

* ``MetricKind`` / ``Metric`` / ``METRIC_L2`` / ``METRIC_IP``  <- core.py:14-53
* ``as_vectors``                                               <- core.py:56-67
* ``SearchResult``                                             <- core.py:70-83
* ``Index`` (train/add/add_with_ids/search/...)                <- core.py:107-173
* ``knn_recall``                                               <- core.py:314-327

Inputs may be numpy arrays, sequences, or torch tensors (CPU or CUDA).
CUDA tensors stay on the device end to end.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Any

import numpy as np

try:  # torch is plumbing (device memory, streams, distributed), not required for numpy callers
    import torch
except ImportError:  # pragma: no cover
    torch = None


class MetricKind(Enum):
    """Distance kinds of the reference (core.py:14-30).  The GPU flat index
    implements L2 (squared Euclidean) and InnerProduct; the others are the
    reference's direct-path metrics and are rejected by ``FlatIndex``."""

    InnerProduct = "ip"
    L2 = "l2"
    L1 = "l1"
    Linf = "linf"
    Lp = "lp"
    Canberra = "canberra"
    BrayCurtis = "braycurtis"
    JensenShannon = "jensenshannon"
    Jaccard = "jaccard"
    NaNEuclidean = "naneuclidean"


@dataclass(frozen=True)
class Metric:
    kind: MetricKind
    arg: float = 0.0

    def __post_init__(self) -> None:
        if self.kind is MetricKind.Lp and not self.arg > 0:
            raise ValueError("Lp metric requires arg > 0")

    @property
    def descending(self) -> bool:
        """Larger is better only for the inner product (core.py:42-45)."""
        return self.kind is MetricKind.InnerProduct

    @property
    def code(self) -> int:
        # _pykernels.py:14-15: IP=0, L2=1 (same numbers as FK_METRIC_*)
        order = ["ip", "l2", "l1", "linf", "lp", "canberra", "braycurtis", "jensenshannon", "jaccard",
                 "naneuclidean"]
        return order.index(self.kind.value)


METRIC_IP = Metric(MetricKind.InnerProduct)
METRIC_L2 = Metric(MetricKind.L2)


def metric_value(metric: Any) -> str:
    """Accept our Metric, the reference's annkit Metric (duck-typed), or 'l2'/'ip'."""
    if isinstance(metric, str):
        return metric.lower()
    kind = getattr(metric, "kind", None)
    val = getattr(kind, "value", None)
    if val is None:
        raise TypeError(f"not a metric: {metric!r}")
    return val


def is_torch(x: Any) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def as_vectors(x: Any, d: int | None = None):
    """Canonical vector-set layout: C-contiguous (n, d) (core.py:56-67).

    numpy / sequences -> float32 ndarray.  torch tensors keep their device;
    float16/bfloat16 tensors keep their dtype (the GPU converts), everything
    else becomes float32.  1-D -> (1, d).  ValueError on ndim != 2, d < 1 or a
    dimension mismatch, in the reference's order.
    """
    if is_torch(x):
        t = x
        if t.dtype not in (torch.float32, torch.float16, torch.bfloat16):
            t = t.to(torch.float32)
        if t.dim() == 1:
            t = t.unsqueeze(0)
        if t.dim() != 2:
            raise ValueError(f"expected a 2-d vector set, got shape {tuple(t.shape)}")
        if t.shape[1] < 1:
            raise ValueError("vector dimension must be >= 1")
        if d is not None and t.shape[1] != d:
            raise ValueError(f"dimension mismatch: got {t.shape[1]}, index has {d}")
        return t.contiguous()
    arr = np.asarray(x)
    if arr.dtype not in (np.float32, np.float16):
        arr = arr.astype(np.float32)
    arr = np.ascontiguousarray(arr)
    if arr.ndim == 1:
        arr = arr[None, :]
    if arr.ndim != 2:
        raise ValueError(f"expected a 2-d vector set, got shape {arr.shape}")
    if arr.shape[1] < 1:
        raise ValueError("vector dimension must be >= 1")
    if d is not None and arr.shape[1] != d:
        raise ValueError(f"dimension mismatch: got {arr.shape[1]}, index has {d}")
    return arr


@dataclass
class SearchResult:
    """Per-query top-k, best first; missing slots are id -1 and the worst value
    (core.py:70-83).  Iterating yields ``(distances, ids)`` so Faiss-style
    ``D, I = index.search(q, k)`` also works."""

    ids: Any  # (nq, k) int64 -- numpy, or a CUDA tensor for CUDA queries
    distances: Any  # (nq, k) float32
    k: int

    @property
    def nq(self) -> int:
        return self.ids.shape[0]

    def __iter__(self):
        yield self.distances
        yield self.ids


@dataclass
class RangeResult:
    """Variable-length per-query results in CSR form (core.py:86-104): query i
    owns entries lims[i]:lims[i+1], each list sorted best first."""

    lims: Any  # (nq + 1,) int64
    ids: Any  # int64
    distances: Any  # float32
    radius: float

    @property
    def nq(self) -> int:
        return len(self.lims) - 1

    def row(self, i: int):
        lo, hi = int(self.lims[i]), int(self.lims[i + 1])
        return self.ids[lo:hi], self.distances[lo:hi]


class Index:
    """Base contract (core.py:107-173): subclasses override the private hooks.

    Reads may run concurrently on a frozen index; mutations need exclusive
    access (core.py:107-112).
    """

    def __init__(self, d: int, metric: Metric = METRIC_L2):
        if d < 1:
            raise ValueError("d must be >= 1")
        self.d = int(d)
        self.metric = metric
        self.ntotal = 0
        self.is_trained = True

    def train(self, x) -> None:
        x = as_vectors(x, self.d)
        self._train(x)
        self.is_trained = True

    def add(self, x) -> None:
        x = as_vectors(x, self.d)
        n = x.shape[0]
        if is_torch(x):
            ids = torch.arange(self.ntotal, self.ntotal + n, dtype=torch.int64, device=x.device)
        else:
            ids = np.arange(self.ntotal, self.ntotal + n, dtype=np.int64)
        self._add_checked(x, ids, sequential=True)

    def add_with_ids(self, x, ids) -> None:
        if not self.is_trained:
            raise RuntimeError("index must be trained before adding vectors")
        x = as_vectors(x, self.d)
        if is_torch(ids):
            ids = ids.to(torch.int64)
            bad_shape = tuple(ids.shape) != (x.shape[0],)
        else:
            ids = np.asarray(ids, dtype=np.int64)
            bad_shape = ids.shape != (x.shape[0],)
        if bad_shape:
            raise ValueError("ids must be a 1-d array matching the vector count")
        if bool((ids < 0).any()):
            raise ValueError("ids must be >= 0 (sign bit is reserved)")
        self._add_checked(x, ids, sequential=False)

    def _add_checked(self, x, ids, sequential: bool) -> None:
        if not self.is_trained:
            raise RuntimeError("index must be trained before adding vectors")
        self._add(x, ids, sequential)
        self.ntotal += x.shape[0]

    def search(self, q, k: int) -> SearchResult:
        if not self.is_trained:
            raise RuntimeError("index must be trained before searching")
        if k < 1:
            raise ValueError("k must be >= 1")
        return self._search(as_vectors(q, self.d), int(k))

    def range_search(self, q, radius: float):
        if not self.is_trained:
            raise RuntimeError("index must be trained before searching")
        return self._range_search(as_vectors(q, self.d), float(radius))

    def remove_ids(self, ids) -> int:
        raise NotImplementedError(f"{type(self).__name__} does not support removal")

    def reconstruct_batch(self, ids):
        raise NotImplementedError(f"{type(self).__name__} does not support reconstruction")

    def _train(self, x) -> None:
        pass

    def _add(self, x, ids, sequential: bool) -> None:
        raise NotImplementedError

    def _search(self, q, k: int) -> SearchResult:
        raise NotImplementedError

    def _range_search(self, q, radius: float):
        raise NotImplementedError(f"{type(self).__name__} does not implement range search")


def knn_recall(result: SearchResult, ground_truth: SearchResult, n: int, k: int) -> float:
    """n-recall@k: mean fraction of the n true neighbours found in the top k
    (core.py:314-327); -1 padding is ignored."""
    if n > k:
        raise ValueError("n-recall@k requires n <= k")
    gt_ids = _host(ground_truth.ids)
    res_ids = _host(result.ids)
    if gt_ids.shape[1] < n:
        raise ValueError("ground truth has fewer than n entries per query")
    got = res_ids[:, :k]
    want = gt_ids[:, :n]
    hits = 0
    for row_got, row_want in zip(got, want):
        keep = row_want[row_want >= 0]
        hits += int(np.isin(keep, row_got[row_got >= 0]).sum())
    return hits / (res_ids.shape[0] * n)


def _host(a):
    if is_torch(a):
        return a.detach().cpu().numpy()
    return np.asarray(a)
