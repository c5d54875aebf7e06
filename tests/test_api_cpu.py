"""Host-side contract of the drop-in (no GPU): validation order and exception
types mirror the reference Index (core.py:107-173), SearchResult/Metric
semantics, and the FlatIndex constructor's own checks."""

import numpy as np
import pytest

from paper_2401_08281_b200 import core as C
from paper_2401_08281_b200.core import (METRIC_IP, METRIC_L2, Index, Metric, MetricKind, SearchResult, as_vectors,
                                        knn_recall)


class Recorder(Index):
    """Index whose hooks record calls (stands in for the GPU storage)."""

    def __init__(self, d, metric=METRIC_L2):
        super().__init__(d, metric)
        self.calls = []

    def _add(self, x, ids, sequential):
        self.calls.append(("add", x.shape, np.asarray(ids).tolist(), sequential))

    def _search(self, q, k):
        self.calls.append(("search", q.shape, k))
        return SearchResult(np.zeros((q.shape[0], k), np.int64), np.zeros((q.shape[0], k), np.float32), k)


def test_as_vectors_rules():
    assert as_vectors([1, 2, 3]).shape == (1, 3)
    assert as_vectors(np.zeros((2, 3), np.float64)).dtype == np.float32
    with pytest.raises(ValueError):
        as_vectors(np.zeros((2, 3, 4)))
    with pytest.raises(ValueError):
        as_vectors(np.zeros((2, 0)))
    with pytest.raises(ValueError):
        as_vectors(np.zeros((2, 3)), d=4)


def test_as_vectors_torch():
    torch = pytest.importorskip("torch")
    t = as_vectors(torch.zeros(5, dtype=torch.float64))
    assert t.shape == (1, 5) and t.dtype == torch.float32
    assert as_vectors(torch.zeros(2, 3, dtype=torch.bfloat16)).dtype == torch.bfloat16
    with pytest.raises(ValueError):
        as_vectors(torch.zeros(2, 3), d=2)


def test_add_assigns_sequential_ids():
    idx = Recorder(3)
    idx.add(np.zeros((2, 3)))
    idx.add(np.zeros((3, 3)))
    assert idx.ntotal == 5
    assert idx.calls[1][2] == [2, 3, 4]


def test_add_with_ids_validation():
    idx = Recorder(2)
    with pytest.raises(ValueError):
        idx.add_with_ids(np.zeros((2, 2)), [1])
    with pytest.raises(ValueError):
        idx.add_with_ids(np.zeros((2, 2)), [1, -1])
    with pytest.raises(ValueError):
        idx.add_with_ids(np.zeros((2, 3)), [1, 2])
    idx.is_trained = False
    with pytest.raises(RuntimeError):
        idx.add_with_ids(np.zeros((2, 2)), [1, 2])


def test_search_validation_order():
    idx = Recorder(4)
    idx.is_trained = False
    with pytest.raises(RuntimeError):  # untrained first, even with k=0
        idx.search(np.zeros((1, 4)), 0)
    idx.is_trained = True
    with pytest.raises(ValueError):  # then k
        idx.search(np.zeros((1, 5)), 0)
    with pytest.raises(ValueError):  # then dimension
        idx.search(np.zeros((1, 5)), 1)
    res = idx.search(np.zeros(4), 3)
    assert res.ids.shape == (1, 3) and res.nq == 1


def test_search_result_unpacks_faiss_style():
    r = SearchResult(np.array([[1, 2]]), np.array([[0.5, 0.7]], np.float32), 2)
    D, I = r
    assert I.tolist() == [[1, 2]] and D.dtype == np.float32


def test_metric_semantics():
    assert METRIC_IP.descending and not METRIC_L2.descending
    assert METRIC_IP.code == 0 and METRIC_L2.code == 1
    with pytest.raises(ValueError):
        Metric(MetricKind.Lp, 0.0)
    assert C.metric_value("L2") == "l2"


def test_reference_metric_objects_are_accepted():
    class FakeKind:
        value = "ip"

    class FakeMetric:
        kind = FakeKind()

    assert C.metric_value(FakeMetric()) == "ip"


def test_knn_recall_mirrors_reference():
    def res(rows):
        a = np.array(rows, np.int64)
        return SearchResult(a, np.zeros(a.shape, np.float32), a.shape[1])

    assert knn_recall(res([[7, 1, 3]]), res([[3, 7, 9]]), 1, 3) == 1.0
    assert knn_recall(res([[7, 5]]), res([[3, 7]]), 2, 2) == 0.5
    assert knn_recall(res([[1, -1]]), res([[1, -1]]), 2, 2) == 0.5
    with pytest.raises(ValueError):
        knn_recall(res([[1]]), res([[1, 2]]), 2, 1)


def test_flat_index_rejects_unsupported_metric_before_touching_gpu():
    from paper_2401_08281_b200.flat import FlatIndex
    with pytest.raises(NotImplementedError):
        FlatIndex(4, Metric(MetricKind.L1))
    with pytest.raises(ValueError):
        FlatIndex(0)
    with pytest.raises(ValueError):
        FlatIndex(4, storage="int8")


def test_flat_index_marks_itself_flat_for_ivf_coarse_cost():
    # annkit's IVF search charges nlist coarse distances per query only for a
    # flat coarse quantizer (ivf.py:401); the GPU index answers the duck-typed
    # check of the INTEGRATION.md patch (class attribute: no GPU needed)
    from paper_2401_08281_b200.flat import FlatIndex, IndexFlatIP, IndexFlatL2
    assert FlatIndex.is_flat and IndexFlatL2.is_flat and IndexFlatIP.is_flat
