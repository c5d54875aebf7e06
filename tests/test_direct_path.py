"""GPU direct path for batches below config.blas_threshold (flat.py:58-62 ->
flat_search flat.py:76-91): exact per-pair distances, (value, position)
order, compared with the oracle's direct restatement and with the
reference's own Index.search goldens (tests/test_gpu_parity.py)."""

import numpy as np
import pytest

from oracle import flat_oracle as O
from parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2401_08281_b200 as P  # noqa: E402
from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex  # noqa: E402


@pytest.mark.parametrize("storage", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("nq,k", [(1, 1), (7, 10), (19, 100), (19, 2048)])
def test_direct_vs_oracle(storage, metric, nq, k):
    rng = np.random.default_rng(nq * 7 + k)
    xb = rng.standard_normal((9000, 96), dtype=np.float32)
    q = rng.standard_normal((nq, 96), dtype=np.float32)
    idx = FlatIndex(96, METRIC_L2 if metric == "l2" else METRIC_IP, storage=storage)
    idx.add(xb)
    res = idx.search(q, k)
    assert idx.last_plan()["kmode"] == -1  # direct path taken
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    want_ids, want_dist = O.flat_search_direct(xr, qr, k, metric)
    s = assert_parity(res.ids, res.distances, want_ids, want_dist, rel_dist=1e-6, abs_dist=1e-6)
    assert s["strict_recall"] >= 0.999


def test_direct_integer_ties_identical():
    rng = np.random.default_rng(3)
    xb = rng.integers(0, 3, size=(5000, 20)).astype(np.float32)
    q = rng.integers(0, 3, size=(12, 20)).astype(np.float32)
    for metric in ("l2", "ip"):
        idx = FlatIndex(20, METRIC_L2 if metric == "l2" else METRIC_IP)
        idx.add(xb)
        res = idx.search(q, 300)
        want_ids, want_dist = O.flat_search_direct(xb, q, 300, metric)
        assert np.array_equal(res.ids, want_ids) and np.array_equal(res.distances, want_dist)


def test_self_distance_exact_zero_all_storages():
    rng = np.random.default_rng(4)
    xb = rng.standard_normal((2000, 50), dtype=np.float32)
    for storage in ("fp32", "fp16", "bf16"):
        idx = FlatIndex(50, METRIC_L2, storage=storage)
        idx.add(xb)
        rows = np.array([0, 17, 999, 1999])
        res = idx.search(O.round_to(xb[rows], storage), 2)
        assert np.array_equal(res.ids[:, 0], rows)
        assert np.all(res.distances[:, 0] == 0.0) and not np.any(np.signbit(res.distances[:, 0]))


def test_threshold_knob_switches_paths():
    rng = np.random.default_rng(5)
    xb = rng.standard_normal((3000, 32), dtype=np.float32)
    q = rng.standard_normal((30, 32), dtype=np.float32)
    idx = FlatIndex(32, METRIC_L2)
    idx.add(xb)
    idx.search(q, 5)
    assert idx.last_plan()["kmode"] != -1  # 30 >= 20: GEMM path
    old = P.config.blas_threshold
    P.config.blas_threshold = 64
    try:
        res = idx.search(q, 5)
        assert idx.last_plan()["kmode"] == -1
    finally:
        P.config.blas_threshold = old
    want_ids, want_dist = O.flat_search_direct(xb, q, 5, "l2")
    assert_parity(res.ids, res.distances, want_ids, want_dist)


def test_direct_device_tensors_and_ids():
    rng = np.random.default_rng(6)
    xb = rng.standard_normal((4000, 24), dtype=np.float32)
    ids = np.arange(4000) * 3 + 5
    idx = FlatIndex(24, METRIC_IP)
    idx.add_with_ids(torch.from_numpy(xb).cuda(), ids)
    q = rng.standard_normal((4, 24), dtype=np.float32)
    res = idx.search(torch.from_numpy(q).cuda(), 9)
    assert res.ids.is_cuda
    want_ids, want_dist = O.flat_search_direct(xb, q, 9, "ip", ids=ids)
    assert_parity(res.ids.cpu().numpy(), res.distances.cpu().numpy(), want_ids, want_dist)


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("nq,k,nb", [(1, 10, 100_000), (5, 1, 70_000), (19, 100, 50_001), (3, 2048, 40_000)])
def test_direct_two_level_selection(metric, nq, k, nb):
    """More rows than 8192-row slices x k: each slice's exact top-k first,
    then the per-query selection over the slices' lists -- the oracle's
    direct answers, ties by position."""
    rng = np.random.default_rng(nb + k)
    xb = rng.integers(-3, 4, size=(nb, 24)).astype(np.float32)  # many exact ties
    q = rng.integers(-3, 4, size=(nq, 24)).astype(np.float32)
    idx = FlatIndex(24, METRIC_L2 if metric == "l2" else METRIC_IP)
    idx.add(xb)
    res = idx.search(q, k)
    assert idx.last_plan()["kmode"] == -1
    want_ids, want_dist = O.flat_search_direct(xb, q, k, metric)
    assert np.array_equal(res.ids, want_ids) and np.array_equal(res.distances, want_dist)


@pytest.mark.parametrize("storage,metric,nq,d", [("fp32", "l2", 19, 128), ("fp16", "ip", 9, 96), ("bf16", "l2", 5, 200),
                                                  ("fp32", "ip", 2, 33)])
def test_direct_batched_reduction_bit_identical(storage, metric, nq, d):
    """The 8-query transposing reduction adds the same pairs in the same
    order as the one-query-at-a-time butterfly: bit-identical distances."""
    import os
    rng = np.random.default_rng(nq * d)
    xb = rng.standard_normal((20000, d), dtype=np.float32)
    q = rng.standard_normal((nq, d), dtype=np.float32)
    idx = FlatIndex(d, METRIC_L2 if metric == "l2" else METRIC_IP, storage=storage)
    idx.add(xb)
    a = idx.search(q, 25)
    os.environ["FK_DIRECT_WARP1"] = "1"
    try:
        b = idx.search(q, 25)
    finally:
        del os.environ["FK_DIRECT_WARP1"]
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.distances, b.distances)
