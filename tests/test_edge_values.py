"""GPU ordering of non-finite and signed-zero values vs the oracle.

The reference ranks by the 64-bit key ``monotone(value) << 32 | column``
(core.py:193-197, 219): +inf above every finite value, a NaN (the positive
quiet NaN that a NaN input such as np.nan carries through the sgemm) above
+inf, equal keys by the smaller column.  IP ranks ``-value`` (core.py:217):
the negated NaN has the sign bit set, so a NaN inner product sorts FIRST.
The L2 clamp ``np.maximum(dmat, 0)`` (flat.py:112) returns +0.0 for every
non-positive dmat (dmat is never -0.0: ``(qn + xn) - 2ip`` of equal operands
rounds to +0), and keeps NaN.

Checked on every operand path: fp32 small (3xTF32, MODE 0), fp32 at >= 262k
rows (1-pass TF32 filter + exact rescoring, MODE 4 -- NaN / inf bounds
disable the certification band and route through the exact fallback),
fp16 and bf16 (folded norms).
"""

import numpy as np
import pytest

from oracle import flat_oracle as O
from parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex, config  # noqa: E402


@pytest.fixture(autouse=True, params=["blas", "direct"])
def path(request):
    """Run every case on both FlatIndex._search branches (flat.py:58-62):
    "blas" forces the fused GEMM + top-k kernel (blas_threshold 0) and is
    checked against flat_search_blas; "direct" keeps the reference threshold
    (these batches are < 20 queries) and is checked against the direct path."""
    saved = config.blas_threshold
    config.blas_threshold = 0 if request.param == "blas" else 20
    yield request.param
    config.blas_threshold = saved


def oracle_search(xb, q, k, metric):
    if config.blas_threshold == 0 or q.shape[0] >= config.blas_threshold:
        return O.flat_search_blas(xb, q, k, metric)
    return O.flat_search_direct(xb, q, k, metric)


def assert_same_order(got_ids, got_dist, want_ids, want_dist):
    """Non-finite reference values: the same id at the same slot with the same
    class (NaN / +inf / -inf); the finite entries go through the tie-aware
    comparator."""
    got_ids, want_ids = np.asarray(got_ids), np.asarray(want_ids)
    got_dist, want_dist = np.asarray(got_dist, np.float32), np.asarray(want_dist, np.float32)
    nonfin = ~np.isfinite(want_dist)
    assert np.array_equal(np.isnan(got_dist), np.isnan(want_dist))
    assert np.array_equal(np.isposinf(got_dist), np.isposinf(want_dist))
    assert np.array_equal(np.isneginf(got_dist), np.isneginf(want_dist))
    assert np.array_equal(got_ids[nonfin], want_ids[nonfin]), (got_ids[nonfin], want_ids[nonfin])
    fin_rows = np.all(np.isfinite(want_dist), axis=1)
    if fin_rows.any():
        assert_parity(got_ids[fin_rows], got_dist[fin_rows], want_ids[fin_rows], want_dist[fin_rows])
    # mixed rows: finite prefix, exact ids on the non-finite tail
    for r in np.nonzero(~fin_rows)[0]:
        f = np.isfinite(want_dist[r])
        if f.any():
            assert set(got_ids[r][f].tolist()) == set(want_ids[r][f].tolist()) or np.allclose(
                np.sort(got_dist[r][f]), np.sort(want_dist[r][f]), rtol=1e-4, atol=1e-4)


def edge_data(nb, d, rng, metric):
    xb = rng.standard_normal((nb, d), dtype=np.float32)
    nan_rows = np.array([3, 11, 12, nb - 1])
    big_rows = np.array([5, 7, nb - 2])
    xb[nan_rows, 2] = np.nan
    if metric == "l2":
        xb[big_rows] = 1e20  # |x|^2 overflows: +inf distance, finite inner products
    q = rng.standard_normal((6, d), dtype=np.float32)
    q[4, 1] = np.nan  # every distance of query 4 is NaN: positions 0.. in order
    return xb, q


@pytest.mark.parametrize("storage", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_nan_inf_order_small(storage, metric):
    rng = np.random.default_rng(31)
    nb, d = 40, 16
    xb, q = edge_data(nb, d, rng, metric)
    if storage == "fp16":
        xb[np.all(xb == 1e20, axis=1)] = 100.0  # fp16 inputs cannot overflow an fp32 norm at d=16
    idx = FlatIndex(d, METRIC_L2 if metric == "l2" else METRIC_IP, storage=storage)
    idx.add(xb)
    res = idx.search(q, nb)  # every row: the whole order is visible
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    with np.errstate(invalid="ignore", over="ignore"):
        want_ids, want_dist = oracle_search(xr, qr, nb, metric)
    assert_same_order(res.ids, res.distances, want_ids, want_dist)
    # NaN query: all NaN, ids by position
    assert np.all(np.isnan(res.distances[4]))
    assert np.array_equal(res.ids[4], np.arange(nb))


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_nan_rows_small_k(metric):
    """k smaller than the number of finite rows: NaN rows never displace a
    finite neighbour in L2, and lead every IP list (reference key of -NaN)."""
    rng = np.random.default_rng(32)
    nb, d = 3000, 24
    xb, q = edge_data(nb, d, rng, metric)
    idx = FlatIndex(d, METRIC_L2 if metric == "l2" else METRIC_IP)
    idx.add(xb)
    res = idx.search(q, 10)
    with np.errstate(invalid="ignore", over="ignore"):
        want_ids, want_dist = oracle_search(xb, q, 10, metric)
    assert_same_order(res.ids, res.distances, want_ids, want_dist)
    if metric == "ip":
        assert np.array_equal(res.ids[0, :4], [3, 11, 12, nb - 1])


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_nan_inf_large_fp32_one_pass_path(metric, path):
    """>= 262144 rows: the 1-pass TF32 + certified rescoring path with NaN /
    inf in the data (unbounded bands -> exact fallback) stays exact."""
    rng = np.random.default_rng(33)
    nb, d = 300_000, 32
    xb, q = edge_data(nb, d, rng, metric)
    idx = FlatIndex(d, METRIC_L2 if metric == "l2" else METRIC_IP)
    idx.add(xb)
    res = idx.search(q, 10)
    assert idx.last_plan()["kmode"] in ((4, 5) if path == "blas" else (-1,))
    with np.errstate(invalid="ignore", over="ignore"):
        want_ids, want_dist = oracle_search(xb, q, 10, metric)
    assert_same_order(res.ids, res.distances, want_ids, want_dist)


def test_clamp_gives_positive_zero():
    """Self-distances of integer data are exactly 0: the clamp (flat.py:112)
    yields +0.0 (never -0.0), on both fp32 paths."""
    rng = np.random.default_rng(34)
    for nb in (500, 300_000):
        xb = rng.integers(-8, 8, size=(nb, 20)).astype(np.float32)
        xb = np.unique(xb, axis=0)[:nb]
        rng.shuffle(xb)
        idx = FlatIndex(20, METRIC_L2)
        idx.add(xb)
        rows = np.arange(0, xb.shape[0], max(1, xb.shape[0] // 50))
        res = idx.search(xb[rows], 3)
        assert np.array_equal(res.ids[:, 0], rows)
        d0 = res.distances[:, 0]
        assert np.all(d0 == 0.0) and not np.any(np.signbit(d0))


def test_ip_signed_zero_order():
    """IP ranks -ip: +0.0 (key of -0.0) before -0.0 (key of +0.0), equal keys
    by position.  Rows orthogonal to the query give exact zeros."""
    d = 4
    xb = np.array([[0, 1, 0, 0], [0, 0, 1, 0], [1, 0, 0, 0], [-1, 0, 0, 0], [0, 0, 0, 1]], np.float32)
    q = np.array([[1, 0, 0, 0]], np.float32)
    idx = FlatIndex(d, METRIC_IP)
    idx.add(xb)
    res = idx.search(q, 5)
    want_ids, want_dist = oracle_search(xb, q, 5, "ip")
    assert np.array_equal(res.ids, want_ids)
    assert np.array_equal(res.distances, want_dist)
