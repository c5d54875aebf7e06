"""fp32 search through the scaled-fp16 filter pass (kernel MODE 5, the
default 1-pass algorithm for fp32 storage with k <= 16 over >= 256k rows).

The fp32 rows and queries get power-of-two-scaled fp16 copies (11 significant
bits, like a tf32 operand); one kind::f16 tensor-core pass ranks k' >= k
candidates per list, band members that full register queues drop go to a
per-query overflow list, the merge certifies each query against the fp16
error band and recomputes the survivors exactly in fp32 (flat.py:111-112),
and uncertified queries take the exact fallback.  The answers must equal the
reference's (north-star parity rules) and -- because the final values come
from the same exact rescoring -- be bit-identical to the tf32 filter (MODE 4).

``set_plan_rows`` makes small test databases take the 1-pass path."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))

from cases import CASES, make_inputs  # noqa: E402
from oracle import flat_oracle as O  # noqa: E402
from parity import assert_parity  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))
FP32_CASES = [n for n in CASES if make_inputs(n)[4] == "fp32"]


def _index(d, metric, plan_rows=1 << 20):
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    idx = FlatIndex(d, METRIC_IP if metric == "ip" else METRIC_L2, storage="fp32")
    idx.set_plan_rows(plan_rows)
    return idx


def _search(idx, q, k, filt=None, kp=None):
    old = {n: os.environ.get(n) for n in ("FK_FP32_FILTER", "FK_KP")}
    try:
        if filt:
            os.environ["FK_FP32_FILTER"] = filt
        if kp:
            os.environ["FK_KP"] = str(kp)
        res = idx.search(q, k)
    finally:
        for n, v in old.items():
            if v is None:
                os.environ.pop(n, None)
            else:
                os.environ[n] = v
    return res


@pytest.mark.parametrize("name", FP32_CASES)
def test_filter16_golden(name):
    xb, q, k, metric, storage, ids = make_inputs(name)
    idx = _index(xb.shape[1], metric)
    if xb.shape[0]:
        if ids is None:
            idx.add(xb)
        else:
            idx.add_with_ids(xb, ids)
    res = idx.search(q, k)
    if xb.shape[0] and k <= 16 and q.shape[0] >= 20:
        assert idx.last_plan()["kmode"] == 5
    assert_parity(res.ids, res.distances, GOLD[f"{name}/blas_ids"], GOLD[f"{name}/blas_dist"])


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("k", [1, 10, 16])
@pytest.mark.parametrize("kp", [None, 16, 8])
def test_filter16_vs_oracle_and_tf32(metric, k, kp):
    """Default k' = 32, and short queues (k' = 16 / 8) that overflow into the
    per-query lists: same answers as the oracle, bit-identical to MODE 4."""
    if kp is not None and kp < k:
        pytest.skip("k' >= k")
    rng = np.random.default_rng(199 + k)
    xb = rng.standard_normal((60000, 64), dtype=np.float32)
    q = rng.standard_normal((300, 64), dtype=np.float32)
    idx = _index(64, metric)
    idx.add(xb)
    r5 = _search(idx, q, k, kp=kp)
    assert idx.last_plan()["kmode"] == 5
    want_ids, want_dist = O.flat_search_blas(xb, q, k, metric)
    assert_parity(r5.ids, r5.distances, want_ids, want_dist)
    r4 = _search(idx, q, k, filt="tf32")
    assert idx.last_plan()["kmode"] == 4
    assert np.array_equal(r5.ids, r4.ids) and np.array_equal(r5.distances, r4.distances)


def test_filter16_integer_ties_exact_band():
    """Integer data is exact in scaled fp16: the band collapses to the
    accumulation slack and the massive exact ties keep the reference order."""
    rng = np.random.default_rng(7)
    xb = rng.integers(0, 256, size=(200_000, 128)).astype(np.float32)
    q = rng.integers(0, 256, size=(64, 128)).astype(np.float32)
    q[:8] = xb[rng.choice(xb.shape[0], 8, replace=False)]  # exact duplicates: distance 0
    idx = _index(128, "l2")
    idx.add(xb)
    res = idx.search(q, 10)
    want_ids, want_dist = O.flat_search_blas(xb, q, 10, "l2")
    assert np.array_equal(res.ids, want_ids) and np.array_equal(res.distances, want_dist)


@pytest.mark.parametrize("scale", [1e-30, 1e-8, 1.0, 3e4, 1e15, 1e18])
def test_filter16_extreme_magnitudes(scale):
    """The power-of-two scales keep 11 bits at any magnitude (and flag an
    unusable scale -> exact fallback); mixed-magnitude rows hit the fp16
    subnormal range, covered by the band's absolute term."""
    rng = np.random.default_rng(int(abs(np.log10(scale))) + 3)
    xb = rng.standard_normal((20000, 48)).astype(np.float32)
    xb[::7] *= 1e-6  # rows far below the base maximum
    xb[3::11, :5] = 0.0
    q = rng.standard_normal((100, 48)).astype(np.float32)
    q[::5] *= 1e-5
    xb = (xb * scale).astype(np.float32)
    q = (q * scale).astype(np.float32)
    for metric in ("l2", "ip"):
        idx = _index(48, metric)
        idx.add(xb)
        res = idx.search(q, 10)
        with np.errstate(over="ignore", under="ignore", invalid="ignore"):
            want_ids, want_dist = O.flat_search_blas(xb, q, 10, metric)
        if np.all(np.isfinite(want_dist)):
            assert_parity(res.ids, res.distances, want_ids, want_dist)
        r4 = _search(idx, q, 10, filt="tf32")
        assert np.array_equal(res.ids, r4.ids) and np.array_equal(res.distances, r4.distances)


def test_filter16_rescale_on_add_and_remove():
    """Adding rows with a larger magnitude changes the base scale (the fp16
    copy is rebuilt); remove_ids invalidates it; results stay exact."""
    rng = np.random.default_rng(11)
    xa = rng.standard_normal((30000, 32), dtype=np.float32)
    xb = (rng.standard_normal((30000, 32)) * 1e6).astype(np.float32)
    q = rng.standard_normal((50, 32), dtype=np.float32)
    idx = _index(32, "l2")
    idx.add(xa)
    r = idx.search(q, 5)
    assert_parity(r.ids, r.distances, *O.flat_search_blas(xa, q, 5, "l2"))
    idx.add(xb)  # new max |x|: every row is re-encoded with the new scale
    both = np.vstack([xa, xb])
    r = idx.search(q, 5)
    assert_parity(r.ids, r.distances, *O.flat_search_blas(both, q, 5, "l2"))
    idx.add(xa[:1000] * 0.5)  # same scale: only the new rows are converted
    both = np.vstack([both, xa[:1000] * 0.5])
    r = idx.search(q, 5)
    assert_parity(r.ids, r.distances, *O.flat_search_blas(both, q, 5, "l2"))
    removed = idx.remove_ids(np.arange(30000, 60000))
    assert removed == 30000
    left = np.vstack([xa, xa[:1000] * 0.5])
    r = idx.search(q, 5)
    want_ids, want_dist = O.flat_search_blas(left, q, 5, "l2")
    want_ids = np.where(want_ids >= 30000, want_ids + 30000, want_ids)  # ids of the last batch
    assert_parity(r.ids, r.distances, want_ids, want_dist)


def test_filter16_inf_rows_and_nan_query():
    rng = np.random.default_rng(12)
    xb = rng.standard_normal((40000, 24), dtype=np.float32)
    xb[5] = np.inf
    xb[9, 3] = np.nan
    q = rng.standard_normal((40, 24), dtype=np.float32)
    q[3, 2] = np.nan
    idx = _index(24, "l2")
    idx.add(xb)
    res = idx.search(q, 10)
    with np.errstate(invalid="ignore", over="ignore"):
        want_ids, want_dist = O.flat_search_blas(xb, q, 10, "l2")
    fin = np.all(np.isfinite(want_dist), axis=1)
    assert_parity(res.ids[fin], res.distances[fin], want_ids[fin], want_dist[fin])
    assert np.all(np.isnan(res.distances[3]))


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("k,nb", [(40, 80_000), (100, 80_000), (1024, 600_000)])
def test_filter16_large_k(metric, k, nb):
    """k > 16 through the 1-pass filter (FK_FP32_1PASS_MAXK): large-k
    candidate lists (KQ = 0), the sampled bound pass (600k rows, k = 1024)
    and the certified rescoring merge -- same answers as the oracle and
    bit-identical to the tf32 filter."""
    rng = np.random.default_rng(500 + k)
    xb = rng.standard_normal((nb, 32), dtype=np.float32)
    q = rng.standard_normal((64, 32), dtype=np.float32)
    idx = _index(32, metric)
    idx.add(xb)
    old = os.environ.get("FK_FP32_1PASS_MAXK")
    os.environ["FK_FP32_1PASS_MAXK"] = "2048"
    try:
        r5 = idx.search(q, k)
        assert idx.last_plan()["kmode"] == 5
        r4 = _search(idx, q, k, filt="tf32")
    finally:
        if old is None:
            os.environ.pop("FK_FP32_1PASS_MAXK")
        else:
            os.environ["FK_FP32_1PASS_MAXK"] = old
    want_ids, want_dist = O.flat_search_blas(xb, q, k, metric)
    assert_parity(r5.ids, r5.distances, want_ids, want_dist)
    assert np.array_equal(r5.ids, r4.ids) and np.array_equal(r5.distances, r4.distances)


@pytest.mark.parametrize("filt", [None, "tf32"])
def test_filter16_coherent_rounding_worst_case(filt):
    """Adversarial rounding: every coordinate of the query and of row A sits
    just below an fp16 / tf32 rounding midpoint, so the filter underestimates
    <q, A> coherently by ~2^-10 |q||A| per pair, while 300 decoy rows are
    exactly representable with a filter value ABOVE A's but a true inner
    product below it.  A must survive the band (through the overflow lists:
    the decoys fill every queue) and win after the exact rescoring."""
    d = 64
    a = 2.0 ** -11 - 2.0 ** -20           # q_i = x_A,i = 1 + a: rounds down to 1 in fp16 and tf32
    q = np.full((24, d), 1 + a, dtype=np.float32)
    x_a = np.full((1, d), 1 + a, dtype=np.float32)
    rng = np.random.default_rng(5)
    decoys = np.ones((300, d), dtype=np.float32)
    for r in range(300):                  # 31 coordinates at 1 + 2^-10: mean 1 + (2^-11 - 2^-16) < 1 + a
        decoys[r, rng.choice(d, 31, replace=False)] = 1 + 2.0 ** -10
    filler = rng.standard_normal((300_000, d)).astype(np.float32) * 0.01
    xb = np.vstack([filler[:150_000], decoys, x_a, filler[150_000:]])
    a_pos = 150_000 + 300
    idx = _index(d, "ip")
    idx.add(xb)
    res = _search(idx, q, 1, filt=filt)
    assert np.all(res.ids[:, 0] == a_pos), res.ids[:, 0]
    want_ids, want_dist = O.flat_search_blas(xb, q, 1, "ip")
    assert np.all(want_ids[:, 0] == a_pos)
    assert_parity(res.ids, res.distances, want_ids, want_dist)


@pytest.mark.parametrize("nq", [200, 600])
def test_filter16_fallback_values_equal_certified_values(nq):
    """Queries forced into the exact fallback (no overflow lists, 8-deep
    queues) return bit-identical values and ids to the certified rescoring
    merge: both sum the fp32 products in the same order (warp_exact_dot /
    thread_exact_dot).  600 queries: past the first 148 failed queries (rows
    split over the grid) the per-CTA whole-base scan answers the rest."""
    rng = np.random.default_rng(21)
    xb = rng.standard_normal((70000, 96), dtype=np.float32)
    q = rng.standard_normal((nq, 96), dtype=np.float32)
    idx = _index(96, "l2")
    idx.add(xb)
    base = idx.search(q, 10)
    old = {n: os.environ.get(n) for n in ("FK_OVF", "FK_KP")}
    os.environ["FK_OVF"] = "0"
    os.environ["FK_KP"] = "10"
    try:
        forced = idx.search(q, 10)
    finally:
        for n, v in old.items():
            if v is None:
                os.environ.pop(n, None)
            else:
                os.environ[n] = v
    assert np.array_equal(base.ids, forced.ids) and np.array_equal(base.distances, forced.distances)


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("k", [24, 40, 64, 128])
def test_filter16_mid_k_default_path(metric, k):
    """16 < k <= 128 on a database large enough for the sampled bound pass
    (k >= ~33 here) takes the 1-pass path by default (k = 24 keeps 3xTF32):
    same answers as the oracle and as the forced 3xTF32 path."""
    rng = np.random.default_rng(900 + k)
    xb = rng.standard_normal((400_000, 32), dtype=np.float32)
    q = rng.standard_normal((96, 32), dtype=np.float32)
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    idx = FlatIndex(32, METRIC_IP if metric == "ip" else METRIC_L2, storage="fp32")
    idx.add(xb)
    res = idx.search(q, k)
    assert idx.last_plan()["kmode"] == (0 if k == 24 else 5)
    want_ids, want_dist = O.flat_search_blas(xb, q, k, metric)
    assert_parity(res.ids, res.distances, want_ids, want_dist)
    os.environ["FK_FP32_3X"] = "1"
    try:
        r3 = idx.search(q, k)
        assert idx.last_plan()["kmode"] == 0
    finally:
        del os.environ["FK_FP32_3X"]
    assert_parity(res.ids, res.distances, r3.ids, r3.distances)


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_filter16_split_query_operand_d768(metric):
    """d = 768 fp32: the scaled-fp16 query operand needs 384 TMEM columns, so
    the 1-pass filter runs the split plan (a_mode 3) -- identical to the
    whole-in-TMEM plan, and the oracle's answers."""
    rng = np.random.default_rng(768)
    xb = rng.standard_normal((20000, 768), dtype=np.float32)
    q = rng.standard_normal((150, 768), dtype=np.float32)
    idx = _index(768, metric)
    idx.add(xb)
    r = _search(idx, q, 10)
    assert idx.last_plan()["kmode"] == 5 and idx.last_plan()["a_mode"] == 3
    os.environ["FK_AMODE3"] = "0"
    try:
        r0 = _search(idx, q, 10)
        assert idx.last_plan()["a_mode"] == 0
    finally:
        del os.environ["FK_AMODE3"]
    assert np.array_equal(r.ids, r0.ids) and np.array_equal(r.distances, r0.distances)
    want_ids, want_dist = O.flat_search_blas(xb, q, 10, metric)
    assert_parity(r.ids, r.distances, want_ids, want_dist)


@pytest.mark.parametrize("nq", [20, 64, 129])
@pytest.mark.parametrize("nan_rows", [False, True])
def test_filter16_small_batches(nq, nan_rows):
    """One query tile split over every SM: S x 2 lists of k' per query.  The
    rescoring merge holds all of them (no spurious exact fallback -- a
    whole-base scan per query), and NaN rows (a NaN max norm) widen the band
    to infinity: those searches are answered exactly by the fallback."""
    rng = np.random.default_rng(nq)
    nb, d = 270_000, 32
    xb = rng.standard_normal((nb, d), dtype=np.float32)
    if nan_rows:
        xb[[5, 77, nb - 1], 3] = np.nan
    q = rng.standard_normal((nq, d), dtype=np.float32)
    idx = _index(d, "l2")
    idx.add(xb)
    r = _search(idx, q, 10)
    assert idx.last_plan()["kmode"] == 5
    with np.errstate(invalid="ignore"):
        want_ids, want_dist = O.flat_search_blas(xb, q, 10, "l2")
    assert_parity(r.ids, r.distances, want_ids, want_dist)


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("k", [12, 13, 14, 16])
def test_filter16_queue_slack_up_to_k16(metric, k):
    """Register queues keep k' - k >= 4 slots of slack (k <= 12: k' = 16;
    12 < k <= 16: k' = 32).  With k' = k a full queue drops a band member at
    almost every late insertion, the 64-entry overflow lists overflow and every
    query went to the whole-base exact fallback (k = 16 on 1M rows, 10k
    queries: 3.3 s instead of 5.7 ms).  Same answers as the oracle, and no
    fallback-sized slowdown against k = 10 on the same index."""
    import time
    rng = np.random.default_rng(1600 + k)
    nb, d, nq = 300_000, 32, 1000
    xb = rng.standard_normal((nb, d), dtype=np.float32)
    q = rng.standard_normal((nq, d), dtype=np.float32)
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    idx = FlatIndex(d, METRIC_IP if metric == "ip" else METRIC_L2, storage="fp32")
    idx.add(xb)

    def timed(kk):
        idx.search(q, kk)
        t0 = time.perf_counter()
        r = idx.search(q, kk)  # host arrays: returns after the device work
        return r, time.perf_counter() - t0

    _, t10 = timed(10)
    res, tk = timed(k)
    plan = idx.last_plan()
    assert plan["kmode"] == 5 and plan["kq"] // 100 == (16 if k <= 12 else 32)
    assert tk < 10 * t10 + 0.005, (tk, t10)
    want_ids, want_dist = O.flat_search_blas(xb, q[:200], k, metric)
    assert_parity(res.ids[:200], res.distances[:200], want_ids, want_dist)


@pytest.mark.parametrize("d,nb", [(256, 300_000), (768, 270_000)])
@pytest.mark.parametrize("nq", [20, 2000])
def test_filter16_k16_wide_rows(d, nb, nq):
    """32-deep queues with one epilogue group beside the wide query operands
    (d = 256: whole in TMEM; d = 768: the split plan), few and many query
    tiles: the oracle's answers."""
    rng = np.random.default_rng(d + nq)
    xb = rng.standard_normal((nb, d), dtype=np.float32)
    q = rng.standard_normal((nq, d), dtype=np.float32)
    from paper_2401_08281_b200 import METRIC_L2, FlatIndex
    idx = FlatIndex(d, METRIC_L2, storage="fp32")
    idx.add(xb)
    res = idx.search(q, 16)
    plan = idx.last_plan()
    assert plan["kmode"] == 5 and plan["kq"] // 100 == 32
    sub = slice(0, 40)
    want_ids, want_dist = O.flat_search_blas(xb, q[sub], 16, "l2")
    assert_parity(res.ids[sub], res.distances[sub], want_ids, want_dist)
