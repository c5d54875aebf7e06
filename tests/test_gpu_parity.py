"""GPU parity: the sm_100a path (through the C ABI) vs the reference.

* every golden case (outputs of the real reference, tests/golden/) through
  ``FlatIndex`` with the tie-aware comparator;
* the reference's flat known-answer tests (test_flat.py) re-expressed;
* the raw tensor-core inner products vs fp64 (3xTF32 accuracy);
* plan invariance (split-N count, resident vs streamed queries) -> identical
  results;
* full-size (cfg2: 1M x 128) properties and a 256-query oracle check.
"""

import os

import numpy as np
import pytest

from cases import CASES, make_inputs
from oracle import flat_oracle as O
from parity import assert_parity, compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex, IndexFlatIP, IndexFlatL2, knn_recall  # noqa
from paper_2401_08281_b200.core import SearchResult  # noqa: E402

SMALL_K = [n for n, c in CASES.items() if c["k"] <= 32]
LARGE_K = [n for n, c in CASES.items() if c["k"] > 32]


def build_index(name):
    xb, q, k, metric, storage, ids = make_inputs(name)
    idx = FlatIndex(xb.shape[1], METRIC_IP if metric == "ip" else METRIC_L2, storage=storage)
    if xb.shape[0]:
        if ids is None:
            idx.add(xb)
        else:
            idx.add_with_ids(xb, ids)
    return idx, q, k


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_case(golden, name):
    idx, q, k = build_index(name)
    res = idx.search(q, k)
    assert res.ids.shape == (q.shape[0], k) and res.ids.dtype == np.int64
    assert res.distances.dtype == np.float32
    # the reference's Index.search output (its own nq < blas_threshold
    # dispatch: direct path for small batches, flat.py:58-62)
    s = assert_parity(res.ids, res.distances, golden[f"{name}/search_ids"], golden[f"{name}/search_dist"])
    assert s["strict_recall"] >= 0.999


def test_device_tensors_roundtrip(golden):
    xb, q, k, metric, storage, _ = make_inputs("cfg1_small_l2")
    idx = IndexFlatL2(xb.shape[1])
    idx.add(torch.from_numpy(xb).cuda())
    res = idx.search(torch.from_numpy(q).cuda(), k)
    assert res.ids.is_cuda and res.distances.is_cuda
    assert_parity(res.ids.cpu().numpy(), res.distances.cpu().numpy(), golden["cfg1_small_l2/blas_ids"],
                  golden["cfg1_small_l2/blas_dist"])
    D, I = idx.search(torch.from_numpy(q).cuda().half(), k)  # 16-bit queries are upcast exactly
    assert I.shape == (q.shape[0], k)


# ---------------------------------------------------------------- test_flat.py re-expressed
def test_nearest_of_two():
    idx = IndexFlatL2(2)
    idx.add(np.array([[0, 0], [1, 0]], np.float32))
    res = idx.search(np.array([[0.1, 0.0]], np.float32), 1)
    assert res.ids[0, 0] == 0
    assert res.distances[0, 0] == pytest.approx(0.01, rel=1e-5)


def test_self_query_is_first():
    xb = np.random.default_rng(0).normal(size=(50, 8)).astype(np.float32)
    idx = IndexFlatL2(8)
    idx.add(xb)
    res = idx.search(xb[17], 3)
    assert res.ids[0, 0] == 17
    assert res.distances[0, 0] == 0.0  # as test_flat.py:37-43 (direct path, nq < blas_threshold)


def test_k_equals_ntotal_is_permutation():
    rng = np.random.default_rng(1)
    idx = IndexFlatL2(4)
    idx.add(rng.normal(size=(64, 4)).astype(np.float32))
    res = idx.search(rng.normal(size=(5, 4)).astype(np.float32), 32)
    for row in res.ids:
        assert len(set(row.tolist())) == 32


def test_row_distances_monotone():
    rng = np.random.default_rng(2)
    xb = rng.normal(size=(100, 6)).astype(np.float32)
    q = rng.normal(size=(20, 6)).astype(np.float32)
    for metric in (METRIC_L2, METRIC_IP):
        idx = FlatIndex(6, metric)
        idx.add(xb)
        diffs = np.diff(idx.search(q, 10).distances, axis=1)
        assert np.all(diffs <= 0 if metric.descending else diffs >= 0)


def test_empty_index_returns_sentinels():
    idx = FlatIndex(4)
    res = idx.search(np.zeros((2, 4), np.float32), 3)
    assert np.all(res.ids == -1) and np.all(np.isinf(res.distances))


def test_dimension_mismatch():
    idx = FlatIndex(4)
    idx.add(np.zeros((3, 4), np.float32))
    with pytest.raises(ValueError):
        idx.search(np.zeros((1, 5), np.float32), 1)


def test_add_with_ids_reconstruct_remove_reset():
    xb = np.arange(12, dtype=np.float32).reshape(3, 4)
    idx = FlatIndex(4)
    idx.add_with_ids(xb, np.array([10, 20, 30]))
    assert np.array_equal(idx.reconstruct_batch(np.array([20])), xb[1:2])
    assert idx.search(xb[2], 1).ids[0, 0] == 30
    with pytest.raises(KeyError):
        idx.reconstruct_batch(np.array([99]))
    rng = np.random.default_rng(3)
    xr = rng.normal(size=(10, 4)).astype(np.float32)
    idx2 = FlatIndex(4)
    idx2.add(xr)
    assert idx2.remove_ids(np.array([3, 7])) == 2
    assert idx2.ntotal == 8
    res = idx2.search(xr, 8)
    assert 3 not in res.ids and 7 not in res.ids
    assert np.array_equal(idx2.reconstruct_batch(np.array([9])), xr[9:10])  # exact fp32 reconstruction
    idx2.reset()
    assert idx2.ntotal == 0
    assert np.all(idx2.search(xr[:2], 2).ids == -1)
    idx2.add(xr[:3])
    assert idx2.search(xr[1], 1).ids[0, 0] == 1


def test_identity_expansion_and_self_distance():
    idx = IndexFlatL2(2)
    idx.add(np.array([[0, 1]], np.float32))
    assert idx.search(np.array([[1, 0]], np.float32), 1).distances[0, 0] == pytest.approx(2.0)
    rng = np.random.default_rng(4)
    xb = rng.normal(size=(30, 16)).astype(np.float32)
    xb /= np.linalg.norm(xb, axis=1, keepdims=True)
    idx = IndexFlatL2(16)
    idx.add(xb)
    res = idx.search(xb, 1)
    assert np.all(np.abs(res.distances[:, 0]) <= 1e-6)
    assert np.all(res.distances >= 0)


def test_incremental_adds_equal_single_add():
    rng = np.random.default_rng(9)
    xb = rng.normal(size=(3000, 40)).astype(np.float32)
    q = rng.normal(size=(77, 40)).astype(np.float32)
    a = IndexFlatIP(40)
    a.add(xb)
    b = IndexFlatIP(40)
    for lo in range(0, 3000, 700):
        b.add(xb[lo:lo + 700])
    ra, rb = a.search(q, 16), b.search(q, 16)
    assert np.array_equal(ra.ids, rb.ids) and np.array_equal(ra.distances, rb.distances)


# ---------------------------------------------------------------- kernel-level checks
def test_tensor_core_inner_products_vs_fp64():
    """Raw TMEM accumulators (debug dump) vs exact fp64: 3xTF32 is fp32-faithful."""
    import ctypes
    from paper_2401_08281_b200 import _native as N
    rng = np.random.default_rng(5)
    xb = rng.standard_normal((700, 128), dtype=np.float32)
    q = rng.standard_normal((300, 128), dtype=np.float32)
    exact = q.astype(np.float64) @ xb.astype(np.float64).T
    for storage in ("fp32", "fp16", "bf16"):
        idx = FlatIndex(128, METRIC_IP, storage=storage)
        idx.add(xb)
        buf = torch.zeros((300, 700), dtype=torch.float32, device="cuda")
        N.check(N.lib().fk_debug_set_ip_dump(idx._h, ctypes.c_void_p(buf.data_ptr())))
        idx.search(q, 4)
        N.check(N.lib().fk_debug_set_ip_dump(idx._h, None))
        got = buf.cpu().numpy().astype(np.float64)
        if storage == "fp32":
            want, tol = exact, 2e-6
        else:
            qr, xr = O.round_to(q, storage).astype(np.float64), O.round_to(xb, storage).astype(np.float64)
            want, tol = qr @ xr.T, 2e-6
        scale = np.abs(q).astype(np.float64) @ np.abs(xb).astype(np.float64).T
        err = np.max(np.abs(got - want) / scale)
        assert err < tol, (storage, err)


def test_folded_norm_accumulators():
    """bf16 L2 with free K padding folds the norms into the operands: the raw
    TMEM accumulator is xn - 2 q.x (base rows stored as -2x | xn split in three
    bf16, queries as q | 1 1 1).  Exact products, fp32 accumulation."""
    import ctypes
    from paper_2401_08281_b200 import _native as N
    rng = np.random.default_rng(15)
    xb = rng.standard_normal((700, 96), dtype=np.float32)
    q = rng.standard_normal((300, 96), dtype=np.float32)
    qr, xr = O.round_to(q, "bf16").astype(np.float64), O.round_to(xb, "bf16").astype(np.float64)
    xn = (xr * xr).sum(1).astype(np.float32).astype(np.float64)
    want = xn[None, :] - 2.0 * (qr @ xr.T)
    idx = FlatIndex(96, METRIC_L2, storage="bf16")
    idx.add(xb)
    buf = torch.zeros((300, 700), dtype=torch.float32, device="cuda")
    N.check(N.lib().fk_debug_set_ip_dump(idx._h, ctypes.c_void_p(buf.data_ptr())))
    idx.search(q, 4)
    N.check(N.lib().fk_debug_set_ip_dump(idx._h, None))
    got = buf.cpu().numpy().astype(np.float64)
    scale = xn[None, :] + 2.0 * (np.abs(qr) @ np.abs(xr).T)
    assert np.max(np.abs(got - want) / scale) < 2e-6
    # reconstruct undoes the -2x scaling exactly
    rec = idx.reconstruct_batch(np.arange(50))
    rec = rec.cpu().numpy() if hasattr(rec, "cpu") else rec
    assert np.array_equal(rec, xr[:50].astype(np.float32))


def test_fold_matches_unfolded_layout():
    """Same top-k from the folded (MODE 3) and the separate-norm-tile layouts."""
    rng = np.random.default_rng(16)
    xb = rng.standard_normal((30000, 96), dtype=np.float32)
    q = rng.standard_normal((500, 96), dtype=np.float32)
    res = []
    for nofold in ("0", "1"):
        os.environ["FK_NO_FOLD"] = nofold
        try:
            idx = FlatIndex(96, METRIC_L2, storage="bf16")
            idx.add(xb)
            res.append(idx.search(q, 10))
        finally:
            del os.environ["FK_NO_FOLD"]
    xr, qr = O.round_to(xb, "bf16"), O.round_to(q, "bf16")
    want_ids, want_dist = O.flat_search_blas(xr, qr, 10, "l2")
    for r in res:
        assert_parity(r.ids, r.distances, want_ids, want_dist)


PLAN_VARIANTS = [("FK_FORCE_S", "1"), ("FK_FORCE_S", "7"), ("FK_FORCE_S", "64"), ("FK_FORCE_AMODE", "1"),
                 ("FK_FORCE_AMODE", "2"), ("FK_EPI", "8"), ("FK_STAGES", "2"), ("FK_ACC", "2"), ("FK_ACC", "3")]


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
@pytest.mark.parametrize("force", PLAN_VARIANTS)
def test_plan_invariance(force, storage):
    rng = np.random.default_rng(6)
    xb = rng.standard_normal((20000, 100), dtype=np.float32)
    q = rng.standard_normal((333, 100), dtype=np.float32)
    idx = FlatIndex(100, METRIC_L2, storage=storage)
    idx.add(xb)
    base = idx.search(q, 10)
    os.environ[force[0]] = force[1]
    try:
        alt = idx.search(q, 10)
    finally:
        del os.environ[force[0]]
    assert np.array_equal(base.ids, alt.ids)
    assert np.array_equal(base.distances, alt.distances)


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
@pytest.mark.parametrize("data", ["normal", "ints"])
@pytest.mark.parametrize("k", [1, 10, 32])
def test_many_chunks_bounded_merge(storage, data, k):
    """More than 128 split-N lists per query (small L2-resident chunks at large
    nb): register-queue lists go through the bounded merge; the order must
    equal the single-list order, ties included (ints: massive exact ties)."""
    rng = np.random.default_rng(21)
    if data == "ints":
        xb = rng.integers(0, 4, size=(40000, 24)).astype(np.float32)
        q = rng.integers(0, 4, size=(150, 24)).astype(np.float32)
    else:
        xb = rng.standard_normal((40000, 24), dtype=np.float32)
        q = rng.standard_normal((150, 24), dtype=np.float32)
    idx = FlatIndex(24, METRIC_L2, storage=storage)
    idx.add(xb)
    os.environ["FK_FORCE_S"] = "200"
    try:
        res = idx.search(q, k)
        plan = idx.last_plan()
    finally:
        del os.environ["FK_FORCE_S"]
    assert plan["S"] * plan["epi"] // 4 > 128, plan
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    want_ids, want_dist = O.flat_search_blas(xr, qr, k, "l2")
    assert_parity(res.ids, res.distances, want_ids, want_dist)
    if data == "ints":  # exact integer distances: the order must be identical
        assert np.array_equal(np.asarray(res.ids), want_ids)


# ---------------------------------------------------------------- full size (cfg2 shape)
@pytest.fixture(scope="module")
def cfg2_index():
    xb = np.random.default_rng(0).standard_normal((1_000_000, 128), dtype=np.float32)
    idx = IndexFlatL2(128)
    idx.add(torch.from_numpy(xb).cuda())
    return idx, xb


def test_cfg2_self_queries_and_order(cfg2_index):
    idx, xb = cfg2_index
    rows = np.arange(0, 1_000_000, 100)  # 10k base rows as queries
    res = idx.search(torch.from_numpy(xb[rows]).cuda(), 10)
    ids = res.ids.cpu().numpy()
    dist = res.distances.cpu().numpy()
    assert np.array_equal(ids[:, 0], rows)
    assert np.all(np.abs(dist[:, 0]) <= 1e-3)
    assert np.all(np.diff(dist, axis=1) >= 0)
    assert np.all(ids >= 0) and np.all(ids < 1_000_000)


def test_cfg2_parity_vs_oracle_subset(cfg2_index):
    idx, xb = cfg2_index
    q = np.random.default_rng(1).standard_normal((10_000, 128), dtype=np.float32)
    res = idx.search(torch.from_numpy(q).cuda(), 10)  # full nq=10k launch
    sub = np.arange(0, 10_000, 40)  # 250 queries checked on the CPU oracle
    want_ids, want_dist = O.flat_search_blas(xb, q[sub], 10, "l2")
    s = assert_parity(res.ids.cpu().numpy()[sub], res.distances.cpu().numpy()[sub], want_ids, want_dist)
    assert s["strict_recall"] >= 0.999


# ---------------------------------------------------------------- large k (candidate buffers + radix select)
@pytest.mark.parametrize("k,metric,data", [(33, "l2", "gauss"), (100, "ip", "gauss"), (257, "l2", "ints"),
                                           (1024, "l2", "gauss"), (2048, "ip", "gauss"), (1000, "l2", "ints")])
def test_large_k_vs_oracle(k, metric, data):
    rng = np.random.default_rng(k)
    if data == "ints":  # massive exact ties: exercises (key, position) ordering in compaction and merge
        xb = rng.integers(0, 3, size=(9000, 24)).astype(np.float32)
        q = rng.integers(0, 3, size=(70, 24)).astype(np.float32)
    else:
        xb = rng.standard_normal((12000, 72), dtype=np.float32)
        q = rng.standard_normal((150, 72), dtype=np.float32)
    idx = FlatIndex(xb.shape[1], METRIC_L2 if metric == "l2" else METRIC_IP)
    idx.add(xb)
    res = idx.search(q, k)
    want_ids, want_dist = O.flat_search_blas(xb, q, k, metric)
    assert_parity(res.ids, res.distances, want_ids, want_dist)
    if data == "ints":  # integer data: exact arithmetic on both sides -> identical order
        assert np.array_equal(res.ids, want_ids)


@pytest.mark.parametrize("force", [("FK_FORCE_S", "1"), ("FK_FORCE_S", "40"), ("FK_EPI", "8"),
                                   ("FK_MERGE_SMC", "64"), ("FK_FORCE_AMODE", "2")])
def test_large_k_plan_invariance(force):
    rng = np.random.default_rng(7)
    xb = rng.integers(0, 5, size=(30000, 40)).astype(np.float32)
    q = rng.integers(0, 5, size=(200, 40)).astype(np.float32)
    idx = IndexFlatL2(40)
    idx.add(xb)
    base = idx.search(q, 300)
    os.environ[force[0]] = force[1]
    try:
        alt = idx.search(q, 300)
    finally:
        del os.environ[force[0]]
    assert np.array_equal(base.ids, alt.ids) and np.array_equal(base.distances, alt.distances)
    want_ids, _ = O.flat_search_blas(xb, q, 300, "l2")
    assert np.array_equal(base.ids, want_ids)


@pytest.mark.parametrize("storage,metric,d", [("bf16", "l2", 96), ("fp16", "ip", 128), ("bf16", "ip", 96)])
def test_16bit_epilogue_width_invariance(storage, metric, d):
    """Long fold / IP searches run one epilogue group (query operand in TMEM,
    two accumulators) instead of two (A in smem, four): the same answers."""
    rng = np.random.default_rng(96)
    xb = rng.standard_normal((60000, d), dtype=np.float32)
    q = rng.standard_normal((700, d), dtype=np.float32)
    idx = FlatIndex(d, METRIC_IP if metric == "ip" else METRIC_L2, storage=storage)
    idx.add(xb)
    base = idx.search(q, 10)
    assert idx.last_plan()["epi"] == 8
    for width in ("4", "8"):
        os.environ["FK_EPI"] = width
        try:
            alt = idx.search(q, 10)
            assert idx.last_plan()["epi"] == int(width)
        finally:
            del os.environ["FK_EPI"]
        assert np.array_equal(base.ids, alt.ids) and np.array_equal(base.distances, alt.distances)
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    want_ids, want_dist = O.flat_search_blas(xr, qr, 10, metric)
    assert_parity(base.ids, base.distances, want_ids, want_dist)


def test_k_equals_ntotal_large():
    rng = np.random.default_rng(1)
    idx = IndexFlatL2(4)
    xb = rng.normal(size=(64, 4)).astype(np.float32)
    idx.add(xb)
    res = idx.search(rng.normal(size=(5, 4)).astype(np.float32), 64)
    for row in res.ids:
        assert sorted(row.tolist()) == list(range(64))
    res = idx.search(xb[:3], 100)  # k > ntotal pads -1 / +inf
    assert np.all(res.ids[:, 64:] == -1) and np.all(np.isinf(res.distances[:, 64:]))


def test_k_above_max_rejected():
    idx = IndexFlatL2(4)
    idx.add(np.zeros((10, 4), np.float32))
    with pytest.raises(NotImplementedError):
        idx.search(np.zeros((1, 4), np.float32), 4096)


@pytest.mark.parametrize("k,metric", [(100, "l2"), (1024, "ip")])
def test_large_k_estimated_bound_path(k, metric):
    """nb large enough that the prefix-sample bound estimate is used."""
    rng = np.random.default_rng(k)
    xb = rng.standard_normal((300_000, 32), dtype=np.float32)
    q = rng.standard_normal((130, 32), dtype=np.float32)
    idx = FlatIndex(32, METRIC_L2 if metric == "l2" else METRIC_IP)
    idx.add(xb)
    res = idx.search(q, k)
    os.environ["FK_NO_EST"] = "1"
    try:
        ref = idx.search(q, k)
    finally:
        del os.environ["FK_NO_EST"]
    assert np.array_equal(res.ids, ref.ids) and np.array_equal(res.distances, ref.distances)
    sub = np.arange(0, 130, 13)
    want_ids, want_dist = O.flat_search_blas(xb, q[sub], k, metric)
    assert_parity(res.ids[sub], res.distances[sub], want_ids, want_dist)


def test_large_k_estimate_fails_certification_and_reruns():
    """Adversarial order: the prefix sample holds all near neighbours, so the
    estimated bound is too tight (< k survivors) -> exact rerun must kick in."""
    rng = np.random.default_rng(3)
    near = rng.standard_normal((40_000, 16), dtype=np.float32) * 0.01
    far = rng.standard_normal((260_000, 16), dtype=np.float32) + 50.0
    xb = np.vstack([near, far])
    q = rng.standard_normal((64, 16), dtype=np.float32) * 0.01
    idx = IndexFlatL2(16)
    idx.add(xb)
    res = idx.search(q, 200)
    want_ids, want_dist = O.flat_search_blas(xb, q, 200, "l2")
    assert_parity(res.ids, res.distances, want_ids, want_dist)


@pytest.mark.parametrize("storage,metric,nq", [("bf16", "l2", 300), ("fp16", "l2", 130), ("bf16", "ip", 257)])
def test_split_query_operand_l2_and_ragged_tiles(storage, metric, nq):
    """a_mode 3 on the L2 (base-norm tile) and bf16 paths, with a ragged last
    query tile; equal to the whole-in-TMEM plan and to the oracle."""
    rng = np.random.default_rng(769)
    xb = rng.standard_normal((20000, 768), dtype=np.float32)
    q = rng.standard_normal((nq, 768), dtype=np.float32)
    idx = FlatIndex(768, METRIC_IP if metric == "ip" else METRIC_L2, storage=storage)
    idx.add(xb)
    base = idx.search(q, 10)
    assert idx.last_plan()["a_mode"] == 3
    os.environ["FK_AMODE3"] = "0"
    try:
        alt = idx.search(q, 10)
        assert idx.last_plan()["a_mode"] == 0
    finally:
        del os.environ["FK_AMODE3"]
    assert np.array_equal(base.ids, alt.ids) and np.array_equal(base.distances, alt.distances)
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    want_ids, want_dist = O.flat_search_blas(xr, qr, 10, metric)
    assert_parity(base.ids, base.distances, want_ids, want_dist)


@pytest.mark.parametrize("k", [10, 100])
def test_large_query_operand_tile_plans(k):
    """d = 768 16-bit (cfg4 shape): the query operand needs 384 TMEM columns.
    The default plan splits it (a_mode 3: 8 K-chunks in TMEM beside two
    128-column accumulators, 4 in smem); FK_AMODE3=0 keeps it whole beside ONE
    accumulator, FK_BN=64 the round-1 plan of two 64-column accumulators --
    identical answers, and the oracle's on the rounded inputs."""
    rng = np.random.default_rng(768)
    xb = rng.standard_normal((30000, 768), dtype=np.float32)
    q = rng.standard_normal((200, 768), dtype=np.float32)
    idx = FlatIndex(768, METRIC_IP, storage="fp16")
    idx.add(xb)
    base = idx.search(q, k)
    assert idx.last_plan()["bn"] == 128 and idx.last_plan()["a_mode"] == 3 and idx.last_plan()["acc_stages"] == 2
    for env, check in (("FK_AMODE3", lambda p: p["a_mode"] == 0 and p["acc_stages"] == 1),
                       ("FK_BN", lambda p: p["bn"] == 64)):
        os.environ[env] = "0" if env == "FK_AMODE3" else "64"
        try:
            alt = idx.search(q, k)
            assert check(idx.last_plan()), idx.last_plan()
        finally:
            del os.environ[env]
        assert np.array_equal(base.ids, alt.ids) and np.array_equal(base.distances, alt.distances)
    xr, qr = O.round_to(xb, "fp16"), O.round_to(q, "fp16")
    want_ids, want_dist = O.flat_search_blas(xr, qr, k, "ip")
    assert_parity(base.ids, base.distances, want_ids, want_dist)


@pytest.mark.parametrize("d,storage,metric,k", [(520, "fp16", "l2", 1), (600, "bf16", "ip", 64), (700, "fp16", "ip", 100),
                                                 (765, "bf16", "l2", 10), (768, "bf16", "l2", 33)])
def test_split_query_operand_shapes(d, storage, metric, k):
    """a_mode 3 across d in (512, 768] (d = 765 bf16 L2 folds its norms into
    the last, smem-resident K-chunk), queue and candidate-buffer k: equal to
    the whole-in-TMEM plan and to the oracle."""
    rng = np.random.default_rng(d + k)
    xb = rng.standard_normal((12000, d), dtype=np.float32)
    q = rng.standard_normal((181, d), dtype=np.float32)
    idx = FlatIndex(d, METRIC_IP if metric == "ip" else METRIC_L2, storage=storage)
    idx.add(xb)
    base = idx.search(q, k)
    assert idx.last_plan()["a_mode"] == 3
    os.environ["FK_AMODE3"] = "0"
    try:
        alt = idx.search(q, k)
    finally:
        del os.environ["FK_AMODE3"]
    assert np.array_equal(base.ids, alt.ids) and np.array_equal(base.distances, alt.distances)
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    want_ids, want_dist = O.flat_search_blas(xr, qr, k, metric)
    assert_parity(base.ids, base.distances, want_ids, want_dist)


@pytest.mark.parametrize("storage,metric", [("fp16", "l2"), ("fp32", "ip")])
def test_large_k_estimate_small_ratio(storage, metric):
    """rows/k between 256 and 512 (300k rows, k = 1000): the estimated
    large-k bound samples 32 tiles; certified or rerun, the oracle's answers."""
    rng = np.random.default_rng(1000)
    xb = rng.standard_normal((300_000, 32), dtype=np.float32)
    q = rng.standard_normal((40, 32), dtype=np.float32)
    idx = FlatIndex(32, METRIC_IP if metric == "ip" else METRIC_L2, storage=storage)
    idx.add(xb)
    res = idx.search(q, 1000)
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    want_ids, want_dist = O.flat_search_blas(xr, qr, 1000, metric)
    assert_parity(res.ids, res.distances, want_ids, want_dist)
