"""Range search (reference flat.py:121-144 via
Index.range_search core.py:152-155) against golden vectors of the real
reference (tests/golden/make_golden_range.py) and the oracle restatement."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from make_golden_range import CASES, range_inputs  # noqa: E402
from oracle import flat_oracle as O  # noqa: E402
from parity import assert_range_parity  # noqa: E402

GOLD = np.load(os.path.join(HERE, "golden", "golden_range.npz"))


def _want(name):
    return GOLD[f"{name}/lims"], GOLD[f"{name}/ids"], GOLD[f"{name}/dist"]


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_range_matches_reference(name):
    xb, q, metric, _, _ = range_inputs(name)
    radius = float(GOLD[f"{name}/radius"])
    got = O.flat_range_search(xb, q, radius, metric)
    assert_range_parity(got, _want(name), radius, metric, exact=CASES[name][4] == "ints")


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_range_matches_reference(name):
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    xb, q, metric, _, _ = range_inputs(name)
    radius = float(GOLD[f"{name}/radius"])
    idx = FlatIndex(xb.shape[1], METRIC_IP if metric == "ip" else METRIC_L2)
    idx.add(xb)
    res = idx.range_search(q, radius)
    assert res.lims.dtype == np.int64 and res.ids.dtype == np.int64 and res.distances.dtype == np.float32
    assert_range_parity((res.lims, res.ids, res.distances), _want(name), radius, metric,
                        exact=CASES[name][4] == "ints")


@pytest.mark.gpu
@pytest.mark.parametrize("storage", ["fp16", "bf16"])
@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("d", [96, 768])
def test_gpu_range_16bit_storage_vs_oracle_on_rounded_inputs(storage, metric, d):
    """(d = 768: the query operand is split between TMEM and smem, a_mode 3)"""
    import torch
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    rng = np.random.default_rng(77)
    xb = rng.standard_normal((20000 if d == 96 else 6000, d), dtype=np.float32)
    q = rng.standard_normal((64, d), dtype=np.float32)
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    dm = O.direct_distances(qr[:8], xr, metric)
    radius = float(np.quantile(dm, 0.995 if metric == "ip" else 0.005))
    idx = FlatIndex(d, METRIC_IP if metric == "ip" else METRIC_L2, storage=storage)
    idx.add(xb)
    res = idx.range_search(torch.from_numpy(q).cuda(), radius)  # device in -> device out
    assert res.ids.is_cuda
    want = O.flat_range_search(xr, qr, radius, metric)
    assert_range_parity((res.lims, res.ids, res.distances), want, radius, metric)


@pytest.mark.gpu
def test_gpu_range_known_answers_and_ids():
    """test_flat.py:163-196 known answers, custom ids, empty index."""
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    idx = FlatIndex(2, METRIC_L2)
    idx.add(np.array([[0, 0], [3, 4]], dtype=np.float32))
    assert idx.range_search(np.zeros((1, 2), np.float32), 0.25).row(0)[0].tolist() == [0]
    assert idx.range_search(np.zeros((1, 2), np.float32), 25.0).row(0)[0].tolist() == [0, 1]
    idx = FlatIndex(2, METRIC_L2)
    idx.add(np.array([[0, 0], [1, 0], [0, 0]], dtype=np.float32))
    assert idx.range_search(np.zeros((1, 2), np.float32), 1e-12).row(0)[0].tolist() == [0, 2]
    ip = FlatIndex(2, METRIC_IP)
    ip.add(np.array([[1, 0], [0, 1], [2, 0]], dtype=np.float32))
    assert ip.range_search(np.array([[1, 0]], np.float32), 1.0).row(0)[0].tolist() == [2, 0]
    idx = FlatIndex(2, METRIC_L2)
    idx.add_with_ids(np.array([[0, 0], [0, 0], [5, 5]], dtype=np.float32), np.array([70, 9, 4], dtype=np.int64))
    assert idx.range_search(np.zeros((1, 2), np.float32), 1.0).row(0)[0].tolist() == [9, 70]  # tie: smaller id first
    empty = FlatIndex(2, METRIC_L2)
    r = empty.range_search(np.zeros((3, 2), np.float32), 1.0)
    assert r.lims.tolist() == [0, 0, 0, 0] and len(r.ids) == 0


@pytest.mark.gpu
def test_gpu_range_candidate_overflow_rerun():
    """More candidates than the first buffer (nq*64 / 1M floor): the counted
    pass reruns with room for all of them (here: every pair, radius inf)."""
    from paper_2401_08281_b200 import METRIC_L2, FlatIndex
    rng = np.random.default_rng(5)
    xb = rng.standard_normal((40000, 16), dtype=np.float32)
    q = rng.standard_normal((40, 16), dtype=np.float32)
    idx = FlatIndex(16, METRIC_L2)
    idx.add(xb)
    res = idx.range_search(q, float("inf"))
    assert res.lims[-1] == 40 * 40000
    want = O.flat_range_search(xb, q, float("inf"), "l2")
    assert_range_parity((res.lims, res.ids, res.distances), want, float("inf"), "l2")
