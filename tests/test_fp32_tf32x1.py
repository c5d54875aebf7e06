"""Experimental fp32 algorithm (FK_FP32_ALGO=1, kernel MODE 4): raw fp32
storage, ONE tf32 tensor-core pass ranking k' >= k candidates per list, then
certification (tf32 error band) + exact fp32 rescoring of the survivors, with
an exact brute-force fallback for uncertified queries.  Must return the same
answers as the default 3xTF32 path under the north-star parity rules."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))
sys.path.insert(0, os.path.dirname(HERE))

from cases import CASES, make_inputs  # noqa: E402
from oracle import flat_oracle as O  # noqa: E402
from parity import assert_parity  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))


def _index(d, metric):
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    os.environ["FK_FP32_ALGO"] = "1"
    try:
        return FlatIndex(d, METRIC_IP if metric == "ip" else METRIC_L2, storage="fp32")
    finally:
        del os.environ["FK_FP32_ALGO"]


FP32_CASES = [n for n in CASES if make_inputs(n)[4] == "fp32"]


@pytest.mark.parametrize("name", FP32_CASES)
def test_tf32x1_golden(name):
    xb, q, k, metric, storage, ids = make_inputs(name)
    idx = _index(xb.shape[1], metric)
    if xb.shape[0]:
        if ids is None:
            idx.add(xb)
        else:
            idx.add_with_ids(xb, ids)
    res = idx.search(q, k)
    assert_parity(res.ids, res.distances, GOLD[f"{name}/blas_ids"], GOLD[f"{name}/blas_dist"])


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("k", [1, 10, 16, 32, 100])
def test_tf32x1_vs_oracle(metric, k):
    rng = np.random.default_rng(99 + k)
    xb = rng.standard_normal((60000, 64), dtype=np.float32)
    q = rng.standard_normal((300, 64), dtype=np.float32)
    idx = _index(64, metric)
    idx.add(xb)
    res = idx.search(q, k)
    want_ids, want_dist = O.flat_search_blas(xb, q, k, metric)
    assert_parity(res.ids, res.distances, want_ids, want_dist)


def test_tf32x1_exact_ties_use_the_certified_fallback():
    """Integer data with massive exact ties: the band test cannot certify the
    queries, the exact fallback must reproduce the reference order exactly."""
    rng = np.random.default_rng(3)
    xb = rng.integers(0, 3, size=(5000, 16)).astype(np.float32)
    q = rng.integers(0, 3, size=(20, 16)).astype(np.float32)
    idx = _index(16, "l2")
    idx.add(xb)
    res = idx.search(q, 10)
    want_ids, want_dist = O.flat_search_blas(xb, q, 10, "l2")
    assert np.array_equal(res.ids, want_ids)
    assert np.array_equal(res.distances, want_dist)


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_default_split_storage_uses_1x_filter_for_small_k(metric):
    """Default fp32 (hi/lo split) index, k <= 16 over >= 262144 rows: the
    1-pass filter runs on the hi half and rescoring uses hi + lo; the answer
    must equal the 3xTF32 path's (FK_FP32_3X=1) and the oracle's."""
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    rng = np.random.default_rng(11)
    xb = rng.standard_normal((300000, 48), dtype=np.float32)
    q = rng.standard_normal((200, 48), dtype=np.float32)
    idx = FlatIndex(48, METRIC_IP if metric == "ip" else METRIC_L2)
    idx.add(xb)
    res = idx.search(q, 10)
    os.environ["FK_FP32_3X"] = "1"
    try:
        res3 = idx.search(q, 10)
    finally:
        del os.environ["FK_FP32_3X"]
    want_ids, want_dist = O.flat_search_blas(xb, q, 10, metric)
    assert_parity(res.ids, res.distances, want_ids, want_dist)
    assert_parity(res3.ids, res3.distances, want_ids, want_dist)


@pytest.mark.parametrize("force", [("FK_EPI", "8"), ("FK_FORCE_S", "7"), ("FK_FORCE_S", "13"), ("FK_FORCE_AMODE", "1"),
                                   ("FK_STAGES", "4"), ("FK_FP32_3X", "1")])
def test_1x_path_plan_invariance(force):
    """Default fp32 index over >= 262144 rows (1-pass filter + exact rescoring):
    bit-identical answers across epilogue widths, odd/even chunk lengths,
    operand placement, pipeline depth and the 3xTF32 path (regression: with
    two epilogue groups the TMEM query operand of the next unit must wait for
    every MMA of the previous unit)."""
    import torch
    from paper_2401_08281_b200 import METRIC_L2, FlatIndex
    rng = np.random.default_rng(12)
    xb = rng.standard_normal((300000, 128), dtype=np.float32)
    q = torch.from_numpy(rng.standard_normal((3000, 128), dtype=np.float32)).cuda()
    idx = FlatIndex(128, METRIC_L2)
    idx.add(torch.from_numpy(xb).cuda())
    base = idx.search(q, 10)
    os.environ[force[0]] = force[1]
    try:
        alt = idx.search(q, 10)
    finally:
        del os.environ[force[0]]
    if force[0] == "FK_FP32_3X":  # different arithmetic: parity, not bit equality
        assert_parity(alt.ids.cpu().numpy(), alt.distances.cpu().numpy(), base.ids.cpu().numpy(),
                      base.distances.cpu().numpy())
    else:
        assert torch.equal(base.ids, alt.ids) and torch.equal(base.distances, alt.distances)


@pytest.mark.parametrize("k", [10, 50])
def test_raw_storage_exact_ties_all_k(k):
    """Raw-fp32 storage (FK_FP32_ALGO=1): massive exact ties around the k-th
    for both list kinds (register queue k <= 16, candidate buffers k > 16);
    uncertified rows must go through the exact fallback and match the
    reference order exactly."""
    rng = np.random.default_rng(33 + k)
    xb = rng.integers(0, 3, size=(300000, 16)).astype(np.float32)
    q = rng.integers(0, 3, size=(40, 16)).astype(np.float32)
    idx = _index(16, "l2")
    idx.add(xb)
    res = idx.search(q, k)
    want_ids, want_dist = O.flat_search_blas(xb, q, k, "l2")
    assert np.array_equal(res.ids, want_ids)
    assert np.array_equal(res.distances, want_dist)


def test_tf32_exact_data_needs_no_fallback():
    """SIFT-like integer data is exactly representable in tf32 (every lo part
    is zero, detected at add/stage time): the band collapses to the fp32
    accumulation slack, so queries certify without the exact fallback."""
    import subprocess
    code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
from paper_2401_08281_b200 import FlatIndex, METRIC_L2
from oracle import flat_oracle as O
from parity import assert_parity
rng = np.random.default_rng(8)
xb = rng.integers(0, 256, size=(300000, 128)).astype(np.float32)
q = rng.integers(0, 256, size=(500, 128)).astype(np.float32)
idx = FlatIndex(128, METRIC_L2); idx.add(xb)
res = idx.search(q, 10)
wi, wd = O.flat_search_blas(xb, q, 10, "l2")
assert np.array_equal(res.ids, wi) and np.array_equal(res.distances, wd)
'''
    env = dict(os.environ, FK_DIAG="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(HERE))
    assert r.returncode == 0, r.stderr[-2000:]
    assert "uncertified=0" in r.stderr, r.stderr[-2000:]
