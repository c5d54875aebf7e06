"""Pin the CPU oracle (oracle/flat_oracle.py) to the reference.

* every golden case (tests/golden/golden.npz, produced by running the real
  reference, tests/golden/make_golden.py) is reproduced by the oracle;
* the reference's own selection tests (test_core.py:86-128) and flat
  known-answer tests (test_flat.py:31-43, 60-81, 107-120) hold for it.
"""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from cases import CASES, digest, make_inputs
from oracle import flat_oracle as O
from parity import assert_parity


def argsort_oracle(values, descending=False):
    return sorted(range(len(values)), key=lambda i: (-values[i] if descending else values[i], i))


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_golden(golden, name):
    xb, q, k, metric, storage, ids = make_inputs(name)
    assert str(golden[f"{name}/digest"]) == digest(xb, q), "regenerated inputs differ from the golden run"
    got_ids, got_dist = O.flat_search_blas(xb, q, k, metric, ids=ids)
    ref_ids = golden[f"{name}/blas_ids"]
    ref_dist = golden[f"{name}/blas_dist"]
    # same algorithm, same host BLAS -> normally bit-identical; allow ulp-level
    # BLAS kernel differences across hosts through the tie-aware comparator
    if np.array_equal(got_ids, ref_ids):
        np.testing.assert_allclose(got_dist, ref_dist, rtol=1e-6, atol=1e-6)
    else:
        assert_parity(got_ids, got_dist, ref_ids, ref_dist, rel_dist=1e-5, abs_dist=1e-5)


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_search_equals_blas_path(golden, name):
    """The reference's own dispatch (direct path for nq < 20) gives the same
    answer as its BLAS path up to ties -- the drop-in may use one GPU path."""
    assert_parity(golden[f"{name}/search_ids"], golden[f"{name}/search_dist"],
                  golden[f"{name}/blas_ids"], golden[f"{name}/blas_dist"])


def test_known_answers(golden):
    assert golden["nearest_of_two/blas_ids"][0, 0] == 0
    assert golden["nearest_of_two/blas_dist"][0, 0] == pytest.approx(0.01, rel=1e-5)
    assert golden["identity_expansion/blas_dist"][0, 0] == pytest.approx(2.0)
    assert golden["add_with_ids/blas_ids"][0, 0] == 30
    assert np.all(golden["empty_index/blas_ids"] == -1)
    assert np.all(np.isinf(golden["empty_index/blas_dist"]))
    assert np.array_equal(golden["self_query/blas_ids"][:, 0], np.arange(30))
    for row in golden["k_eq_ntotal/blas_ids"]:
        assert sorted(row.tolist()) == list(range(64))
    assert np.all(golden["k_gt_ntotal_l2/blas_ids"][:, 5:] == -1)
    assert np.all(golden["k_gt_ntotal_l2/blas_dist"][:, 5:] == np.inf)
    assert np.all(golden["k_gt_ntotal_ip/blas_dist"][:, 5:] == -np.inf)


class TestTopkRows:
    """core.py:205-236 behaviour (test_core.py:86-128)."""

    def test_basic(self):
        ids, vals = O.topk_rows(np.array([[5, 1, 3, 2]], np.float32), 2)
        assert ids[0].tolist() == [1, 3] and vals[0].tolist() == [1, 2]

    def test_tie_break_by_smaller_id(self):
        ids, _ = O.topk_rows(np.array([[1, 1, 2]], np.float32), 2)
        assert ids[0].tolist() == [0, 1]

    def test_padding(self):
        ids, vals = O.topk_rows(np.array([[4.0, 2.0]], np.float32), 4)
        assert ids[0].tolist() == [1, 0, -1, -1]
        assert vals[0, 2] == np.inf and vals[0, 3] == np.inf

    def test_k_zero_rejected(self):
        with pytest.raises(ValueError):
            O.topk_rows(np.array([[1.0]], np.float32), 0)

    def test_descending(self):
        ids, vals = O.topk_rows(np.array([[5, 1, 3]], np.float32), 2, descending=True)
        assert ids[0].tolist() == [0, 2] and vals[0].tolist() == [5, 3]

    def test_nan_sorts_last_and_negzero_first(self):
        ids, _ = O.topk_rows(np.array([[np.nan, 0.0, -0.0, np.inf]], np.float32), 4)
        assert ids[0].tolist() == [2, 1, 3, 0]

    def test_matches_sort_oracle_random(self):
        vals = np.random.default_rng(0).random(1000).astype(np.float32)
        ids, got = O.topk_rows(vals[None, :], 100)
        want = argsort_oracle(vals)[:100]
        assert ids[0].tolist() == want
        assert np.array_equal(got[0], vals[want])

    @settings(max_examples=200, deadline=None)
    @given(st.lists(st.integers(0, 7), min_size=1, max_size=60), st.integers(1, 70), st.booleans())
    def test_property_equals_stable_argsort(self, raw, k, descending):
        vals = np.array(raw, dtype=np.float32)
        ids, _ = O.topk_rows(vals[None, :], k, descending)
        got = [i for i in ids[0].tolist() if i >= 0]
        want = argsort_oracle(vals, descending)[:k]
        assert got == want[: len(got)] and len(got) == min(k, len(vals))


def test_monotone_key_order():
    v = np.array([-np.inf, -2.0, -0.0, 0.0, 1e-30, 3.0, np.inf, np.nan], np.float32)
    keys = O.monotone_key(v)
    assert np.all(np.diff(keys.astype(np.int64)) > 0)


def test_knn_recall():
    a = np.array([[7, 1, 3]])
    b = np.array([[3, 7, 9]])
    assert O.knn_recall(a, b, 1, 3) == 1.0
    assert O.knn_recall(np.array([[7, 5]]), np.array([[3, 7]]), 2, 2) == 0.5
    with pytest.raises(ValueError):
        O.knn_recall(a, b, 4, 3)


def test_exact_fp64_agrees_with_reference_order(golden):
    """The fp64 second opinion agrees with the reference BLAS order modulo ties."""
    xb, q, k, metric, _, _ = make_inputs("blas_1000x32")
    pos, d64 = O.flat_search_exact(xb, q, k, metric)
    assert_parity(pos, d64, golden["blas_1000x32/blas_ids"], golden["blas_1000x32/blas_dist"])


def test_round_to_bf16_is_rne():
    x = np.array([1.0, 1.00390625, 1.0078125, 1.01171875, -3.3], np.float32)
    r = O.round_to(x, "bf16")
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.0078125 and r[3] == 1.015625
    assert abs(r[4] - -3.3) < 0.02
