"""Device-side storage ops and refine_search.

* ``refine_search`` (reference core.py:368-394) and ``remove_ids`` /
  ``reconstruct_batch`` / the id -> position map (flat.py:34-56) against
  golden vectors produced by the REAL reference
  (tests/golden/make_golden_storage.py) and the oracle restatement.
* CPU tests pin the oracle to the golden vectors; GPU tests run the CUDA path
  (``fk_refine``, ``fk_remove_ids``, ``fk_positions``) through the C ABI.
"""
import os

import numpy as np
import pytest

from make_golden_storage import REFINE_CASES, REMOVE_CASES, refine_inputs, remove_inputs
from oracle import flat_oracle as O
from parity import assert_parity

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden_storage.npz"))


# ---------------------------------------------------------------- oracle pinning (CPU)
@pytest.mark.parametrize("name", list(REFINE_CASES))
def test_oracle_refine_matches_reference(name):
    xb, coarse, q, ids, metric, k, shortlist = refine_inputs(name)
    cand = GOLD[f"refine/{name}/cand"]
    got_ids, got_dist = O.refine_rerank(xb, ids, q, cand, k, metric)
    assert_parity(got_ids, got_dist, GOLD[f"refine/{name}/ids"], GOLD[f"refine/{name}/dist"])
    if REFINE_CASES[name][4] == "ints":  # exact integer distances: identical order
        assert np.array_equal(got_ids, GOLD[f"refine/{name}/ids"])


@pytest.mark.parametrize("name", list(REMOVE_CASES))
def test_oracle_remove_matches_reference(name):
    xb, ids, kill, q, recon, metric = remove_inputs(name)
    assert np.array_equal(xb[O.positions(ids, recon)], GOLD[f"remove/{name}/recon"])
    v, i, removed = O.remove_ids(xb, ids, kill)
    assert removed == int(GOLD[f"remove/{name}/removed"])
    assert np.array_equal(i, GOLD[f"remove/{name}/ids"])
    assert np.array_equal(v, GOLD[f"remove/{name}/vectors"].reshape(v.shape))


def test_oracle_positions_last_wins_and_keyerror():
    table = np.array([5, 7, 5, 9], dtype=np.int64)
    assert O.positions(table, [5, 9, 7]).tolist() == [2, 3, 1]
    with pytest.raises(KeyError):
        O.positions(table, [6])


# ---------------------------------------------------------------- GPU
def _flat(d, metric, storage="fp32"):
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex
    return FlatIndex(d, METRIC_IP if metric == "ip" else METRIC_L2, storage=storage)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(REFINE_CASES))
def test_gpu_refine_matches_reference(name):
    from paper_2401_08281_b200 import refine_search
    xb, coarse, q, ids, metric, k, shortlist = refine_inputs(name)
    fast, exact = _flat(xb.shape[1], metric), _flat(xb.shape[1], metric)
    fast.add_with_ids(coarse, ids)
    exact.add_with_ids(xb, ids)
    res = refine_search(fast, exact, q, k, shortlist)
    assert isinstance(res.ids, np.ndarray) and res.ids.shape == (q.shape[0], k)
    assert_parity(res.ids, res.distances, GOLD[f"refine/{name}/ids"], GOLD[f"refine/{name}/dist"])
    if REFINE_CASES[name][4] == "ints":
        assert np.array_equal(res.ids, GOLD[f"refine/{name}/ids"])
        assert np.array_equal(res.distances, GOLD[f"refine/{name}/dist"])


@pytest.mark.gpu
@pytest.mark.parametrize("storage", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_gpu_refine_vs_oracle_on_same_shortlist(storage, metric):
    """Re-ranking of the GPU fast index's own shortlist equals the oracle's
    re-ranking of that shortlist over the stored (rounded) vectors; CUDA
    queries return CUDA tensors."""
    import torch
    from paper_2401_08281_b200 import refine_search
    rng = np.random.default_rng(3)
    xb = rng.standard_normal((6000, 48), dtype=np.float32)
    q = rng.standard_normal((70, 48), dtype=np.float32)
    ids = rng.permutation(6000).astype(np.int64) + 100
    fast, exact = _flat(48, metric, "bf16"), _flat(48, metric, storage)
    fast.add_with_ids(xb, ids)
    exact.add_with_ids(xb, ids)
    res = refine_search(fast, exact, torch.from_numpy(q).cuda(), 12, 60)
    assert res.ids.is_cuda and res.distances.is_cuda
    cand = fast.search(q, 60).ids
    want_ids, want_dist = O.refine_rerank(O.round_to(xb, storage), ids, q, cand, 12, metric)
    assert_parity(res.ids.cpu().numpy(), res.distances.cpu().numpy(), want_ids, want_dist)


@pytest.mark.gpu
def test_gpu_refine_errors():
    from paper_2401_08281_b200 import refine_search
    rng = np.random.default_rng(0)
    xb = rng.standard_normal((100, 8), dtype=np.float32)
    fast, exact = _flat(8, "l2"), _flat(8, "l2")
    fast.add_with_ids(xb, np.arange(100) + 1000)
    exact.add_with_ids(xb[:50], np.arange(50) + 1000)  # exact lacks half of fast's ids
    with pytest.raises(ValueError):
        refine_search(fast, exact, xb[:3], 10, 5)  # shortlist < k (core.py:371-372)
    with pytest.raises(KeyError):
        refine_search(fast, exact, xb[60:63], 5, 10)  # unknown id (reconstruct_batch KeyError)
    with pytest.raises(ValueError):
        refine_search(fast, _flat(4, "l2"), xb[:3], 5, 10)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(REMOVE_CASES))
@pytest.mark.parametrize("cuda_ids", [False, True])
def test_gpu_remove_and_reconstruct_match_reference(name, cuda_ids):
    import torch
    xb, ids, kill, q, recon, metric = remove_inputs(name)
    idx = _flat(xb.shape[1], metric)
    idx.add_with_ids(xb, ids)
    rec = idx.reconstruct_batch(torch.from_numpy(recon).cuda() if cuda_ids else recon)
    rec = rec.cpu().numpy() if cuda_ids else rec
    assert np.array_equal(rec, GOLD[f"remove/{name}/recon"])
    removed = idx.remove_ids(torch.from_numpy(kill).cuda() if cuda_ids else kill)
    assert removed == int(GOLD[f"remove/{name}/removed"])
    assert idx.ntotal == len(GOLD[f"remove/{name}/ids"])
    assert np.array_equal(idx.ids, GOLD[f"remove/{name}/ids"])
    assert np.array_equal(idx.vectors, GOLD[f"remove/{name}/vectors"].reshape(idx.ntotal, xb.shape[1]))
    if idx.ntotal:
        res = idx.search(q, 7)
        assert_parity(res.ids, res.distances, GOLD[f"remove/{name}/s_ids"], GOLD[f"remove/{name}/s_dist"])
        # after compaction the index answers exactly like a fresh one holding the survivors
        fresh = _flat(xb.shape[1], metric)
        fresh.add_with_ids(GOLD[f"remove/{name}/vectors"].reshape(idx.ntotal, -1), GOLD[f"remove/{name}/ids"])
        ref = fresh.search(q, 7)
        assert np.array_equal(res.ids, ref.ids) and np.array_equal(res.distances, ref.distances)
        with pytest.raises(KeyError):
            idx.reconstruct_batch(np.array([int(kill[0])]))


@pytest.mark.gpu
def test_gpu_remove_large_multi_slice_bf16():
    """Compaction over more rows than one 256 MB gather slice (bf16 d=768:
    1536 B/row -> 174k rows per slice) keeps order and the search answer."""
    import torch
    n, d = 400_000, 768
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((n, d), device="cuda", generator=g)
    idx = _flat(d, "ip", "bf16")
    idx.add(x)
    kill = torch.arange(0, n, 3, device="cuda")
    assert idx.remove_ids(kill) == kill.numel()
    keep = torch.ones(n, dtype=torch.bool, device="cuda")
    keep[kill] = False
    survivors = torch.nonzero(keep).reshape(-1)
    assert np.array_equal(idx.ids, survivors.cpu().numpy())
    pick = survivors[::9973]
    got = idx.reconstruct_batch(pick)
    want = x[pick].to(torch.bfloat16).float()
    assert torch.equal(got, want)
    fresh = _flat(d, "ip", "bf16")
    fresh.add_with_ids(x[survivors], survivors)
    q = torch.randn((64, d), device="cuda", generator=g)
    a, b = idx.search(q, 10), fresh.search(q, 10)
    assert torch.equal(a.ids, b.ids) and torch.equal(a.distances, b.distances)
