"""1-GPU tests of the multi-GPU merge path.

The box has one GPU, so the row-sharded index is exercised two ways:
* G shards held by G ``FlatIndex`` objects on the same device, each searched
  with positions, positions offset to GLOBAL ones, stacked [G, nq, k] and
  merged by the CUDA ``shard_merge_kernel`` (``fk_merge_shards``): the result
  must equal the unsharded index bit for bit (same per-pair values, same
  (value, global position) order) and the oracle;
* ``ShardedFlatIndex`` end to end under a world-size-1 NCCL process group
  (position table, all-gather plumbing, merge kernel).
"""

import os
import socket

import numpy as np
import pytest

from oracle import flat_oracle as O
from parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex  # noqa: E402
from paper_2401_08281_b200.sharded import native_merge, shard_range  # noqa: E402


def sharded_search(xb, q, k, metric, storage, G, bounds=None):
    nb = xb.shape[0]
    Ds, Ps, Is = [], [], []
    for g in range(G):
        lo, hi = bounds[g] if bounds else shard_range(nb, g, G)
        idx = FlatIndex(xb.shape[1], METRIC_L2 if metric == "l2" else METRIC_IP, storage=storage)
        if hi > lo:
            idx.add_with_ids(torch.from_numpy(xb[lo:hi]).cuda(), torch.arange(lo, hi, device="cuda") + 1000)
        idx.set_plan_rows(nb)
        res, P = idx.search_with_positions(torch.from_numpy(q).cuda(), k)
        Ds.append(res.distances)
        Is.append(res.ids)
        Ps.append(torch.where(P >= 0, P + lo, P))
    D, I = native_merge(metric, torch.stack(Ds), torch.stack(Ps), torch.stack(Is), k)
    return D.cpu().numpy(), I.cpu().numpy()


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("storage", ["fp32", "bf16", "fp16"])
@pytest.mark.parametrize("G", [2, 5, 33])
def test_shard_merge_equals_unsharded(metric, storage, G):
    rng = np.random.default_rng(G)
    xb = rng.standard_normal((20_000, 40), dtype=np.float32)
    q = rng.standard_normal((300, 40), dtype=np.float32)
    k = 10
    D, I = sharded_search(xb, q, k, metric, storage, G)
    full = FlatIndex(40, METRIC_L2 if metric == "l2" else METRIC_IP, storage=storage)
    full.add_with_ids(xb, np.arange(20_000) + 1000)
    ref = full.search(q, k)
    assert np.array_equal(I, ref.ids) and np.array_equal(D, ref.distances)
    xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
    want_ids, want_dist = O.flat_search_blas(xr, qr, k, metric, ids=np.arange(20_000) + 1000)
    assert_parity(I, D, want_ids, want_dist)


@pytest.mark.parametrize("k", [1, 32, 200])
def test_shard_merge_exact_ties_uneven_shards(k):
    """Integer data (massive exact ties across shards), uneven and empty
    shards, k larger than some shards: identical to the oracle's order."""
    rng = np.random.default_rng(k)
    xb = rng.integers(0, 3, size=(6000, 12)).astype(np.float32)
    q = rng.integers(0, 3, size=(90, 12)).astype(np.float32)
    bounds = [(0, 100), (100, 100), (100, 2500), (2500, 2600), (2600, 6000)]
    D, I = sharded_search(xb, q, k, "l2", "fp32", len(bounds), bounds)
    want_ids, want_dist = O.flat_search_blas(xb, q, k, "l2", ids=np.arange(6000) + 1000)
    assert np.array_equal(I, want_ids)
    assert np.array_equal(D, want_dist)


def test_shard_merge_k_beyond_total_pads():
    xb = np.random.default_rng(0).standard_normal((7, 8), dtype=np.float32)
    q = np.random.default_rng(1).standard_normal((3, 8), dtype=np.float32)
    D, I = sharded_search(xb, q, 12, "ip", "fp32", 3)
    assert np.all(I[:, 7:] == -1) and np.all(np.isneginf(D[:, 7:]))
    want_ids, _ = O.flat_search_blas(xb, q, 12, "ip", ids=np.arange(7) + 1000)
    assert np.array_equal(I, want_ids)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_index_world1_nccl():
    import torch.distributed as dist
    from paper_2401_08281_b200 import ShardedFlatIndex
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda:0"))
    try:
        rng = np.random.default_rng(5)
        xb = rng.standard_normal((300_000, 32), dtype=np.float32)
        q = rng.standard_normal((200, 32), dtype=np.float32)
        sh = ShardedFlatIndex(32, METRIC_L2, storage="fp32", device=0)
        sh.add(xb[:120_000])
        sh.add_with_ids(xb[120_000:], np.arange(120_000, 300_000) + 7)
        res = sh.search(torch.from_numpy(q).cuda(), 10)
        ids_table = np.concatenate([np.arange(120_000), np.arange(120_000, 300_000) + 7])
        want_ids, want_dist = O.flat_search_blas(xb, q, 10, "l2", ids=ids_table)
        assert_parity(res.ids.cpu().numpy(), res.distances.cpu().numpy(), want_ids, want_dist)
        # the shard planned the fp32 algorithm on the global row count
        sh.local.search(q[:50], 10)
        assert sh.local.last_plan()["kmode"] in (4, 5)
    finally:
        dist.destroy_process_group()
