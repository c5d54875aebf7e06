"""World-size-2 gloo test of the sharded index's host logic on CPU.

The per-rank GPU index and CUDA merge kernel are replaced by CPU stand-ins
built on the oracle (test infrastructure), so this checks what the GPU run
cannot check on a 1-GPU box: row partitioning, global positions across
several adds, the all-gather plumbing and the (distance, global position)
merge order == the unsharded reference answer.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import flat_oracle as O  # noqa: E402


class OracleLocal:
    """CPU stand-in for the per-rank FlatIndex (exact same API surface)."""

    def __init__(self, d, metric, storage, device):
        self.d, self.mv = d, ("ip" if getattr(metric, "descending", False) else "l2")
        self.xb = np.zeros((0, d), np.float32)
        self.ids = np.zeros(0, np.int64)

    def add_with_ids(self, x, ids):
        self.xb = np.vstack([self.xb, np.asarray(x, np.float32)])
        self.ids = np.concatenate([self.ids, np.asarray(ids, np.int64)])

    def reset(self):
        self.__init__(self.d, None, None, None)

    def search_with_positions(self, q, k):
        from paper_2401_08281_b200.core import SearchResult
        pos, dist_ = O.flat_search_blas(self.xb, np.asarray(q), k, self.mv)  # positions (ids=None)
        ids = np.where(pos >= 0, self.ids[np.maximum(pos, 0)], -1) if len(self.ids) else pos
        return SearchResult(ids, dist_, k), pos


def oracle_merge(mv, D, P, I, k):
    D, P, I = D.numpy(), P.numpy(), I.numpy()
    G, nq, _ = D.shape
    outD = np.full((nq, k), -np.inf if mv == "ip" else np.inf, np.float32)
    outI = np.full((nq, k), -1, np.int64)
    for q in range(nq):
        cand = [(O.monotone_key(np.float32(-D[g, q, j] if mv == "ip" else D[g, q, j])[None])[0], P[g, q, j],
                 D[g, q, j], I[g, q, j]) for g in range(G) for j in range(k) if P[g, q, j] >= 0]
        cand.sort(key=lambda t: (int(t[0]), int(t[1])))
        for j, c in enumerate(cand[:k]):
            outD[q, j], outI[q, j] = c[2], c[3]
    return torch.from_numpy(outD), torch.from_numpy(outI)


def _worker(rank, world, port, metric, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2401_08281_b200.core import METRIC_IP, METRIC_L2
        from paper_2401_08281_b200.sharded import ShardedFlatIndex
        m = METRIC_IP if metric == "ip" else METRIC_L2
        idx = ShardedFlatIndex(16, m, local_factory=OracleLocal, merge_fn=oracle_merge)
        rng = np.random.default_rng(0)
        xb1 = rng.standard_normal((301, 16), dtype=np.float32)
        xb2 = rng.integers(0, 3, (150, 16)).astype(np.float32)  # exact ties across shards
        q = rng.standard_normal((23, 16), dtype=np.float32)
        q[:5] = xb2[:5]
        idx.add(xb1)
        idx.add_with_ids(xb2, np.arange(1000, 1150))
        res = idx.search(q, 12)
        big = idx.search(q, 500)  # k > ntotal: padding
        if rank == 0:
            result_q.put((res.ids, res.distances, big.ids, big.distances, idx.ntotal))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_sharded_equals_single_index(metric):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, metric, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, dist_, big_ids, big_dist, ntotal = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ntotal == 451
    rng = np.random.default_rng(0)
    xb1 = rng.standard_normal((301, 16), dtype=np.float32)
    xb2 = rng.integers(0, 3, (150, 16)).astype(np.float32)
    qq = rng.standard_normal((23, 16), dtype=np.float32)
    qq[:5] = xb2[:5]
    xb = np.vstack([xb1, xb2])
    all_ids = np.concatenate([np.arange(301), np.arange(1000, 1150)])
    want_ids, want_dist = O.flat_search_blas(xb, qq, 12, metric, ids=all_ids)
    # exact equality: (distance, global position) order == the unsharded order
    assert np.array_equal(ids, want_ids)
    np.testing.assert_allclose(dist_, want_dist, rtol=1e-5, atol=1e-5)
    w2, d2 = O.flat_search_blas(xb, qq, 500, metric, ids=all_ids)
    assert np.array_equal(big_ids, w2)
    assert np.all(big_ids[:, 451:] == -1)


def test_shard_range_partition():
    from paper_2401_08281_b200.sharded import shard_range
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
