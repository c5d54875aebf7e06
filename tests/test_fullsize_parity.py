"""GPU parity at the FULL BASELINE.json config sizes.

Every config is searched with its real shape (all nq = 1k / 10k queries in
one launch, so the planner takes the branches the benchmark takes: split-N
lists, 64-column tiles, large-k estimate pass, the bounded merge) and a
query subset is checked against the CPU oracle.  For the multi-GB databases
(cfg4: 10M x 768 fp16, cfg5: 100M x 96 bf16) the oracle runs shard by shard
(1M rows, global positions) and the shard lists are merged by the
reference's (value, position) order (``oracle.merge_topk``) -- exactly the
unsharded reference answer (SURVEY 8(d) "Parity for cfg4/5").  The rows are
generated on the device (as bench.py does), added to the index and copied
to the host chunk by chunk, so host RAM never holds the whole database.

Tolerances are the north star's: ids equal except among ties within 1e-5
relative distance, distances within 1e-4 relative, tie-aware recall 1.0
(tests/parity.py).  16-bit storage: the oracle runs on the same RNE-rounded
values (round_to), the GPU accumulates exact 16-bit products in fp32.
"""

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import flat_oracle as O
from parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from bench import CONFIGS, gen_base, gen_base_device, gen_queries  # noqa: E402
from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex  # noqa: E402

NQ_CHECK = int(os.environ.get("FK_FULLSIZE_NQ", "256"))
CHUNK = 1_000_000


def _shard_topk(xr, lo, qr, k, metric):
    """Oracle top-k of one 1M-row shard with GLOBAL positions as ids."""
    pos, val = O.flat_search_blas(xr, qr, k, metric, ids=np.arange(lo, lo + xr.shape[0], dtype=np.int64))
    return pos, val


def build_and_oracle(cfg, sub):
    """Build the full-size index shard by shard; evaluate the oracle for the
    query subset `sub` on each shard in a thread pool; merge."""
    nb, d, k, metric, storage = cfg["nb"], cfg["d"], cfg["k"], cfg["metric"], cfg["storage"]
    idx = FlatIndex(d, METRIC_L2 if metric == "l2" else METRIC_IP, storage=storage)
    q = gen_queries(cfg)
    qr = O.round_to(q[sub], storage)
    gate = threading.Semaphore(12)  # bound the host chunks in flight

    def job(xh, lo):
        try:
            return _shard_topk(O.round_to(xh, storage), lo, qr, k, metric)
        finally:
            gate.release()

    futures = []
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        for lo in range(0, nb, CHUNK):
            hi = min(nb, lo + CHUNK)
            if nb <= 1_000_000:
                xh = gen_base(cfg, lo, hi)
                idx.add(torch.from_numpy(xh).cuda())
            else:
                x = gen_base_device(cfg, lo, hi)
                idx.add(x)
                xh = x.cpu().numpy()
                del x
            gate.acquire()
            futures.append(ex.submit(job, xh, lo))
            del xh
        parts = [f.result() for f in futures]
    torch.cuda.empty_cache()
    want_pos, want_dist = O.merge_topk(parts, k, descending=(metric == "ip"))
    return idx, q, want_pos, want_dist


@pytest.mark.parametrize("cfgn", [1, 3, 4, 5])
def test_fullsize_config_vs_sharded_oracle(cfgn):
    cfg = CONFIGS[cfgn]
    nq = cfg["nq"]
    n_check = min(nq, NQ_CHECK)
    sub = np.linspace(0, nq - 1, n_check).astype(np.int64)
    idx, q, want_ids, want_dist = build_and_oracle(cfg, sub)
    assert idx.ntotal == cfg["nb"]
    res = idx.search(torch.from_numpy(q).cuda(), cfg["k"])  # the full nq launch
    plan = idx.last_plan()
    got_ids = res.ids.cpu().numpy()[sub]
    got_dist = res.distances.cpu().numpy()[sub]
    s = assert_parity(got_ids, got_dist, want_ids, want_dist)
    assert s["strict_recall"] >= 0.999, s
    print(f"cfg{cfgn}: {n_check} queries checked, plan {plan}, stats {s}")
    del idx
    torch.cuda.empty_cache()
