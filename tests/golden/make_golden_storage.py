"""Golden storage-op and refine_search vectors from the REAL reference
(build container only)::

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_storage.py

* ``refine/<case>``: annkit ``refine_search(fast, exact, q, k, shortlist)``
  (core.py:368-394).  ``fast`` is a reference ``FlatIndex`` over a coarsened
  copy of the data (the approximate stage), ``exact`` a ``FlatIndex`` over
  the true vectors with the same user ids, so re-ranking changes the order.
  The shortlist fast returned is stored too, so the GPU re-ranking can be
  checked on exactly the candidates the reference saw.
* ``remove/<case>``: ``add_with_ids`` -> ``remove_ids`` (flat.py:46-56) ->
  ``ids``, ``vectors`` and a search over the survivors;
  ``reconstruct_batch`` of an id list with repeats (flat.py:34-44).

Inputs are regenerated from seeds by ``refine_inputs`` / ``remove_inputs``.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

REFINE_CASES = {
    # name: (nb, nq, d, metric, kind, k, shortlist)
    "l2_basic": (2000, 50, 32, "l2", "normal", 10, 40),
    "ip_basic": (2000, 50, 32, "ip", "normal", 10, 40),
    "l2_ints_ties": (1500, 40, 8, "l2", "ints", 8, 64),
    "ip_ints_ties": (1500, 40, 8, "ip", "ints", 8, 64),
    "l2_pad": (30, 12, 16, "l2", "normal", 10, 50),  # shortlist > ntotal: -1 candidates
    "l2_k_eq_short": (1000, 20, 24, "l2", "normal", 16, 16),
    "l2_d128": (4000, 64, 128, "l2", "normal", 10, 100),
}

REMOVE_CASES = {
    # name: (nb, d, metric, n_remove, with_dup_ids)
    "l2_some": (3000, 24, "l2", 700, False),
    "ip_some": (3000, 24, "ip", 50, False),
    "l2_all": (400, 8, "l2", 400, False),
    "l2_dups": (1200, 16, "l2", 100, True),
}


def refine_inputs(name):
    nb, nq, d, metric, kind, k, shortlist = REFINE_CASES[name]
    rng = np.random.default_rng(sum(map(ord, name)) + 7)
    if kind == "ints":
        xb = rng.integers(0, 3, size=(nb, d)).astype(np.float32)
        q = rng.integers(0, 3, size=(nq, d)).astype(np.float32)
        coarse = xb.copy()
        coarse[:, -1] = 0.0  # fast stage ignores the last coordinate
    else:
        xb = rng.standard_normal((nb, d), dtype=np.float32)
        q = rng.standard_normal((nq, d), dtype=np.float32)
        coarse = (np.round(xb * 2.0) / 2.0).astype(np.float32)  # coarse quantisation
    ids = (rng.permutation(nb).astype(np.int64) * 3 + 11)  # non-sequential user ids
    return xb, coarse, q, ids, metric, k, shortlist


def remove_inputs(name):
    nb, d, metric, n_remove, dups = REMOVE_CASES[name]
    rng = np.random.default_rng(sum(map(ord, name)) + 13)
    xb = rng.standard_normal((nb, d), dtype=np.float32)
    ids = np.arange(nb, dtype=np.int64) * 2 + 5
    if dups:
        ids[rng.choice(nb, nb // 4, replace=False)] = ids[rng.choice(nb, nb // 4)]  # repeated ids
    kill = rng.choice(ids, n_remove, replace=False) if n_remove < nb else ids.copy()
    kill = np.concatenate([kill, np.array([10 ** 12, -3], dtype=np.int64)])  # unknown ids are ignored
    q = rng.standard_normal((30, d), dtype=np.float32)
    recon = rng.choice(ids, 25)
    recon = np.concatenate([recon, recon[:5]])  # repeats
    return xb, ids, kill, q, recon, metric


def main() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    from annkit.core import METRIC_IP, METRIC_L2, refine_search
    from annkit.flat import FlatIndex

    out = {}
    for name in REFINE_CASES:
        xb, coarse, q, ids, metric, k, shortlist = refine_inputs(name)
        m = METRIC_IP if metric == "ip" else METRIC_L2
        fast, exact = FlatIndex(xb.shape[1], m), FlatIndex(xb.shape[1], m)
        fast.add_with_ids(coarse, ids)
        exact.add_with_ids(xb, ids)
        cand = fast.search(q, shortlist)
        res = refine_search(fast, exact, q, k, shortlist)
        out[f"refine/{name}/cand"] = cand.ids
        out[f"refine/{name}/ids"] = res.ids
        out[f"refine/{name}/dist"] = res.distances
        print(f"refine {name:14s} changed-vs-fast={np.mean(res.ids != cand.ids[:, :k]):.3f}")
    for name in REMOVE_CASES:
        xb, ids, kill, q, recon, metric = remove_inputs(name)
        m = METRIC_IP if metric == "ip" else METRIC_L2
        idx = FlatIndex(xb.shape[1], m)
        idx.add_with_ids(xb, ids)
        rec = idx.reconstruct_batch(recon)
        removed = idx.remove_ids(kill)
        out[f"remove/{name}/recon"] = rec
        out[f"remove/{name}/removed"] = np.array(removed)
        out[f"remove/{name}/ids"] = idx.ids
        out[f"remove/{name}/vectors"] = idx.vectors
        if idx.ntotal:
            res = idx.search(q, 7)
            out[f"remove/{name}/s_ids"] = res.ids
            out[f"remove/{name}/s_dist"] = res.distances
        print(f"remove {name:10s} removed={removed} left={idx.ntotal}")
    np.savez_compressed(os.path.join(HERE, "golden_storage.npz"), **out)


if __name__ == "__main__":
    main()
