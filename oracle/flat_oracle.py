"""CPU restatement of the reference's exact flat k-NN path -- TEST INFRASTRUCTURE ONLY.

This module is the parity oracle.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` leg may import it; the
product package (``paper_2401_08281_b200``) never does, and has no CPU
fallback.

It restates, in plain numpy, the reference annkit BLAS search path
(``/root/reference`` = arxiv/paper_2401_08281):

* ``monotone_key``      <- ``pkg/src/annkit/core.py:193-197`` (_monotone_key)
* ``topk_rows``         <- ``pkg/src/annkit/core.py:205-236``
* ``add_norms``         <- ``pkg/src/annkit/flat.py:31`` (einsum f32 norms at add)
* ``flat_search_blas``  <- ``pkg/src/annkit/flat.py:94-118`` (256-query chunks,
                           ``(qn + xn) - 2 ip`` in f32, clamp at 0, top-k)
* ``finish``            <- ``pkg/src/annkit/flat.py:68-73`` (position -> id)
* ``knn_recall``        <- ``pkg/src/annkit/core.py:314-327``
* ``flat_range_search`` <- ``pkg/src/annkit/flat.py:121-144`` (direct pairwise
                           distances, <= radius / >= for IP, (value, id) order)
* ``flat_search_direct``<- ``pkg/src/annkit/flat.py:76-91`` (flat_search: the
                           direct path FlatIndex._search takes for batches below
                           config.blas_threshold, flat.py:58-62) with pairwise
                           -> dist_one (``_ckernels.pyx:49-57``): L2 sum (q-x)^2,
                           IP sum q x, here accumulated in fp64 and rounded once
* ``refine_rerank``     <- ``pkg/src/annkit/core.py:368-394`` (refine_search's
                           re-ranking of a given shortlist: reconstruct from
                           the exact index, direct distances, (value, id) order)
* ``remove_ids``        <- ``pkg/src/annkit/flat.py:46-56`` (isin mask, order kept)
* ``positions``         <- ``pkg/src/annkit/flat.py:34-41`` ({id: pos}: last wins)
* ``merge_topk``        <- the total order of ``core.py:205-236`` (64-bit key
                           ``monotone(value) << 32 | column``) applied to the
                           union of per-shard top-k lists carrying GLOBAL
                           columns: equals ``topk_rows`` over the concatenated
                           rows (each shard's top-k holds every global top-k
                           member of that shard).  Used to evaluate the oracle
                           over a large database shard by shard.

Parity pinning: ``tests/test_oracle.py`` checks this restatement against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by importing and running the real reference in the build container.
"""

from __future__ import annotations

import numpy as np

QUERY_CHUNK = 256  # flat.py:11 (_QUERY_CHUNK)

METRIC_L2 = "l2"
METRIC_IP = "ip"


def monotone_key(values: np.ndarray) -> np.ndarray:
    """float32 -> order-preserving uint32 (NaN above +inf, -0.0 below +0.0).

    Restates core.py:193-197.
    """
    bits = np.ascontiguousarray(values, dtype=np.float32).view(np.uint32)
    neg = bits >= np.uint32(0x80000000)
    return np.where(neg, ~bits, bits | np.uint32(0x80000000))


def topk_rows(distances: np.ndarray, k: int, descending: bool = False):
    """Row-wise top-k with (value, column) lexicographic order; pads -1 / worst.

    Restates core.py:205-236 (64-bit composite key = key<<32 | column,
    np.partition then np.sort).
    """
    if k < 1:
        raise ValueError("k must be >= 1")
    distances = np.atleast_2d(distances)
    nq, n = distances.shape
    vals = np.ascontiguousarray(distances, dtype=np.float32)
    key_vals = -vals if descending else vals
    cols = np.arange(n, dtype=np.uint64)
    keys = (monotone_key(key_vals).astype(np.uint64) << np.uint64(32)) | cols
    kk = min(k, n)
    if kk > 0:
        part = np.partition(keys, kk - 1, axis=1)[:, :kk] if kk < n else keys
        part = np.sort(part, axis=1)
        top_ids = (part & np.uint64(0xFFFFFFFF)).astype(np.int64)
        top_vals = np.take_along_axis(vals, top_ids, axis=1)
    else:
        top_ids = np.empty((nq, 0), dtype=np.int64)
        top_vals = np.empty((nq, 0), dtype=np.float32)
    if kk < k:
        pad = np.float32(-np.inf) if descending else np.float32(np.inf)
        top_ids = np.hstack([top_ids, np.full((nq, k - kk), -1, dtype=np.int64)])
        top_vals = np.hstack([top_vals, np.full((nq, k - kk), pad, dtype=np.float32)])
    return top_ids, top_vals


def merge_topk(parts, k: int, descending: bool = False):
    """Merge per-shard (global positions (nq, k_s) int64, values (nq, k_s) f32)
    lists into the top-k under the reference's (value, column) order
    (core.py:205-236); -1 / worst padding as topk_rows."""
    pos = np.concatenate([p for p, _ in parts], axis=1)
    vals = np.concatenate([v for _, v in parts], axis=1).astype(np.float32)
    nq = pos.shape[0]
    key_vals = -vals if descending else vals
    keys = (monotone_key(key_vals).astype(np.uint64) << np.uint64(32)) | pos.astype(np.uint64)
    keys = np.where(pos >= 0, keys, np.uint64(0xFFFFFFFFFFFFFFFF))
    order = np.argsort(keys, axis=1, kind="stable")[:, :k]
    out_pos = np.take_along_axis(pos, order, axis=1)
    out_val = np.take_along_axis(vals, order, axis=1)
    if out_pos.shape[1] < k:
        pad = k - out_pos.shape[1]
        out_pos = np.hstack([out_pos, np.full((nq, pad), -1, np.int64)])
        out_val = np.hstack([out_val, np.full((nq, pad), np.nan, np.float32)])
    worst = np.float32(-np.inf) if descending else np.float32(np.inf)
    out_val = np.where(out_pos >= 0, out_val, worst).astype(np.float32)
    return out_pos.astype(np.int64), out_val


def add_norms(xb: np.ndarray) -> np.ndarray:
    """Squared norms of stored vectors, f32 einsum (flat.py:31)."""
    xb = np.ascontiguousarray(xb, dtype=np.float32)
    return np.einsum("nd,nd->n", xb, xb)


def finish(ids_table: np.ndarray, pos: np.ndarray, ntotal: int) -> np.ndarray:
    """Storage position -> user id, keeping -1 sentinels (flat.py:68-73)."""
    if ntotal == 0:
        return pos
    return np.where(pos >= 0, ids_table[np.maximum(pos, 0)], -1)


def flat_search_blas(xb: np.ndarray, q: np.ndarray, k: int, metric: str = METRIC_L2,
                     norms: np.ndarray | None = None, ids: np.ndarray | None = None,
                     chunk: int = QUERY_CHUNK):
    """Exact top-k by the norm decomposition; returns (ids int64, dist float32).

    Restates flat.py:94-118: per ``chunk`` queries, ``ip = q @ xb.T`` (f32
    sgemm), L2: ``dmat = qn[:,None] + norms[None,:] - 2.0*ip`` then
    ``maximum(dmat, 0)``; IP: ``dmat = ip``; ``topk_rows`` (descending for IP);
    then position -> id.
    """
    xb = np.ascontiguousarray(xb, dtype=np.float32)
    q = np.ascontiguousarray(q, dtype=np.float32)
    if q.ndim == 1:
        q = q[None, :]
    nq = q.shape[0]
    nb = xb.shape[0]
    if norms is None:
        norms = add_norms(xb)
    if ids is None:
        ids = np.arange(nb, dtype=np.int64)
    all_ids = np.empty((nq, k), dtype=np.int64)
    all_dist = np.empty((nq, k), dtype=np.float32)
    descending = metric == METRIC_IP
    for lo in range(0, nq, chunk):
        hi = min(lo + chunk, nq)
        ip = q[lo:hi] @ xb.T
        if metric == METRIC_L2:
            qn = np.einsum("nd,nd->n", q[lo:hi], q[lo:hi])
            dmat = qn[:, None] + norms[None, :] - 2.0 * ip
            np.maximum(dmat, 0.0, out=dmat)
        else:
            dmat = ip
        pos, vals = topk_rows(dmat, k, descending)
        all_ids[lo:hi] = pos
        all_dist[lo:hi] = vals
    return finish(ids, all_ids, nb), all_dist


def flat_search_direct(xb: np.ndarray, q: np.ndarray, k: int, metric: str = METRIC_L2,
                       ids: np.ndarray | None = None, rows: int = 4096):
    """Direct-path top-k (flat.py:76-91): per-pair direct distances in fp64
    (difference form for L2), rounded to fp32, ranked by ``topk_rows``."""
    xb = np.ascontiguousarray(xb, dtype=np.float32)
    q = np.atleast_2d(np.ascontiguousarray(q, dtype=np.float32))
    nq, nb = q.shape[0], xb.shape[0]
    q64 = q.astype(np.float64)
    dmat = np.empty((nq, nb), dtype=np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        for lo in range(0, nb, rows):
            x64 = xb[lo:lo + rows].astype(np.float64)
            if metric == METRIC_L2:
                d = ((q64[:, None, :] - x64[None, :, :]) ** 2).sum(-1)
            else:
                d = q64 @ x64.T
            dmat[:, lo:lo + rows] = d.astype(np.float32)
    if ids is None:
        ids = np.arange(nb, dtype=np.int64)
    pos, vals = topk_rows(dmat, k, metric == METRIC_IP)
    return finish(ids, pos, nb), vals


def flat_search_exact(xb: np.ndarray, q: np.ndarray, k: int, metric: str = METRIC_L2):
    """fp64-exact distances (direct differences), same (value, position) order.

    Not a reference function: a second, rounding-free opinion used by the
    tie-aware comparator to classify near-ties.  Returns (pos, dist64).
    """
    xb64 = np.asarray(xb, dtype=np.float64)
    q64 = np.atleast_2d(np.asarray(q, dtype=np.float64))
    if metric == METRIC_L2:
        d = ((q64[:, None, :] - xb64[None, :, :]) ** 2).sum(-1)
        order = np.lexsort((np.broadcast_to(np.arange(xb64.shape[0]), d.shape), d), axis=1)
    else:
        d = q64 @ xb64.T
        order = np.lexsort((np.broadcast_to(np.arange(xb64.shape[0]), d.shape), -d), axis=1)
    pos = order[:, :k]
    return pos, np.take_along_axis(d, pos, axis=1)


def knn_recall(result_ids: np.ndarray, gt_ids: np.ndarray, n: int, k: int) -> float:
    """n-recall@k, ignoring -1 (core.py:314-327)."""
    if n > k:
        raise ValueError("n-recall@k requires n <= k")
    if gt_ids.shape[1] < n:
        raise ValueError("ground truth has fewer than n entries per query")
    got = result_ids[:, :k]
    want = gt_ids[:, :n]
    hits = 0
    for row_got, row_want in zip(got, want):
        keep = row_want[row_want >= 0]
        hits += np.isin(keep, row_got[row_got >= 0]).sum()
    return hits / (result_ids.shape[0] * n)


def round_to(x: np.ndarray, storage: str) -> np.ndarray:
    """Round f32 to the 16-bit storage type (RNE) and back to f32.

    The fp16/bf16 configs run the reference on the same rounded values
    (SURVEY.md 8(d), cfg4/cfg5).
    """
    x = np.ascontiguousarray(x, dtype=np.float32)
    if storage == "fp16":
        return x.astype(np.float16).astype(np.float32)
    if storage == "bf16":
        bits = x.view(np.uint32).astype(np.uint64)
        # round-to-nearest-even on the top 16 bits; NaN kept quiet
        rnd = ((bits >> 16) & 1) + 0x7FFF
        out = ((bits + rnd) >> 16) << 16
        nan = np.isnan(x)
        out = out.astype(np.uint32)
        out[nan] = (x.view(np.uint32)[nan] | 0x00400000) & 0xFFFF0000
        return out.view(np.float32)
    return x


def direct_distances(q: np.ndarray, xb: np.ndarray, metric: str = METRIC_L2) -> np.ndarray:
    """core.py:184-188 pairwise_distances -> _kernels.pairwise (per-pair direct
    loops, _ckernels.pyx:49-57): L2 sum (q - x)^2, IP sum q x.  Accumulated in
    fp64 and rounded once to fp32 (the reference's fp32 loops differ by ulps)."""
    q64, x64 = q.astype(np.float64), xb.astype(np.float64)
    if metric == METRIC_IP:
        return (q64 @ x64.T).astype(np.float32)
    d = (q64 * q64).sum(1)[:, None] + (x64 * x64).sum(1)[None, :] - 2.0 * (q64 @ x64.T)
    # exact-enough for the small oracle cases; recompute the near-zero entries directly
    small = np.abs(d) < 1e-3 * ((q64 * q64).sum(1)[:, None] + (x64 * x64).sum(1)[None, :] + 1e-30)
    if small.any():
        ii, jj = np.nonzero(small)
        d[ii, jj] = ((q64[ii] - x64[jj]) ** 2).sum(1)
    return np.maximum(d, 0.0).astype(np.float32)


def flat_range_search(xb: np.ndarray, q: np.ndarray, radius: float, metric: str = METRIC_L2,
                      ids: np.ndarray | None = None):
    """flat.py:121-144: (lims, ids, distances) with every stored vector within
    the radius (<= for distances, >= for IP), best first, ties by smaller id."""
    ids_table = np.arange(xb.shape[0], dtype=np.int64) if ids is None else ids
    nq = q.shape[0]
    lims = np.zeros(nq + 1, dtype=np.int64)
    out_i, out_d = [], []
    desc = metric == METRIC_IP
    dmat = direct_distances(q, xb, metric) if xb.shape[0] else np.zeros((nq, 0), np.float32)
    for r in range(nq):
        row = dmat[r]
        mask = row >= radius if desc else row <= radius
        pos = np.nonzero(mask)[0]
        vals = row[pos]
        order = np.lexsort((ids_table[pos], -vals if desc else vals))
        out_i.append(ids_table[pos][order])
        out_d.append(vals[order])
        lims[r + 1] = len(pos)
    np.cumsum(lims, out=lims)
    cat_i = np.concatenate(out_i) if out_i else np.empty(0, np.int64)
    cat_d = np.concatenate(out_d) if out_d else np.empty(0, np.float32)
    return lims, cat_i, cat_d.astype(np.float32)


def positions(ids_table: np.ndarray, ids) -> np.ndarray:
    """flat.py:34-41: id -> position through ``{int(v): i for i, v in
    enumerate(ids)}`` (a repeated id maps to its LAST position); KeyError."""
    pos_of = {int(v): i for i, v in enumerate(ids_table)}
    try:
        return np.array([pos_of[int(v)] for v in np.atleast_1d(ids)], dtype=np.int64)
    except KeyError as exc:
        raise KeyError(f"unknown id {exc.args[0]}") from None


def remove_ids(xb: np.ndarray, ids_table: np.ndarray, kill):
    """flat.py:46-56: drop every row whose id is in ``kill``, keep order.
    Returns (vectors, ids, removed)."""
    mask = np.isin(ids_table, np.asarray(kill, dtype=np.int64))
    return xb[~mask], ids_table[~mask], int(mask.sum())


def refine_rerank(xb: np.ndarray, ids_table: np.ndarray, q: np.ndarray, cand: np.ndarray, k: int,
                  metric: str = METRIC_L2):
    """core.py:368-394 given the fast index's shortlist ``cand`` (nq, L):
    per query drop -1, reconstruct the candidates from the exact index
    (flat.py:43-44), direct distances (pairwise_distances), keep the first k
    by (value best first, id) with Python's stable sort, pad -1 / +-inf."""
    nq = q.shape[0]
    desc = metric == METRIC_IP
    out_ids = np.full((nq, k), -1, dtype=np.int64)
    out_dist = np.full((nq, k), -np.inf if desc else np.inf, dtype=np.float32)
    for i in range(nq):
        c = cand[i][cand[i] >= 0]
        if len(c) == 0:
            continue
        vecs = xb[positions(ids_table, c)]
        dists = direct_distances(q[i:i + 1], vecs, metric)[0]
        order = sorted(range(len(c)), key=lambda j: (-dists[j] if desc else dists[j], c[j]))[:k]
        for slot, j in enumerate(order):
            out_ids[i, slot] = c[j]
            out_dist[i, slot] = dists[j]
    return out_ids, out_dist
