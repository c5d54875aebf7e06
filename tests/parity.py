"""Tie-aware comparison of a k-NN result against the reference/oracle answer.

Rules (BASELINE.json north_star):
  1. distances agree to ``rel_dist`` relative (plus ``abs_dist`` for near-zero);
  2. per position the ids are equal, or the two positions' reference distances
     tie within ``rel_tie`` relative (order among near-ties is free);
  3. id sets are equal except ids whose reference distance is within
     ``rel_tie`` of the reference k-th distance (boundary near-ties);
  4. tie-aware recall@k == 1.0 (recall over the non-boundary-tie ids).
Returns a dict of counts so callers can assert and report.
"""

from __future__ import annotations

import numpy as np


def _close(a, b, rel, absol):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    with np.errstate(invalid="ignore"):
        return both_inf | (np.abs(a - b) <= rel * np.abs(b) + absol)


def compare(got_ids, got_dist, ref_ids, ref_dist, rel_dist=1e-4, abs_dist=1e-4, rel_tie=1e-5, abs_tie=1e-5):
    got_ids = np.asarray(got_ids)
    ref_ids = np.asarray(ref_ids)
    got_dist = np.asarray(got_dist, dtype=np.float64)
    ref_dist = np.asarray(ref_dist, dtype=np.float64)
    assert got_ids.shape == ref_ids.shape, (got_ids.shape, ref_ids.shape)
    nq, k = ref_ids.shape
    stats = dict(rows=nq, dist_bad=0, pos_bad=0, set_bad=0, tie_swaps=0, boundary_ties=0,
                 strict_recall=0.0, tie_recall=0.0)
    hits = strict_hits = want_total = 0
    for i in range(nq):
        ok = _close(got_dist[i], ref_dist[i], rel_dist, abs_dist)
        stats["dist_bad"] += int((~ok).sum())
        for j in range(k):
            if got_ids[i, j] != ref_ids[i, j]:
                if _close(got_dist[i, j], ref_dist[i, j], rel_tie, abs_tie):
                    stats["tie_swaps"] += 1
                else:
                    stats["pos_bad"] += 1
        valid = ref_ids[i] >= 0
        if valid.any():
            kth = ref_dist[i][valid][-1]
            near_kth = _close(ref_dist[i], np.full(k, kth), rel_tie, abs_tie) & valid
        else:
            near_kth = np.zeros(k, dtype=bool)
        core = set(ref_ids[i][valid & ~near_kth].tolist())
        got = set(got_ids[i][got_ids[i] >= 0].tolist())
        missing = core - got
        stats["set_bad"] += len(missing)
        stats["boundary_ties"] += int(near_kth.sum())
        extra = got - set(ref_ids[i][valid].tolist())
        # an extra id is legitimate only if it replaced a boundary near-tie
        if len(extra) > int(near_kth.sum()):
            stats["set_bad"] += len(extra) - int(near_kth.sum())
        hits += len(core & got)
        want_total += len(core)
        strict_hits += len(set(ref_ids[i][valid].tolist()) & got)
    nvalid = int((ref_ids >= 0).sum())
    stats["strict_recall"] = strict_hits / nvalid if nvalid else 1.0
    stats["tie_recall"] = hits / want_total if want_total else 1.0
    return stats


def assert_parity(got_ids, got_dist, ref_ids, ref_dist, **kw):
    s = compare(got_ids, got_dist, ref_ids, ref_dist, **kw)
    assert s["dist_bad"] == 0, s
    assert s["pos_bad"] == 0, s
    assert s["set_bad"] == 0, s
    assert s["tie_recall"] == 1.0, s
    return s


def assert_range_parity(got, want, radius, metric, rel_tie=1e-5, abs_tie=1e-6, rel_dist=1e-4, abs_dist=1e-5,
                        exact=False):
    """Range-search parity (flat.py:121-144 semantics): per query the id sets
    agree except ids whose distance is within ``rel_tie`` of the radius
    (boundary near-ties), common ids agree on distance, and the returned list
    is best first with ties by smaller id.  ``exact``: identical CSR output
    (integer-valued data, where every distance is exact)."""
    (gl, gi, gd), (wl, wi, wd) = [tuple(np.asarray(a.cpu() if hasattr(a, "cpu") else a) for a in t) for t in (got, want)]
    assert gl.shape == wl.shape, (gl.shape, wl.shape)
    if exact:
        assert np.array_equal(gl, wl) and np.array_equal(gi, wi)
        assert np.array_equal(gd.astype(np.float32), wd.astype(np.float32))
        return
    desc = metric == "ip"
    rad = float(radius)
    for r in range(len(gl) - 1):
        g_ids, g_d = gi[gl[r]:gl[r + 1]], gd[gl[r]:gl[r + 1]].astype(np.float64)
        w_ids, w_d = wi[wl[r]:wl[r + 1]], wd[wl[r]:wl[r + 1]].astype(np.float64)
        gm, wm = dict(zip(g_ids.tolist(), g_d)), dict(zip(w_ids.tolist(), w_d))
        near = lambda v: np.isfinite(rad) and abs(v - rad) <= rel_tie * max(abs(rad), abs(v)) + abs_tie  # noqa: E731
        for i in set(wm) - set(gm):
            assert near(wm[i]), f"row {r}: id {i} (d={wm[i]!r}) missing, radius {rad!r}"
        for i in set(gm) - set(wm):
            assert near(gm[i]), f"row {r}: extra id {i} (d={gm[i]!r}), radius {rad!r}"
        for i in set(gm) & set(wm):
            assert abs(gm[i] - wm[i]) <= rel_dist * abs(wm[i]) + abs_dist, (r, i, gm[i], wm[i])
        # best first, ties by smaller id, on our own values
        key = -g_d if desc else g_d
        for a in range(len(g_ids) - 1):
            assert key[a] < key[a + 1] or (key[a] == key[a + 1] and g_ids[a] < g_ids[a + 1]), (r, a)
