"""Seeded input generators for the golden parity cases.

Shared by ``make_golden.py`` (which runs the real reference, in the build
container only) and the tests (which regenerate the same inputs from the
seeds and compare against the committed outputs).  Inputs follow SURVEY.md
8(d): ``np.random.default_rng(seed).standard_normal(shape, dtype=float32)``.
"""

from __future__ import annotations

import hashlib

import numpy as np


def _gauss(seed, shape):
    return np.random.default_rng(seed).standard_normal(shape, dtype=np.float32)


def _round(x, storage):
    # same RNE rounding as oracle.flat_oracle.round_to, restated here so the
    # generator has no product/oracle dependency
    if storage == "fp16":
        return x.astype(np.float16).astype(np.float32)
    if storage == "bf16":
        bits = x.view(np.uint32).astype(np.uint64)
        rnd = ((bits >> 16) & 1) + 0x7FFF
        return ((((bits + rnd) >> 16) << 16).astype(np.uint32)).view(np.float32)
    return x


def make_inputs(name: str):
    """Return (xb, q, k, metric, storage, ids_or_None) for a named case."""
    c = CASES[name]
    kind = c["kind"]
    if kind == "literal":
        xb = np.array(c["xb"], dtype=np.float32)
        q = np.array(c["q"], dtype=np.float32).reshape(-1, xb.shape[1] if xb.size else c["d"])
        if xb.size == 0:
            xb = xb.reshape(0, c["d"])
    elif kind == "gauss":
        xb = _gauss(c["seed_b"], (c["nb"], c["d"]))
        q = _gauss(c["seed_q"], (c["nq"], c["d"]))
        if c.get("normalize"):
            xb /= np.linalg.norm(xb, axis=1, keepdims=True)
    elif kind == "selfq":
        xb = _gauss(c["seed_b"], (c["nb"], c["d"]))
        q = xb[c["rows"]].copy()
    elif kind == "ints":
        rng = np.random.default_rng(c["seed_b"])
        xb = rng.integers(0, c["hi"], size=(c["nb"], c["d"])).astype(np.float32)
        q = np.random.default_rng(c["seed_q"]).integers(0, c["hi"], size=(c["nq"], c["d"])).astype(np.float32)
    else:
        raise KeyError(kind)
    storage = c.get("storage", "fp32")
    xb = _round(np.ascontiguousarray(xb), storage)
    q = _round(np.ascontiguousarray(q), storage)
    ids = np.array(c["ids"], dtype=np.int64) if "ids" in c else None
    return xb, q, c["k"], c["metric"], storage, ids


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


CASES = {
    # test_flat.py:31-35 -- nearest of two, dist 0.01
    "nearest_of_two": dict(kind="literal", xb=[[0, 0], [1, 0]], q=[[0.1, 0.0]], k=1, metric="l2"),
    # test_flat.py:107-111 -- BLAS identity expansion, dist 2.0
    "identity_expansion": dict(kind="literal", xb=[[0, 1]], q=[[1, 0]], k=1, metric="l2"),
    # test_flat.py:88-94 -- add_with_ids then search
    "add_with_ids": dict(kind="literal", xb=[[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11]],
                         q=[[8, 9, 10, 11]], k=1, metric="l2", ids=[10, 20, 30]),
    # test_flat.py:77-81 -- empty index -> sentinels
    "empty_index": dict(kind="literal", xb=[], d=4, q=[[0, 0, 0, 0], [0, 0, 0, 0]], k=3, metric="l2"),
    # test_flat.py:37-43 / 113-120 -- self queries (normalised rows)
    "self_query": dict(kind="selfq", seed_b=4, nb=30, d=16, rows=list(range(30)), k=1, metric="l2"),
    # test_flat.py:45-58 shape, L2 and IP
    "naive_l2": dict(kind="gauss", seed_b=42, seed_q=43, nb=200, nq=10, d=8, k=10, metric="l2"),
    "naive_ip": dict(kind="gauss", seed_b=42, seed_q=43, nb=200, nq=10, d=8, k=10, metric="ip"),
    # test_flat.py:60-66 -- k == ntotal is a permutation
    "k_eq_ntotal": dict(kind="gauss", seed_b=1, seed_q=2, nb=64, nq=5, d=4, k=64, metric="l2"),
    # k > ntotal pads -1 / +inf (core.py:232-235)
    "k_gt_ntotal_l2": dict(kind="gauss", seed_b=5, seed_q=6, nb=5, nq=3, d=4, k=8, metric="l2"),
    "k_gt_ntotal_ip": dict(kind="gauss", seed_b=5, seed_q=6, nb=5, nq=3, d=4, k=8, metric="ip"),
    # test_flat.py:122-132 shape
    "blas_1000x32": dict(kind="gauss", seed_b=5, seed_q=7, nb=1000, nq=64, d=32, k=10, metric="l2"),
    # cfg1-shaped (SIFT d=128), reduced nb so the reference runs in seconds
    "cfg1_small_l2": dict(kind="gauss", seed_b=0, seed_q=1, nb=20000, nq=300, d=128, k=10, metric="l2"),
    "cfg1_small_ip": dict(kind="gauss", seed_b=0, seed_q=1, nb=20000, nq=300, d=128, k=10, metric="ip"),
    # ragged sizes: nb, nq, d not multiples of any tile
    "ragged": dict(kind="gauss", seed_b=11, seed_q=12, nb=1237, nq=131, d=37, k=7, metric="l2"),
    "ragged_ip": dict(kind="gauss", seed_b=11, seed_q=12, nb=1237, nq=131, d=37, k=32, metric="ip"),
    # exact-tie stress: small-integer data (SURVEY 8(d) tie-stress variant)
    "int_ties_l2": dict(kind="ints", seed_b=21, seed_q=22, nb=3000, nq=100, d=16, hi=4, k=20, metric="l2"),
    "int_ties_ip": dict(kind="ints", seed_b=21, seed_q=22, nb=3000, nq=100, d=16, hi=4, k=20, metric="ip"),
    # large k (cfg3 shape, reduced)
    "large_k_1024": dict(kind="gauss", seed_b=0, seed_q=1, nb=8000, nq=64, d=128, k=1024, metric="l2"),
    "large_k_100_ip": dict(kind="gauss", seed_b=3, seed_q=4, nb=6000, nq=64, d=64, k=100, metric="ip"),
    # fp16 storage, IP, Contriever-shaped d=768 (cfg4, reduced)
    "fp16_ip_768": dict(kind="gauss", seed_b=0, seed_q=1, nb=4000, nq=40, d=768, k=100, metric="ip",
                        storage="fp16"),
    # bf16 storage, L2, Deep1B-shaped d=96 (cfg5, reduced)
    "bf16_l2_96": dict(kind="gauss", seed_b=0, seed_q=1, nb=5000, nq=50, d=96, k=10, metric="l2",
                       storage="bf16"),
}
