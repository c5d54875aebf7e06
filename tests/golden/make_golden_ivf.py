"""Golden vectors for the SURVEY 8(f) consumers of the flat path, produced by
running the REAL reference (build container only; /root/reference is absent
on the GPU box)::

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_ivf.py

* IVF coarse quantizer (ivf.py:198-203 train, :213-214 ``_assign_vectors``,
  :324-326 ``probe_lists``): an ``IvfIndex`` (IVF-Flat) is trained with the
  reference k-means; its centroids, the coarse assignment of the added
  vectors and the nprobe probe lists of the queries are stored, for L2 and for
  the spherical (inner-product routed) variant.
* k-means assignment (quantize.py:38-62 ``_assign``, fp64): assignment and
  squared-L2 error for fp64 centroids, L2 and by-inner-product.

Inputs are regenerated from the seed by the tests (``ivf_inputs``); only a
digest of them is stored.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

D, NLIST, NPROBE, N_ADD, N_Q = 32, 64, 8, 20000, 300


def ivf_inputs():
    """(xt, xa, q, c64): training/add/query vectors and fp64 centroids."""
    rng = np.random.default_rng(31)
    xt = rng.standard_normal((8000, D), dtype=np.float32)
    xa = rng.standard_normal((N_ADD, D), dtype=np.float32)
    q = rng.standard_normal((N_Q, D), dtype=np.float32)
    c64 = rng.standard_normal((NLIST, D)) * 0.7
    return xt, xa, q, c64


def digest(*arrays) -> str:
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def main() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    from annkit import quantize as ref_quantize
    from annkit.core import METRIC_L2
    from annkit.ivf import IvfIndex

    xt, xa, q, c64 = ivf_inputs()
    out = {"digest": np.array(digest(xt, xa, q))}
    for tag, spherical in (("l2", False), ("sph", True)):
        ivf = IvfIndex(D, NLIST, metric=METRIC_L2, nprobe=NPROBE, spherical=spherical, kmeans_niter=8, seed=3)
        ivf.train(xt)
        ivf.add(xa)
        out[f"{tag}/centroids"] = ivf.centroids
        out[f"{tag}/assign"] = ivf._assign_vectors(xa)
        out[f"{tag}/probes"] = ivf.probe_lists(q, NPROBE)
    # k-means assignment in fp64 against fp64 centroids (not fp32-representable)
    x64 = xa[:5000].astype(np.float64)
    for tag, by_ip in (("l2", False), ("ip", True)):
        a, err = ref_quantize._assign(x64, c64, by_ip=by_ip)
        out[f"km_{tag}/assign"] = a
        out[f"km_{tag}/err"] = err
    path = os.path.join(HERE, "golden_ivf.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
