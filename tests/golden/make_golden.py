"""Generate the golden parity vectors by running the REAL reference.

Run in the build container only (``/root/reference`` does not exist on the GPU
box)::

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports annkit read-only from ``/root/reference/pkg/src`` and, for every
case in ``cases.py``, stores:

* ``<case>/blas_ids, blas_dist``   -- ``annkit.flat.flat_search_blas``
  (flat.py:94-118, the hot path the GPU replaces);
* ``<case>/search_ids, search_dist`` -- ``FlatIndex.search`` (core.py:145-150,
  with the reference's own nq<20 direct-path dispatch, flat.py:58-62);
* ``<case>/digest`` -- sha256 prefix of the generated inputs, so the tests can
  prove they regenerated the same inputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import annkit  # noqa: E402
from annkit import flat as ref_flat  # noqa: E402
from annkit.core import METRIC_IP, METRIC_L2  # noqa: E402

from cases import CASES, digest, make_inputs  # noqa: E402


def main() -> None:
    out = {}
    for name in CASES:
        xb, q, k, metric, storage, ids = make_inputs(name)
        m = METRIC_L2 if metric == "l2" else METRIC_IP
        index = ref_flat.FlatIndex(xb.shape[1], m)
        if xb.shape[0]:
            if ids is None:
                index.add(xb)
            else:
                index.add_with_ids(xb, ids)
        blas = ref_flat.flat_search_blas(index, q, k)
        srch = index.search(q, k)
        out[f"{name}/blas_ids"] = blas.ids
        out[f"{name}/blas_dist"] = blas.distances
        out[f"{name}/search_ids"] = srch.ids
        out[f"{name}/search_dist"] = srch.distances
        out[f"{name}/digest"] = np.array(digest(xb, q))
        print(f"{name:20s} nb={xb.shape[0]:6d} nq={q.shape[0]:5d} d={xb.shape[1]:4d} k={k:5d} "
              f"{metric} {storage}")
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, "annkit COMPILED =", annkit.COMPILED)


if __name__ == "__main__":
    main()
