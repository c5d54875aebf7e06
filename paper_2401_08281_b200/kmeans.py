"""Consumers of the flat path: the IVF coarse quantizer and the
k-means assignment step, both on the GPU flat search.

* ``coarse_quantizer`` / ``assign_vectors`` / ``probe_lists`` mirror
  ``annkit.ivf.IvfIndex`` (ivf.py:198-203 build, :213-214 ``_assign_vectors``,
  :324-326 ``probe_lists``).  The reference's coarse quantizer *is* a
  ``FlatIndex``, so ``IvfIndex(d, nlist, coarse=FlatIndex(d, METRIC_L2))``
  plugs this package in directly; these helpers restate the
  two calls the IVF makes on it.
* ``kmeans_assign`` replaces ``annkit.quantize._assign`` (quantize.py:38-62),
  which the reference computes in fp64 against fp64 centroids: the fp32
  (3xTF32) GPU flat search over the fp32-rounded centroids yields a shortlist
  per row, ``fk_kmeans_rescore`` re-evaluates the shortlist exactly in fp64
  and certifies it (gap between the shortlist's best and last fp32 distance
  above the fp32 error bound); uncertified rows are rescored over every
  centroid.  No CPU fallback: every step is a CUDA kernel.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _native as N
from .core import METRIC_IP, METRIC_L2, Metric, MetricKind, is_torch
from .flat import FlatIndex, _stream_of

# fp32 error bound of a 3xTF32 distance over fp32-rounded centroids, relative
# to |x|^2 + max|c|^2 (~2^-21 of GEMM rounding + 2^-23 of centroid rounding,
# with a wide safety factor)
_MARGIN = 2.0 ** -16


# One reusable shortlist index per (device, d, metric): k-means calls the
# assignment every iteration, and creating + freeing an index per call costs
# more than the search (allocation; cudaFree synchronizes the device).
_SHORTLIST: dict = {}
_SHORTLIST_LOCK = threading.Lock()


def _shortlist_index(device: int, d: int, by_ip: bool):
    key = (device, d, bool(by_ip))
    with _SHORTLIST_LOCK:
        ent = _SHORTLIST.get(key)
        if ent is None:
            ent = (FlatIndex(d, METRIC_IP if by_ip else METRIC_L2, storage="fp32", device=device), threading.Lock())
            _SHORTLIST[key] = ent
    return ent


def coarse_quantizer(d: int, spherical: bool = False, storage: str = "fp32", device: int | None = None) -> FlatIndex:
    """ivf.py:198-203: spherical clustering routes by inner product, the
    default is L2 assignment regardless of the IVF's own metric."""
    return FlatIndex(d, METRIC_IP if spherical else METRIC_L2, storage=storage, device=device)


def assign_vectors(coarse: FlatIndex, x) -> np.ndarray:
    """ivf.py:213-214: nearest coarse centroid per row."""
    ids = coarse.search(x, 1).ids
    return ids[:, 0]


def probe_lists(coarse: FlatIndex, q, nprobe: int) -> np.ndarray:
    """ivf.py:324-326: the nprobe coarse cells to visit, best first."""
    return coarse.search(q, nprobe).ids


def kmeans_assign(x, centroids, by_ip: bool = False, shortlist: int = 8, device: int | None = None):
    """quantize.py:38-62: (assignment int64, squared-L2 error float64).

    ``x``: (n, d) float32 (the reference's ``x64`` is fp32 data widened);
    ``centroids``: (k, d) float64.  Returns numpy arrays for numpy input and
    CUDA tensors for CUDA input."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    cuda_in = is_torch(x) and x.is_cuda
    xt = torch.as_tensor(x, dtype=torch.float32).to(dev).contiguous()
    ct = torch.as_tensor(centroids, dtype=torch.float64).to(dev).contiguous()
    if xt.ndim != 2 or ct.ndim != 2 or xt.shape[1] != ct.shape[1]:
        raise ValueError("x must be (n, d) and centroids (k, d)")
    n, d = xt.shape
    nc = ct.shape[0]
    if nc < 1:
        raise ValueError("need at least one centroid")
    cnorm = torch.einsum("kd,kd->k", ct, ct).contiguous()  # quantize.py:47 (fp64)
    cmax = float(cnorm.max().item())
    assign = torch.empty(n, dtype=torch.int64, device=dev)
    err = torch.empty(n, dtype=torch.float64, device=dev)
    stream = _stream_of(dev.index)
    kc = min(shortlist, nc)
    if kc < nc:
        idx, lock = _shortlist_index(dev.index, d, by_ip)
        with lock:  # reset + add + search of one caller at a time (stream-ordered on the device)
            idx.reset()
            idx.add(ct.float())
            res = idx.search(xt, kc)
        cand = res.ids.contiguous()
        approx = res.distances.contiguous()
        unc = torch.empty(n, dtype=torch.int32, device=dev)
        N.check(N.lib().fk_kmeans_rescore(xt.data_ptr(), n, d, ct.data_ptr(), cnorm.data_ptr(), nc, cand.data_ptr(),
                                          kc, int(by_ip), approx.data_ptr(), _MARGIN, cmax, assign.data_ptr(),
                                          err.data_ptr(), unc.data_ptr(), stream))
        rows = torch.nonzero(unc, as_tuple=False).flatten()
    else:
        rows = torch.arange(n, device=dev)
    if rows.numel():  # exact fp64 over every centroid for the uncertified rows
        xs = xt.index_select(0, rows).contiguous()
        a2 = torch.empty(rows.numel(), dtype=torch.int64, device=dev)
        e2 = torch.empty(rows.numel(), dtype=torch.float64, device=dev)
        N.check(N.lib().fk_kmeans_rescore(xs.data_ptr(), rows.numel(), d, ct.data_ptr(), cnorm.data_ptr(), nc, None,
                                          nc, int(by_ip), None, 0.0, cmax, a2.data_ptr(), e2.data_ptr(), None,
                                          stream))
        assign.index_copy_(0, rows, a2)
        err.index_copy_(0, rows, e2)
    if cuda_in:
        return assign, err
    return assign.cpu().numpy(), err.cpu().numpy()


__all__ = ["coarse_quantizer", "assign_vectors", "probe_lists", "kmeans_assign", "Metric", "MetricKind"]
