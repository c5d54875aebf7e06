"""GPU FlatIndex: drop-in for the reference ``annkit.flat.FlatIndex`` (flat.py:14-65).

Every search runs the sm_100a path through the C ABI (``include/flatknn.h``):
query prep kernel -> fused tcgen05 GEMM + top-k kernel -> merge kernel.
There is no CPU fallback.  The reference's ``nq < config.blas_threshold``
dispatch (flat.py:58-62) is kept: small batches take a GPU direct path
(exact per-pair distances, flat.py:76-91), so e.g. a self-distance is
exactly 0.0 as test_flat.py:37-43 asserts.

Storage modes:
  "fp32" -- fp32 vectors (stored as an exact tf32 hi/lo split), searched with
  one tf32 tensor-core pass + certified exact fp32 rescoring (k <= 16 over
  >= 256k rows) or 3xTF32 -- fp32-faithful either way;
  "fp16" / "bf16" -- vectors (and queries) rounded RNE to 16 bits, single
  tensor-core pass; norms are computed from the rounded values, so results
  equal the reference run on the same rounded inputs.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from . import config
from .core import (METRIC_IP, METRIC_L2, Index, Metric, RangeResult, SearchResult, as_vectors, is_torch,
                   metric_value)

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

_STORAGE = {"fp32": N.FK_F32, "float32": N.FK_F32, "fp16": N.FK_F16, "float16": N.FK_F16,
            "bf16": N.FK_BF16, "bfloat16": N.FK_BF16}


def _dtype_code(x) -> int:
    if is_torch(x):
        return {torch.float32: N.FK_F32, torch.float16: N.FK_F16, torch.bfloat16: N.FK_BF16}[x.dtype]
    return {np.dtype(np.float32): N.FK_F32, np.dtype(np.float16): N.FK_F16}[x.dtype]


def _ptr(x) -> int:
    return x.data_ptr() if is_torch(x) else x.ctypes.data


def _host_out(shape, dtype):
    """Output array for host results: pinned (torch caching host allocator)
    when CUDA is usable and the array is large (>= 8 MB), else plain numpy.
    Either way a fresh numpy array owned by the caller."""
    n = int(np.prod(shape))
    # (a fresh pinned block costs ~0.5 ms: only worth it for large results,
    # e.g. k = 1024 -- 82 MB of ids -- where pageable copies run at ~6 GB/s)
    if torch is not None and n * np.dtype(dtype).itemsize >= (8 << 20) and torch.cuda.is_available():
        tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.int64): torch.int64}[np.dtype(dtype)]
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    return np.empty(shape, dtype=dtype)


def _stream_of(device: int) -> int:
    if torch is None or not torch.cuda.is_available():
        return 0
    return torch.cuda.current_stream(device).cuda_stream


class FlatIndex(Index):
    """Exact k-NN over raw vectors stored in HBM (reference flat.py:14-26).

    Parameters mirror the reference (``d``, ``metric``) plus the B200 storage
    mode and the CUDA device ordinal.
    """

    # exhaustive index: annkit's IVF search charges nlist coarse distances per
    # query for a flat coarse quantizer (ivf.py:401)
    is_flat = True

    def __init__(self, d: int, metric: Metric = METRIC_L2, storage: str = "fp32", device: int | None = None):
        super().__init__(d, metric)
        mv = metric_value(metric)
        if mv not in ("l2", "ip"):
            raise NotImplementedError(
                f"metric {mv!r}: the GPU flat index implements L2 and inner product "
                "(the reference's BLAS path, flat.py:94-118)")
        if storage not in _STORAGE:
            raise ValueError(f"storage must be one of fp32/fp16/bf16, got {storage!r}")
        self.storage = storage
        self._mcode = N.FK_METRIC_L2 if mv == "l2" else N.FK_METRIC_IP
        if device is None:
            device = torch.cuda.current_device() if (torch is not None and torch.cuda.is_available()) else 0
        self.device = int(device)
        L = N.lib()
        h = ctypes.c_void_p()
        N.check(L.fk_create(self.device, self.d, self._mcode, _STORAGE[storage], ctypes.byref(h)))
        self._h = h
        self._blas_threshold = 20  # the native default (config.py:9)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().fk_destroy(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------------ storage
    def _add(self, x, ids, sequential: bool) -> None:
        """flat.py:28-32: append vectors, ids and norms (on device)."""
        if x.shape[0] == 0:
            return
        dev = is_torch(x) and x.is_cuda
        if dev and x.device.index != self.device:
            x = x.to(f"cuda:{self.device}")
        if not dev and is_torch(x):
            x = x.contiguous()
        ids_arg = None
        keep = None
        if not sequential:
            if dev:
                t = ids if is_torch(ids) else torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int64))
                keep = t.to(device=x.device, dtype=torch.int64).contiguous()
            else:
                keep = np.ascontiguousarray(ids.cpu().numpy() if is_torch(ids) else ids, dtype=np.int64)
            ids_arg = _ptr(keep)
        stream = _stream_of(self.device) if dev else 0
        N.check(N.lib().fk_add(self._h, _ptr(x), x.shape[0], _dtype_code(x), ids_arg, int(dev), stream))

    def reset(self) -> None:
        """Drop every vector (Faiss ``Index::reset``; not in the reference)."""
        N.check(N.lib().fk_reset(self._h))
        self.ntotal = 0

    @property
    def ids(self) -> np.ndarray:
        """Stored ids in storage order (the reference's ``FlatIndex.ids``)."""
        out = np.empty(self.ntotal, dtype=np.int64)
        if self.ntotal:
            N.check(N.lib().fk_get_ids(self._h, out.ctypes.data))
        return out

    @property
    def vectors(self) -> np.ndarray:
        """Stored vectors as float32 (the reference's ``FlatIndex.vectors``)."""
        pos = np.arange(self.ntotal, dtype=np.int64)
        return self._reconstruct_positions(pos)

    def _positions_dev(self, ids):
        """flat.py:34-41 on the device: id -> storage position through the
        sorted id table (a duplicated id maps to its last position, like the
        reference's dict); KeyError on unknown ids.  Returns a CUDA tensor."""
        dev = f"cuda:{self.device}"
        t = ids if is_torch(ids) else torch.from_numpy(np.ascontiguousarray(np.atleast_1d(np.asarray(ids)),
                                                                            dtype=np.int64))
        t = t.reshape(-1).to(device=dev, dtype=torch.int64).contiguous()
        pos = torch.empty_like(t)
        if t.numel():
            N.check(N.lib().fk_positions(self._h, _ptr(t), t.numel(), _ptr(pos), 1, _stream_of(self.device)))
        return pos

    def _positions(self, ids) -> np.ndarray:
        """flat.py:34-41: id -> storage position, KeyError on unknown ids."""
        return self._positions_dev(ids).cpu().numpy()

    def _reconstruct_positions(self, pos: np.ndarray) -> np.ndarray:
        out = np.empty((len(pos), self.d), dtype=np.float32)
        if len(pos):
            N.check(N.lib().fk_reconstruct(self._h, np.ascontiguousarray(pos).ctypes.data, len(pos),
                                           out.ctypes.data, 0, 0))
        return out

    def reconstruct_batch(self, ids):
        """flat.py:43-44 (exact: fp32 storage keeps hi+lo == x).  CUDA ids
        give a CUDA tensor; anything else a numpy array.  The id lookup and
        the gather both run on the device."""
        pos = self._positions_dev(ids)
        out = torch.empty((pos.numel(), self.d), dtype=torch.float32, device=pos.device)
        if pos.numel():
            N.check(N.lib().fk_reconstruct(self._h, _ptr(pos), pos.numel(), _ptr(out), 1,
                                           _stream_of(self.device)))
        return out if (is_torch(ids) and ids.is_cuda) else out.cpu().numpy()

    def remove_ids(self, ids) -> int:
        """flat.py:46-56: drop matching ids, keep storage order (mask and
        compaction on the device)."""
        removed = ctypes.c_int64(0)
        if is_torch(ids) and ids.is_cuda:
            t = ids.reshape(-1).to(device=f"cuda:{self.device}", dtype=torch.int64).contiguous()
            N.check(N.lib().fk_remove_ids(self._h, _ptr(t), t.numel(), 1, ctypes.byref(removed),
                                          _stream_of(self.device)))
        else:
            if is_torch(ids):
                ids = ids.cpu().numpy()
            arr = np.ascontiguousarray(np.atleast_1d(np.asarray(ids, dtype=np.int64)))
            N.check(N.lib().fk_remove_ids(self._h, arr.ctypes.data, arr.size, 0, ctypes.byref(removed), 0))
        self.ntotal -= int(removed.value)
        return int(removed.value)

    # ------------------------------------------------------------------ search
    def _search(self, q, k: int, with_positions: bool = False):
        """flat.py:58-62 on the GPU: batches of >= ``config.blas_threshold``
        queries run the fused GEMM + top-k path (flat_search_blas, 94-118),
        smaller ones the direct per-pair path (flat_search, 76-91).  Returns
        SearchResult (+ storage positions)."""
        nq = q.shape[0]
        L = N.lib()
        bt = int(config.blas_threshold)
        if bt != self._blas_threshold:
            N.check(L.fk_set_option(self._h, N.FK_OPT_BLAS_THRESHOLD, bt))
            self._blas_threshold = bt
        if is_torch(q) and q.is_cuda:
            if q.device.index != self.device:
                q = q.to(f"cuda:{self.device}")
            dev = q.device
            D = torch.empty((nq, k), dtype=torch.float32, device=dev)
            I = torch.empty((nq, k), dtype=torch.int64, device=dev)
            P = torch.empty((nq, k), dtype=torch.int64, device=dev) if with_positions else None
            N.check(L.fk_search(self._h, _ptr(q), nq, _dtype_code(q), k, _ptr(D), _ptr(I),
                                _ptr(P) if P is not None else None, 1, _stream_of(self.device)))
        else:
            if is_torch(q):
                q = q.contiguous()
            # large results land in page-locked host memory so the D2H copy
            # runs at DMA speed; the numpy arrays keep their block alive
            D = _host_out((nq, k), np.float32)
            I = _host_out((nq, k), np.int64)
            P = _host_out((nq, k), np.int64) if with_positions else None
            N.check(L.fk_search(self._h, _ptr(q), nq, _dtype_code(q), k, D.ctypes.data, I.ctypes.data,
                                P.ctypes.data if P is not None else None, 0, 0))
        res = SearchResult(I, D, k)
        return (res, P) if with_positions else res

    def _range_search(self, q, radius: float) -> RangeResult:
        """flat.py:121-144 on the GPU: direct distances (<= radius; >= for
        IP), each query's list best first, ties by smaller id (flat.py:137).
        The entries come back in a per-call native result object, so
        concurrent range searches on one index cannot mix results."""
        nq = q.shape[0]
        L = N.lib()
        total = ctypes.c_int64(0)
        res = ctypes.c_void_p()
        try:
            if is_torch(q) and q.is_cuda:
                if q.device.index != self.device:
                    q = q.to(f"cuda:{self.device}")
                stream = _stream_of(self.device)
                lims = torch.empty(nq + 1, dtype=torch.int64, device=q.device)
                N.check(L.fk_range_search(self._h, _ptr(q), nq, _dtype_code(q), float(radius), _ptr(lims),
                                          ctypes.byref(total), ctypes.byref(res), 1, stream))
                ids = torch.empty(total.value, dtype=torch.int64, device=q.device)
                dist = torch.empty(total.value, dtype=torch.float32, device=q.device)
                N.check(L.fk_range_fetch(res, _ptr(ids), _ptr(dist), total.value, 1, stream))
            else:
                if is_torch(q):
                    q = q.contiguous()
                lims = np.empty(nq + 1, dtype=np.int64)
                N.check(L.fk_range_search(self._h, _ptr(q), nq, _dtype_code(q), float(radius), lims.ctypes.data,
                                          ctypes.byref(total), ctypes.byref(res), 0, 0))
                ids = np.empty(total.value, dtype=np.int64)
                dist = np.empty(total.value, dtype=np.float32)
                N.check(L.fk_range_fetch(res, ids.ctypes.data, dist.ctypes.data, total.value, 0, 0))
        finally:
            if res.value:
                L.fk_range_free(res)
        return RangeResult(lims, ids, dist, float(radius))

    def set_plan_rows(self, rows: int) -> None:
        """Choose the fp32 algorithm as for a database of ``rows`` rows (a
        shard of a row-sharded index passes the global count; 0 = own)."""
        N.check(N.lib().fk_set_option(self._h, N.FK_OPT_PLAN_ROWS, int(rows)))

    def search_with_positions(self, q, k: int):
        """Search returning (SearchResult, storage positions) -- the sharded
        index orders cross-shard ties by global position."""
        if k < 1:
            raise ValueError("k must be >= 1")
        return self._search(as_vectors(q, self.d), int(k), with_positions=True)

    # ------------------------------------------------------------------ instrumentation
    def set_profiling(self, on: bool, reserve: int = 64) -> None:
        """Record CUDA events around the kernels of each search; the events of
        ``reserve`` searches are created now (none inside a timed loop)."""
        N.check(N.lib().fk_set_profiling(self._h, max(1, int(reserve)) if on else 0))

    def kernel_times(self):
        """(prep_ms, fused_ms, merge_ms), launches of the last search."""
        ms = (ctypes.c_float * 3)()
        nl = ctypes.c_int(0)
        N.check(N.lib().fk_kernel_times(self._h, ms, ctypes.byref(nl)))
        return (ms[0], ms[1], ms[2]), nl.value

    def last_plan(self) -> dict:
        v = (ctypes.c_int * 12)()  # FK_PLAN_INTS
        N.check(N.lib().fk_last_plan(self._h, v))
        keys = ("grid", "S", "chunk_tiles", "units", "stages", "a_mode", "smem", "kq", "acc_stages", "epi", "bn", "kmode")
        return dict(zip(keys, list(v)))


def refine_search(fast: Index, exact: FlatIndex, q, k: int, shortlist: int) -> SearchResult:
    """Two-stage search (reference core.py:368-394): a ``shortlist`` from the
    fast index, re-ranked with exact distances of the vectors stored in
    ``exact`` -- on the GPU (``fk_refine``: id lookup, direct fp64-accumulated
    distance per candidate, (value, id) order, -1 / +-inf padding).  ``fast``
    is any index with ``search``; ``exact`` must be a GPU ``FlatIndex``.
    The metric is the fast index's (core.py:375)."""
    if shortlist < k:
        raise ValueError("shortlist must be >= k")
    q = as_vectors(q, fast.d)
    if not isinstance(exact, FlatIndex):
        raise TypeError("refine_search: `exact` must be a paper_2401_08281_b200.FlatIndex")
    if exact.d != fast.d:
        raise ValueError(f"dimension mismatch: fast d={fast.d}, exact d={exact.d}")
    metric = fast.metric
    coarse = fast.search(q, shortlist)
    dev = f"cuda:{exact.device}"
    on_cuda = is_torch(q) and q.is_cuda
    qt = q if is_torch(q) else torch.from_numpy(np.ascontiguousarray(q))
    qt = qt.to(device=dev, dtype=torch.float32).contiguous()
    cand = coarse.ids if is_torch(coarse.ids) else torch.from_numpy(np.ascontiguousarray(coarse.ids))
    cand = cand.to(device=dev, dtype=torch.int64).contiguous()
    nq = qt.shape[0]
    D = torch.empty((nq, k), dtype=torch.float32, device=dev)
    I = torch.empty((nq, k), dtype=torch.int64, device=dev)
    N.check(N.lib().fk_refine(exact._h, metric.code, _ptr(qt), nq, _ptr(cand), int(cand.shape[1]), int(k),
                              _ptr(D), _ptr(I), 1, _stream_of(exact.device)))
    if on_cuda:
        return SearchResult(I, D, k)
    return SearchResult(I.cpu().numpy(), D.cpu().numpy(), k)


class IndexFlatL2(FlatIndex):
    """Faiss-style alias: ``IndexFlatL2(d)``."""

    def __init__(self, d: int, storage: str = "fp32", device: int | None = None):
        super().__init__(d, METRIC_L2, storage=storage, device=device)


class IndexFlatIP(FlatIndex):
    """Faiss-style alias: ``IndexFlatIP(d)``."""

    def __init__(self, d: int, storage: str = "fp32", device: int | None = None):
        super().__init__(d, METRIC_IP, storage=storage, device=device)
