"""Multi-GPU flat search: database rows sharded across ranks.

One process per GPU (``torch.distributed``; NCCL over NVLink/NVSwitch on the
B200 box).  Rank r holds a contiguous slice of every added batch; queries are
replicated; each rank runs the fused GEMM + top-k over its shard and returns
(distance, GLOBAL storage position, id) lists; one all-gather exchanges them
(nq x k x 20 B per rank) and the merge kernel (``fk_merge_shards``) orders
the union by (distance, global position) -- exactly the unsharded reference
order (flat.py:94-118 + core.py:205-236 on the concatenated database).

``exchange="p2p"`` replaces the all-gather + merge by the peer-memory
exchange (``fk_xchg_*``): every rank's merge kernel reads the other ranks'
lists directly over NVLink P2P (CUDA IPC), with device-side ready/done
counters instead of a collective or a host synchronisation.

The reference has no distributed search (SPEC.md:115 lists distributed result
merging as a non-goal); parity here means: sharded result == single-index
result on the same data.
"""

from __future__ import annotations

import numpy as np

from .core import METRIC_L2, Metric, SearchResult, as_vectors, is_torch, metric_value

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row range [lo, hi) of an n-row batch owned by `rank`."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return lo, hi


def native_merge(metric: str, D, P, I, k: int):
    """Merge [G, nq, k] device tensors with the CUDA merge kernel."""
    from . import _native as N
    G, nq, _ = D.shape
    Dout = torch.empty((nq, k), dtype=torch.float32, device=D.device)
    Iout = torch.empty((nq, k), dtype=torch.int64, device=D.device)
    code = N.FK_METRIC_IP if metric == "ip" else N.FK_METRIC_L2
    stream = torch.cuda.current_stream(D.device).cuda_stream
    N.check(N.lib().fk_merge_shards(code, G, nq, k, D.data_ptr(), P.data_ptr(), I.data_ptr(), Dout.data_ptr(),
                                    Iout.data_ptr(), stream))
    return Dout, Iout


class ShardedFlatIndex:
    """Row-sharded exact flat index; every rank calls every method collectively.

    ``local_factory(d, metric, storage, device)`` builds the per-rank index
    (default: the GPU :class:`FlatIndex`); ``merge_fn(metric, D, P, I, k)``
    merges the gathered [world, nq, k] lists (default: the CUDA merge kernel).
    Both are injectable so the partition / position / collective logic is
    testable with a CPU stand-in under the gloo backend.
    """

    def __init__(self, d: int, metric: Metric = METRIC_L2, storage: str = "fp32", group=None, device=None,
                 local_factory=None, merge_fn=None, exchange: str = "nccl"):
        if dist is None or not dist.is_initialized():
            raise RuntimeError("ShardedFlatIndex needs an initialised torch.distributed process group")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.d = int(d)
        self.metric = metric
        self._mv = metric_value(metric)
        self.storage = storage
        if local_factory is None:
            from .flat import FlatIndex
            local_factory = FlatIndex
        self.local = local_factory(d, metric, storage, device)
        self.merge_fn = merge_fn or native_merge
        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.exchange = exchange
        self._xchg = None
        self._xcap = (0, 0)
        self.ntotal = 0
        self.is_trained = True
        self._gpos_parts: list = []
        self._gpos = None

    # ------------------------------------------------------------------ add
    def add(self, x) -> None:
        """Every rank passes the same global batch; rank r keeps its slice."""
        x = as_vectors(x, self.d)
        n = x.shape[0]
        lo, hi = shard_range(n, self.rank, self.world)
        self._add_local(x[lo:hi], self.ntotal + lo, ids=None)
        self.ntotal += n
        self._sync_plan_rows()

    def add_with_ids(self, x, ids) -> None:
        x = as_vectors(x, self.d)
        n = x.shape[0]
        ids = np.asarray(ids.cpu() if is_torch(ids) else ids, dtype=np.int64)
        if ids.shape != (n,):
            raise ValueError("ids must be a 1-d array matching the vector count")
        if np.any(ids < 0):
            raise ValueError("ids must be >= 0 (sign bit is reserved)")
        lo, hi = shard_range(n, self.rank, self.world)
        self._add_local(x[lo:hi], self.ntotal + lo, ids=ids[lo:hi])
        self.ntotal += n
        self._sync_plan_rows()

    def add_local_shard(self, x_local, global_offset: int, n_global: int, ids_local=None) -> None:
        """Add this rank's own slice of a global batch of ``n_global`` rows whose
        slice starts at global row ``global_offset`` (ranks generate their own
        shard, e.g. the 100M-row config).  Collective: every rank calls it."""
        x_local = as_vectors(x_local, self.d)
        self._add_local(x_local, self.ntotal + global_offset, ids=ids_local)
        self.ntotal += int(n_global)
        self._sync_plan_rows()

    def add_shard_rows(self, x_rows, global_row0: int) -> None:
        """Append rows of this rank's shard whose positions in the global batch
        being built start at ``global_row0`` (relative to ntotal before the
        batch).  Call ``finish_global_batch(n_global)`` once on every rank when
        all ranks have added their rows (bulk loads generated in pieces)."""
        x_rows = as_vectors(x_rows, self.d)
        self._add_local(x_rows, self.ntotal + global_row0, ids=None)

    def finish_global_batch(self, n_global: int) -> None:
        self.ntotal += int(n_global)
        self._sync_plan_rows()

    def _sync_plan_rows(self) -> None:
        # every shard runs the algorithm the unsharded search would choose
        # (e.g. fp32 1-pass vs 3xTF32 is decided on the GLOBAL row count)
        if hasattr(self.local, "set_plan_rows"):
            self.local.set_plan_rows(self.ntotal)

    def _add_local(self, xs, gpos0: int, ids) -> None:
        m = xs.shape[0]
        if m == 0:
            return
        if ids is None:
            ids = np.arange(gpos0, gpos0 + m, dtype=np.int64)
        self.local.add_with_ids(xs, ids)
        part = np.arange(gpos0, gpos0 + m, dtype=np.int64)
        self._gpos_parts.append(part)
        self._gpos = None

    def reset(self) -> None:
        self.local.reset()
        self.ntotal = 0
        self._sync_plan_rows()
        self._gpos_parts = []
        self._gpos = None

    # ------------------------------------------------------------------ search
    def _gpos_table(self, like):
        if self._gpos is None:
            table = (np.concatenate(self._gpos_parts) if self._gpos_parts else np.zeros(0, dtype=np.int64))
            self._gpos = torch.from_numpy(table)
        if is_torch(like) and like.is_cuda and self._gpos.device != like.device:
            self._gpos = self._gpos.to(like.device)
        return self._gpos

    def search(self, q, k: int) -> SearchResult:
        if k < 1:
            raise ValueError("k must be >= 1")
        q = as_vectors(q, self.d)
        if self.exchange == "p2p":
            return self._search_p2p(q, int(k))
        res, P = self.local.search_with_positions(q, int(k))
        D, I = res.distances, res.ids
        if not is_torch(D):
            D, I, P = torch.from_numpy(np.ascontiguousarray(D)), torch.from_numpy(I), torch.from_numpy(P)
        table = self._gpos_table(P)
        if table.numel():
            Pg = torch.where(P >= 0, table[P.clamp(min=0)], torch.full_like(P, -1))
        else:
            Pg = torch.full_like(P, -1)
        Dg = self._all_gather(D.contiguous())
        Pg = self._all_gather(Pg.contiguous())
        Ig = self._all_gather(I.contiguous())
        Dm, Im = self.merge_fn(self._mv, Dg, Pg, Ig, int(k))
        if not (is_torch(q) and q.is_cuda):
            Dm = Dm.cpu().numpy() if is_torch(Dm) else Dm
            Im = Im.cpu().numpy() if is_torch(Im) else Im
        return SearchResult(Im, Dm, int(k))

    def _all_gather(self, t):
        if self.world == 1:
            return t.unsqueeze(0)
        if t.is_cuda and dist.get_backend(self.group) == "nccl":
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t, group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=self.group)
        return torch.stack(parts)

    # ------------------------------------------------------------------ peer-memory exchange
    def _global_positions(self, P):
        table = self._gpos_table(P)
        if table.numel():
            return torch.where(P >= 0, table[P.clamp(min=0)], torch.full_like(P, -1))
        return torch.full_like(P, -1)

    def _xchg_ensure(self, nq: int, k: int, device: int):
        """(Re)create the exchange when the result shape outgrows it -- every
        rank sees the same (nq, k) (queries are replicated), so all ranks do
        this collectively: handles are exchanged with all_gather_object."""
        from . import _native as N
        import ctypes
        if self._xchg is not None and nq <= self._xcap[0] and k <= self._xcap[1]:
            return self._xchg
        L = N.lib()
        self._xchg_close()
        cap = (max(nq, self._xcap[0]), max(k, self._xcap[1]))
        hb = L.fk_xchg_handle_bytes()
        handle = (ctypes.c_char * hb)()
        x = ctypes.c_void_p()
        N.check(L.fk_xchg_create(device, self.rank, self.world, cap[0], cap[1], ctypes.byref(x), handle))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=self.group)
        allh = (ctypes.c_char * (hb * self.world)).from_buffer_copy(b"".join(handles))
        N.check(L.fk_xchg_connect(x, allh))
        self._xchg, self._xcap = x, cap
        return x

    def _xchg_close(self):
        if self._xchg is not None:
            from . import _native as N
            torch.cuda.synchronize()
            dist.barrier(group=self.group)  # no peer still reads this rank's block
            N.lib().fk_xchg_destroy(self._xchg)
            self._xchg = None

    def xchg_status(self) -> None:
        """Synchronise and raise if a device-side exchange wait timed out."""
        if self._xchg is not None:
            from . import _native as N
            N.check(N.lib().fk_xchg_status(self._xchg))

    def _search_p2p(self, q, k: int) -> SearchResult:
        from . import _native as N
        host = not (is_torch(q) and q.is_cuda)
        dev = self.local.device
        qd = q.to(f"cuda:{dev}") if is_torch(q) else torch.from_numpy(np.ascontiguousarray(q)).to(f"cuda:{dev}")
        res, P = self.local.search_with_positions(qd, k)
        nq = qd.shape[0]
        Pg = self._global_positions(P).contiguous()
        x = self._xchg_ensure(nq, k, dev)
        L = N.lib()
        stream = torch.cuda.current_stream(dev).cuda_stream
        Dm = torch.empty((nq, k), dtype=torch.float32, device=qd.device)
        Im = torch.empty((nq, k), dtype=torch.int64, device=qd.device)
        code = N.FK_METRIC_IP if self._mv == "ip" else N.FK_METRIC_L2
        N.check(L.fk_xchg_acquire(x, stream))
        N.check(L.fk_xchg_put(x, nq, k, res.distances.data_ptr(), Pg.data_ptr(), res.ids.data_ptr(), stream))
        N.check(L.fk_xchg_merge(x, code, nq, k, Dm.data_ptr(), Im.data_ptr(), stream))
        if host:
            return SearchResult(Im.cpu().numpy(), Dm.cpu().numpy(), k)
        return SearchResult(Im, Dm, k)

    def __del__(self):
        try:
            if self._xchg is not None:
                from . import _native as N
                N.lib().fk_xchg_destroy(self._xchg)
                self._xchg = None
        except Exception:
            pass
