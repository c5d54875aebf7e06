"""Peer-memory exchange of the row-sharded index (``exchange="p2p"``,
``fk_xchg_*``; SURVEY 8(e) fused alternative to all-gather + merge).

The GPU box has one device, so two ranks run as two PROCESSES on cuda:0:
each exports its result block through CUDA IPC and the other opens it -- the
same code path as two GPUs over NVLink P2P (peer pointers, device-side
ready/done counters, no collective in the search).  Control plane: gloo.
Every rank's answer must equal the unsharded index bit for bit, over
repeated searches (the done counters gate list reuse) and a search that
outgrows the exchange (collective re-creation)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, metric, storage, out_dir):
    import torch.distributed as dist
    os.environ["FK_XCHG_TIMEOUT_MS"] = "60000"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex, ShardedFlatIndex
    m = METRIC_IP if metric == "ip" else METRIC_L2
    rng = np.random.default_rng(77)
    xb = rng.standard_normal((50_000, 48), dtype=np.float32)
    ids = rng.permutation(50_000).astype(np.int64) * 5 + 3
    qs = [rng.standard_normal((n, 48), dtype=np.float32) for n in (300, 300, 700)]
    sh = ShardedFlatIndex(48, m, storage=storage, device=0, exchange="p2p")
    sh.add_with_ids(xb[:20_000], ids[:20_000])
    sh.add_with_ids(xb[20_000:], ids[20_000:])
    full = FlatIndex(48, m, storage=storage, device=0)
    full.add_with_ids(xb, ids)
    ok = True
    for i, q in enumerate(qs):
        k = 10 if i < 2 else 25  # the last search outgrows the exchange (re-created collectively)
        a = sh.search(torch.from_numpy(q).cuda(), k)
        b = full.search(q, k)
        sh.xchg_status()
        ok &= bool(np.array_equal(a.ids.cpu().numpy(), b.ids) and np.array_equal(a.distances.cpu().numpy(), b.distances))
    np.save(os.path.join(out_dir, f"ok_{rank}.npy"), np.array([ok]))
    dist.barrier()
    del sh
    dist.destroy_process_group()


@pytest.mark.parametrize("metric,storage", [("l2", "fp32"), ("ip", "bf16")])
def test_p2p_exchange_two_processes_equals_unsharded(tmp_path, metric, storage):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, metric, storage, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        assert bool(np.load(os.path.join(tmp_path, f"ok_{r}.npy"))[0]), f"rank {r} differs from the unsharded index"
