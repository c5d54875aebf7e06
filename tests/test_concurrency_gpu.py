"""Concurrent reads on one index (core.py:107-112: reads are
safe from many threads): searches and range searches from several threads,
each on its own CUDA stream, give results bit-identical to serial runs
(the handle's scratch is stream-ordered; range results are per call)."""

import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_08281_b200 import METRIC_L2, FlatIndex  # noqa: E402


@pytest.mark.parametrize("nb", [50_000, 300_000])
def test_threads_on_streams_match_serial(nb):
    rng = np.random.default_rng(nb)
    xb = rng.standard_normal((nb, 64), dtype=np.float32)
    idx = FlatIndex(64, METRIC_L2)
    idx.add(xb)
    qs = [torch.from_numpy(rng.standard_normal((1000 + 37 * i, 64), dtype=np.float32)).cuda() for i in range(6)]
    ks = [1, 10, 16, 100, 10, 5]
    serial = [idx.search(q, k) for q, k in zip(qs, ks)]
    torch.cuda.synchronize()
    out = [None] * len(qs)

    def worker(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                r = idx.search(qs[i], ks[i])
            s.synchronize()
            out[i] = (r.ids.clone(), r.distances.clone())
            s.synchronize()

    th = [threading.Thread(target=worker, args=(i,)) for i in range(len(qs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(len(qs)):
        assert torch.equal(out[i][0], serial[i].ids) and torch.equal(out[i][1], serial[i].distances), i


def test_concurrent_range_searches():
    rng = np.random.default_rng(3)
    xb = rng.standard_normal((20_000, 16), dtype=np.float32)
    idx = FlatIndex(16, METRIC_L2)
    idx.add(xb)
    qs = [rng.standard_normal((50 * (i + 1), 16), dtype=np.float32) for i in range(5)]
    radii = [4.0, 6.0, 8.0, 5.0, 7.0]
    serial = [idx.range_search(q, r) for q, r in zip(qs, radii)]
    out = [None] * 5

    def worker(i):
        for _ in range(4):
            out[i] = idx.range_search(qs[i], radii[i])

    th = [threading.Thread(target=worker, args=(i,)) for i in range(5)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(5):
        assert np.array_equal(out[i].lims, serial[i].lims)
        assert np.array_equal(out[i].ids, serial[i].ids) and np.array_equal(out[i].distances, serial[i].distances)
