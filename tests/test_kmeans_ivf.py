"""SURVEY 8(f) consumers of the flat path, checked against golden vectors
produced by the REAL reference (tests/golden/make_golden_ivf.py):

* IVF coarse quantizer: ``IvfIndex._assign_vectors`` (ivf.py:213-214) and
  ``probe_lists`` (ivf.py:324-326) over the reference-trained centroids, L2
  and spherical (inner-product routed);
* k-means ``_assign`` (quantize.py:38-62) in fp64 against fp64 centroids.
"""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
sys.path.insert(0, os.path.dirname(HERE))

from make_golden_ivf import NPROBE, digest, ivf_inputs  # noqa: E402

GOLD = np.load(os.path.join(HERE, "golden", "golden_ivf.npz"))


def _ties_ok(x, cents, got, want, metric):
    """Rows where the ids differ must be fp32-level ties of the reference's
    own fp32 coarse search (|d_got - d_want| <= 1e-5 relative)."""
    diff = np.nonzero(got != want)[0]
    if diff.size == 0:
        return True
    xd, cd = x[diff].astype(np.float64), cents.astype(np.float64)
    if metric == "ip":
        vg = np.einsum("nd,nd->n", xd, cd[got[diff]])
        vw = np.einsum("nd,nd->n", xd, cd[want[diff]])
    else:
        vg = ((xd - cd[got[diff]]) ** 2).sum(1)
        vw = ((xd - cd[want[diff]]) ** 2).sum(1)
    return bool(np.all(np.abs(vg - vw) <= 1e-5 * np.maximum(np.abs(vw), 1e-6)))


def test_inputs_match_the_golden_run():
    xt, xa, q, c64 = ivf_inputs()
    assert digest(xt, xa, q) == str(GOLD["digest"])


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["l2", "sph"])
def test_coarse_quantizer_matches_reference_ivf(tag):
    from paper_2401_08281_b200 import assign_vectors, coarse_quantizer, probe_lists
    _, xa, q, _ = ivf_inputs()
    cents = GOLD[f"{tag}/centroids"]
    coarse = coarse_quantizer(cents.shape[1], spherical=(tag == "sph"))
    coarse.add(cents)  # ivf.py:202
    a = assign_vectors(coarse, xa)
    want = GOLD[f"{tag}/assign"]
    assert a.dtype == np.int64 and a.shape == want.shape
    assert _ties_ok(xa, cents, a, want, "ip" if tag == "sph" else "l2")
    assert (a == want).mean() > 0.999
    pr = probe_lists(coarse, q, NPROBE)
    wp = GOLD[f"{tag}/probes"]
    assert pr.shape == wp.shape
    for i in np.nonzero((pr != wp).any(1))[0]:  # only near-tie swaps allowed
        assert set(pr[i]) == set(wp[i]) or _ties_ok(q[i:i + 1].repeat(NPROBE, 0), cents, pr[i], wp[i],
                                                     "ip" if tag == "sph" else "l2")


@pytest.mark.gpu
@pytest.mark.parametrize("tag,by_ip", [("l2", False), ("ip", True)])
@pytest.mark.parametrize("shortlist", [1, 8, 64])
def test_kmeans_assign_fp64_matches_reference(tag, by_ip, shortlist):
    from paper_2401_08281_b200 import kmeans_assign
    _, xa, _, c64 = ivf_inputs()
    x = xa[:5000]
    a, err = kmeans_assign(x, c64, by_ip=by_ip, shortlist=shortlist)
    assert np.array_equal(a, GOLD[f"km_{tag}/assign"])  # fp64: exact (no ties at this precision)
    np.testing.assert_allclose(err, GOLD[f"km_{tag}/err"], rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_kmeans_assign_duplicate_centroids_first_index_wins():
    """np.argmin/argmax return the first index on exact ties (quantize.py:53-55)."""
    from paper_2401_08281_b200 import kmeans_assign
    rng = np.random.default_rng(4)
    c = rng.standard_normal((10, 16))
    c = np.concatenate([c, c[::-1]])  # every centroid twice
    x = rng.standard_normal((500, 16)).astype(np.float32)
    for by_ip in (False, True):
        a, _ = kmeans_assign(x, c, by_ip=by_ip)
        x64 = x.astype(np.float64)
        ip = x64 @ c.T
        want = ip.argmax(1) if by_ip else ((c * c).sum(1)[None, :] - 2 * ip).argmin(1)
        assert np.array_equal(a, want)
