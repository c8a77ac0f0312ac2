"""Scene clusters for the rasterizer's cluster cull (device.build_clusters; CPU)."""

import numpy as np

from paper_2111_11103_b200.synth import make_room


def test_build_clusters_partition():
    from paper_2111_11103_b200.device import CLUSTER, build_clusters

    v, t = make_room((6.0, 5.0, 3.0), 7)
    ct, cb = build_clusters(v, t)
    assert len(ct) == len(cb) * CLUSTER and len(cb) == (len(t) + CLUSTER - 1) // CLUSTER
    ids = ct[ct >= 0]
    np.testing.assert_array_equal(np.sort(ids), np.arange(len(t)))
    for c in range(len(cb)):
        mem = ct[c * CLUSTER:(c + 1) * CLUSTER]
        pts = v[t[mem[mem >= 0]]].reshape(-1, 3)
        assert (pts >= cb[c, :3]).all() and (pts <= cb[c, 3:]).all()
