"""Scene clusters for the rasterizer's cluster cull (device.build_clusters; CPU)."""

import numpy as np

from paper_2111_11103_b200.device import CLUSTER, CLUSTER_V, build_clusters
from paper_2111_11103_b200.synth import make_icosphere, make_room


def _check(v, t):
    cl = build_clusters(v, t)
    assert cl.dtype.itemsize == 1856
    tri = cl["tri"]
    ids = tri[:, :, 0].ravel()
    np.testing.assert_array_equal(np.sort(ids[ids >= 0]), np.arange(len(t)))  # a partition
    assert len(cl) <= 2 * ((len(t) + 63) // 64) + 1
    for c in range(len(cl)):
        nv = int(cl["nverts"][c])
        assert 0 < nv <= CLUSTER_V
        verts = cl["verts"][c, :nv]
        assert len(np.unique(verts)) == nv
        for i in range(CLUSTER):
            if tri[c, i, 0] < 0:
                continue
            np.testing.assert_array_equal(tri[c, i, 1:], t[tri[c, i, 0]])
            loc = int(cl["local"][c, i])
            np.testing.assert_array_equal([verts[(loc >> (8 * k)) & 0xFF] for k in range(3)], t[tri[c, i, 0]])
        pts = v[verts]
        assert (pts >= cl["box"][c, :3]).all() and (pts <= cl["box"][c, 3:]).all()
        assert (pts.min(0) == cl["box"][c, :3]).all() and (pts.max(0) == cl["box"][c, 3:]).all()


def test_build_clusters_room():
    v, t = make_room((6.0, 5.0, 3.0), 7)
    _check(v, t)


def test_build_clusters_split_when_vertices_exceed_128():
    # a triangle soup: 64 triangles with 192 distinct vertices -> clusters split in halves
    rng = np.random.default_rng(0)
    v = rng.normal(size=(600, 3))
    t = np.arange(600, dtype=np.int32).reshape(200, 3)
    _check(v, t)
    m = make_icosphere(1.0, 2)
    _check(m.vertices, m.triangles)
