"""Golden SMPB / SMTX files written by the *reference* writers (formats.py).

Run in the build container only (imports the reference read-only from
/root/reference/pkg/src); the tests compare this package's readers and
writers against the committed files byte for byte:

    python tests/golden/make_golden_formats.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import texelfuse as tf  # noqa: E402
from texelfuse import formats  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "formats")


def strip_mesh(m):
    """m triangles in a strip (same shape as the reference tests' helper)."""
    v = [[float(i // 2), float(i % 2), 1.0] for i in range(m + 2)]
    t = [[i, i + 1, i + 2] if i % 2 == 0 else [i + 1, i, i + 2] for i in range(m)]
    return tf.Mesh.from_arrays(np.array(v), np.array(t, dtype=np.int32))


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(11)
    p = rng.random((12, 17, 5)).astype(np.float32) + 1e-3
    p /= p.sum(axis=2, keepdims=True)
    formats.write_probability_image(os.path.join(OUT, "probs_12x17x5.smpb"), p)
    np.save(os.path.join(OUT, "probs_12x17x5.npy"), p)
    q = rng.random((3, 4, 40)).astype(np.float32)
    q /= q.sum(axis=2, keepdims=True)
    formats.write_probability_image(os.path.join(OUT, "probs_3x4x40.smpb"), q)
    np.save(os.path.join(OUT, "probs_3x4x40.npy"), q)

    mesh = strip_mesh(4)
    layout = tf.build_texel_layout(mesh, np.array([400.0, 0.0, 25.0, 100.0]), 0.2)
    n = layout.total_texels
    rows = rng.random((n, 3)).astype(np.float32)
    rows /= rows.sum(axis=1, keepdims=True)
    counts = rng.integers(0, 50, size=n).astype(np.int64)
    unobs = counts % 7 == 0
    formats.write_texture(os.path.join(OUT, "texture.smtx"), layout, rows, counts, unobserved=unobs)
    np.savez(os.path.join(OUT, "texture.npz"), steps=layout.steps, origins=layout.origins,
             offsets=layout.offsets, rows=rows, counts=counts, unobserved=unobs)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
