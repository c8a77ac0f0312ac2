import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2111_11103_b200 import Mesh, TexelLayout, rasterize
from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics
z = np.load(os.path.join(ROOT, "tests/golden/raster_cases.npz"))
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    for name in [str(n) for n in z["names"]]:
        mesh = Mesh(z[name + "/verts"], z[name + "/tris"])
        steps = z[name + "/steps"]
        layout = TexelLayout(steps, z[name + "/origins"], z[name + "/offsets"], int(((steps.astype(np.int64) ** 2 + steps) // 2).sum()))
        W, H = (int(x) for x in z[name + "/wh"])
        for f, c in enumerate(z[name + "/cams"]):
            ids = rasterize(mesh, layout, CameraFrame(f, Intrinsics(c[12], c[13], c[14], c[15], W, H), c[:9].reshape(3, 3), c[9:12]))
            g = z[name + "/tri"][f]
            bad = np.argwhere(ids.triangle != g)
            if len(bad):
                print("rep", rep, name, f, "n", len(bad), [(tuple(b), int(ids.triangle[tuple(b)]), int(g[tuple(b)])) for b in bad[:4]], flush=True)
print("done")
