"""Debug: repeat the golden raster cases many times, report mismatches per case."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2111_11103_b200 import Mesh, TexelLayout
from paper_2111_11103_b200.device import DeviceScene
from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics

z = np.load(os.path.join(ROOT, "tests/golden/raster_cases.npz"))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for clusters in ("0", "1"):
    os.environ["TFB_NO_CLUSTERS"] = "1" if clusters == "0" else "0"
    for name in [str(n) for n in z["names"]]:
        mesh = Mesh(z[name + "/verts"], z[name + "/tris"])
        steps = z[name + "/steps"]
        layout = TexelLayout(steps, z[name + "/origins"], z[name + "/offsets"],
                             int(((steps.astype(np.int64) ** 2 + steps) // 2).sum()))
        W, H = (int(x) for x in z[name + "/wh"])
        cams = z[name + "/cams"]
        sc = DeviceScene(mesh, layout)
        frames = [CameraFrame(i, Intrinsics(c[12], c[13], c[14], c[15], W, H), c[:9].reshape(3, 3), c[9:12]) for i, c in enumerate(cams)]
        ct = sc.cams_tensor(frames)
        B = len(frames)
        bad = 0
        for r in range(reps):
            for want_depth in (False, True):
                rows = torch.empty((B, W * H), dtype=torch.int32, device="cuda")
                tri = torch.empty((B, W * H), dtype=torch.int32, device="cuda")
                tex = torch.empty((B, W * H), dtype=torch.int32, device="cuda")
                dep = torch.empty((B, W * H), dtype=torch.float64, device="cuda") if want_depth else None
                u = torch.empty((B, W * H), dtype=torch.float64, device="cuda") if want_depth else None
                v = torch.empty((B, W * H), dtype=torch.float64, device="cuda") if want_depth else None
                sc.rasterize(ct, W, H, rows, None, tri, tex, dep, u, v)
                t = tri.cpu().numpy().reshape(B, H, W)
                for f in range(B):
                    gold = z[name + "/tri"][f]
                    nbad = int((t[f] != gold).sum())
                    if nbad:
                        bad += 1
                        idx = np.argwhere(t[f] != gold)[:3]
                        print("MISMATCH clusters=%s case=%s frame=%d depth=%s rep=%d npix=%d m=%d WxH=%dx%d ex=%s got=%s want=%s" % (
                            clusters, name, f, want_depth, r, nbad, mesh.num_triangles, W, H, idx.tolist(),
                            [int(t[f][tuple(i)]) for i in idx], [int(gold[tuple(i)]) for i in idx]), flush=True)
        print("case", name, "clusters", clusters, "bad", bad, flush=True)
