import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2111_11103_b200 import Mesh, TexelLayout, rasterize
from paper_2111_11103_b200.device import DeviceScene
from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics
z = np.load(os.path.join(ROOT, "tests/golden/raster_cases.npz"))
for name in ("chain", "clip0", "random0"):
    mesh = Mesh(z[name + "/verts"], z[name + "/tris"])
    steps = z[name + "/steps"]
    layout = TexelLayout(steps, z[name + "/origins"], z[name + "/offsets"], int(((steps.astype(np.int64) ** 2 + steps) // 2).sum()))
    W, H = (int(x) for x in z[name + "/wh"])
    c = z[name + "/cams"][0]
    fr = CameraFrame(0, Intrinsics(c[12], c[13], c[14], c[15], W, H), c[:9].reshape(3, 3), c[9:12])
    g = z[name + "/tri"][0]
    a = rasterize(mesh, layout, fr).triangle
    sc = DeviceScene(mesh, layout)
    ct = sc.cams_tensor([fr])
    for B in (1,):
        rows = torch.empty((1, W * H), dtype=torch.int32, device="cuda")
        tri = torch.empty((1, W * H), dtype=torch.int32, device="cuda")
        tex = torch.empty((1, W * H), dtype=torch.int32, device="cuda")
        sc.rasterize(ct, W, H, rows, None, tri, tex)
        b = tri.cpu().numpy().reshape(H, W)
    print(name, "api bad", int((a != g).sum()), "direct bad", int((b != g).sum()), "api!=direct", int((a != b).sum()), "cams equal", bool(torch.equal(ct, rasterize.__globals__['scene_for'](mesh, layout).cams_tensor([fr]))))
