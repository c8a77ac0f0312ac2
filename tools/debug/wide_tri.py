import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2111_11103_b200 import Mesh, uniform_layout
from paper_2111_11103_b200.device import DeviceScene
from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics
os.environ["TFB_NO_CLUSTERS"] = "1"
W = H = 64
v = np.array([[-10, -10, 5], [10, -10, 5], [0, 10, 5]], dtype=np.float64)
for ntri in (1, 2, 3):
    vs = np.concatenate([v + [0, 0, k * 0.1] for k in range(ntri)])
    t = np.arange(3 * ntri, dtype=np.int32).reshape(ntri, 3)
    mesh = Mesh.from_arrays(vs, t)
    layout = uniform_layout(mesh, 1)
    sc = DeviceScene(mesh, layout)
    fr = CameraFrame(0, Intrinsics(32.0, 32.0, 31.5, 31.5, W, H), np.eye(3), np.zeros(3))
    ct = sc.cams_tensor([fr])
    rows = torch.empty((1, W * H), dtype=torch.int32, device="cuda")
    tri = torch.empty((1, W * H), dtype=torch.int32, device="cuda")
    tex = torch.empty((1, W * H), dtype=torch.int32, device="cuda")
    sc.rasterize(ct, W, H, rows, None, tri, tex)
    a = tri.cpu().numpy().reshape(H, W)
    cov = (a >= 0).reshape(8, 8, 4, 16).any(axis=(1, 3))  # tile rows x tile cols covered
    print(ntri, "tiles covered (TYxTX):")
    print(cov.astype(int))
