"""First GPU parity checks: rasterizer bit-exactness on the golden cases."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.gpu
def test_raster_golden_cases_bitexact():
    import torch
    from paper_2111_11103_b200 import Mesh, TexelLayout, rasterize
    from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics
    z = np.load(os.path.join(GOLD, "raster_cases.npz"))
    for name in [str(n) for n in z["names"]]:
        mesh = Mesh(z[name + "/verts"], z[name + "/tris"])
        offs = z[name + "/offsets"]
        steps = z[name + "/steps"]
        layout = TexelLayout(steps, z[name + "/origins"], offs, int(((steps.astype(np.int64) ** 2 + steps) // 2).sum()))
        W, H = (int(x) for x in z[name + "/wh"])
        for f, cam in enumerate(z[name + "/cams"]):
            fr = CameraFrame(0, Intrinsics(cam[12], cam[13], cam[14], cam[15], W, H), cam[:9].reshape(3, 3), cam[9:12])
            ids = rasterize(mesh, layout, fr)
            np.testing.assert_array_equal(ids.triangle, z[name + "/tri"][f], err_msg=name)
            np.testing.assert_array_equal(ids.texel, z[name + "/texel"][f], err_msg=name)
            np.testing.assert_array_equal(ids.depth, z[name + "/depth"][f], err_msg=name)
            cov = ids.triangle >= 0
            np.testing.assert_array_equal(ids.u[cov], z[name + "/u"][f][cov], err_msg=name)
            np.testing.assert_array_equal(ids.v[cov], z[name + "/v"][f][cov], err_msg=name)
