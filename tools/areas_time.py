import time, sys
sys.path.insert(0, '.')
import torch
from paper_2111_11103_b200 import Mesh, compute_worst_case_areas
from paper_2111_11103_b200.synth import make_room, random_room_trajectory, scannet_intrinsics
v, t = make_room((6.0, 5.0, 3.0), 158)
mesh = Mesh.from_arrays(v, t)
frames = random_room_trajectory(2000, scannet_intrinsics(), seed=0)
compute_worst_case_areas(mesh, frames[:8])
torch.cuda.synchronize()
t0 = time.time()
a = compute_worst_case_areas(mesh, frames)
torch.cuda.synchronize()
print("areas 2000 frames x 300k tris: %.3f s" % (time.time() - t0), a.shape, float(a.max()))
