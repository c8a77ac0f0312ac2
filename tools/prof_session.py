"""cProfile of the per-frame session loop (add_frame) on the cfg2 scene: where the
host time per queued frame goes.  python tools/prof_session.py [frames]"""
import cProfile
import os
import pstats
import sys
import tempfile

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2111_11103_b200 import Mesh, save_ply, save_trajectory  # noqa: E402
from paper_2111_11103_b200.session import add_frame, open_session  # noqa: E402
from paper_2111_11103_b200.synth import make_room, random_room_trajectory, scannet_intrinsics, softmax_maps  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    v, t = make_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    frames = random_room_trajectory(n, scannet_intrinsics(), seed=0)
    maps = softmax_maps(8, 480, 640, 40, seed=0)
    views = [maps[i] for i in range(8)]
    with tempfile.TemporaryDirectory() as d:
        mp, tp = os.path.join(d, "m.ply"), os.path.join(d, "t.txt")
        save_ply(mp, mesh)
        save_trajectory(tp, frames)
        s = open_session(mp, tp, 0.0, "mul", "images_iid", 40)
        for fr in frames[:300]:
            add_frame(s, fr.frame_id, views[0])
        s.ann.flush()
        torch.cuda.synchronize()
        pr = cProfile.Profile()
        pr.enable()
        for i, fr in enumerate(frames):
            add_frame(s, fr.frame_id, views[i % 8])
        s.ann.flush()
        torch.cuda.synchronize()
        pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
