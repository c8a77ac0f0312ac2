"""The exchange's NCCL calls on real CUDA tensors (a one-rank NCCL group on the
test box's single GPU): reduce_scatter_tensor over the accumulator rows and the
int32 counts of every accumulator dtype (float32, fixed64 = int64, float64
parity mode), and all_gather_into_tensor of the int32 labels -- the branch of
dist.reduce_scatter_finalize that a multi-GPU run takes (dist.py).  The
multi-rank slicing and padding are covered by tests/test_dist_gloo.py on CPU."""

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(
    """
    import numpy as np, torch, torch.distributed as dist
    from paper_2111_11103_b200 import Mesh, MeshAnnotation, uniform_layout
    from paper_2111_11103_b200.dist import reduce_scatter_rows, reduce_scatter_finalize
    from paper_2111_11103_b200.geometry import Intrinsics
    from paper_2111_11103_b200.synth import make_room, random_room_trajectory, softmax_maps

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:PORT", rank=0, world_size=1)
    for dt in (torch.float32, torch.float64, torch.int64, torch.int32):
        t = (torch.arange(7 * 5, device="cuda") % 11).to(dt).reshape(7, 5)
        (got,), (lo, hi) = reduce_scatter_rows([t])
        assert (lo, hi) == (0, 7) and got.dtype == dt and torch.equal(got, t), dt

    v, t = make_room((6.0, 5.0, 3.0), 24)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    frames = random_room_trajectory(6, Intrinsics(100.0, 100.0, 63.5, 47.5, 128, 96), seed=4)
    probs = softmax_maps(6, 96, 128, 12, seed=1)
    for accum in ("float32", "fixed64", "float64"):
        a = MeshAnnotation(mesh, layout, num_classes=12, aggregator="mul", max_batch=6, accum_dtype=accum)
        b = MeshAnnotation(mesh, layout, num_classes=12, aggregator="mul", max_batch=6, accum_dtype=accum)
        a.add_batch(probs, frames)
        b.add_batch(probs, frames)
        tex = a.texture
        tex._push_host()
        seen = []

        def fin(acc, cnt, tex=tex, seen=seen):
            seen.append(int(acc.shape[0]))
            from paper_2111_11103_b200 import _native as N
            n = int(acc.shape[0])
            labels = torch.empty(n, dtype=torch.int32, device=acc.device)
            unobs = torch.empty(n, dtype=torch.uint8, device=acc.device)
            N.call("tfb_finalize", N.ptr(acc), tex.accum_kind, tex.stride, N.ptr(cnt), n, 12,
                   N.AGG_IDS[tex.aggregator], None, N.ptr(unobs), N.ptr(labels),
                   N.stream_handle(torch.cuda.current_stream(acc.device)))
            return labels

        got = reduce_scatter_finalize(tex._accum, tex._counts, fin, exchange_single=True)
        torch.cuda.synchronize()
        assert seen == [layout.total_texels], seen
        np.testing.assert_array_equal(got.cpu().numpy(), b.labels(host=True))
    dist.destroy_process_group()
    print("OK")
    """
)


def test_nccl_exchange_calls_one_rank():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("PORT", str(port))], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
