"""Per-frame APIs at batched speed: MeshAnnotation.add and the session's
add_frame queue frames and fold them as batches (annotation.py).  Results
must equal the batched add_batch / the immediate library path; inputs that
are not ready-to-read device float32 (host arrays, float16, permuted, on a
busy stream) are converted without races; in-place writes to a queued tensor
are detected."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scene(n=10, c=12, seed=4):
    from paper_2111_11103_b200 import Mesh, uniform_layout
    from paper_2111_11103_b200.geometry import Intrinsics
    from paper_2111_11103_b200.synth import make_room, random_room_trajectory, softmax_maps

    v, t = make_room((6.0, 5.0, 3.0), 24)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    frames = random_room_trajectory(n, Intrinsics(100.0, 100.0, 63.5, 47.5, 128, 96), seed=seed)
    probs = softmax_maps(n, 96, 128, c, seed=1)
    return mesh, layout, frames, probs


def _state(ann):
    tex = ann.texture
    return tex._accum[:, : tex.num_classes].double().cpu().numpy(), tex._counts.cpu().numpy()


@pytest.mark.parametrize("agg,acc", [("mul", "float32"), ("sum", "float64")])
@pytest.mark.parametrize("max_batch", [None, 3])
def test_add_queue_equals_add_batch(agg, acc, max_batch):
    from paper_2111_11103_b200 import MeshAnnotation

    mesh, layout, frames, probs = _scene()
    a = MeshAnnotation(mesh, layout, num_classes=12, aggregator=agg, accum_dtype=acc, max_batch=max_batch)
    b = MeshAnnotation(mesh, layout, num_classes=12, aggregator=agg, accum_dtype=acc, max_batch=10)
    for k, fr in enumerate(frames):
        a.add(probs[k], fr)
    assert a.frames_added < len(frames) or max_batch == 3  # still queued (auto batch > 10 frames)
    b.add_batch(probs, frames)
    acc_a, cnt_a = _state(a)
    acc_b, cnt_b = _state(b)
    assert a.frames_added == len(frames)
    np.testing.assert_array_equal(cnt_a, cnt_b)
    np.testing.assert_allclose(acc_a, acc_b, rtol=1e-5, atol=1e-5)
    top2 = np.sort(acc_b, axis=1)[:, -2:]
    decided = (cnt_b > 0) & ((top2[:, 1] - top2[:, 0]) > 1e-4 * np.maximum(1.0, np.abs(acc_b).max(axis=1)))
    np.testing.assert_array_equal(a.labels(host=True)[decided], b.labels(host=True)[decided])


def test_queue_flushes_on_size_change_and_reads():
    from paper_2111_11103_b200 import MeshAnnotation
    from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics

    mesh, layout, frames, probs = _scene(n=4)
    small = Intrinsics(50.0, 50.0, 31.5, 23.5, 64, 48)
    fr_small = CameraFrame(frame_id=99, intrinsics=small, rotation=frames[0].rotation,
                           translation=frames[0].translation)
    a = MeshAnnotation(mesh, layout, num_classes=12, aggregator="sum")
    b = MeshAnnotation(mesh, layout, num_classes=12, aggregator="sum")
    p_small = probs[0, :48, :64].contiguous()
    for k in range(2):
        a.add(probs[k], frames[k])
    a.add(p_small, fr_small)  # size change folds the first two
    assert a.frames_added == 2
    a.add(probs[2], frames[2])
    b.add_batch(probs[:2], frames[:2])
    b.add_batch([p_small], [fr_small])
    b.add_batch(probs[2:3], frames[2:3])
    np.testing.assert_array_equal(a.texture.counts, b.texture.counts)
    assert a.frames_added == 4
    np.testing.assert_allclose(a.texture.accum, b.texture.accum, rtol=1e-5, atol=1e-6)


def test_queue_detects_in_place_modification():
    from paper_2111_11103_b200 import MeshAnnotation

    mesh, layout, frames, probs = _scene(n=2)
    a = MeshAnnotation(mesh, layout, num_classes=12, aggregator="sum")
    buf = probs[0].clone()
    a.add(buf, frames[0])
    buf.mul_(0.5)
    with pytest.raises(RuntimeError, match="modified in place"):
        a.flush()


def test_converted_inputs_follow_the_producer_stream():
    """float16 and permuted CUDA maps written by a slow kernel on the caller's stream
    (the conversion must not race the producer), plus host arrays."""
    import torch

    from paper_2111_11103_b200 import MeshAnnotation

    mesh, layout, frames, probs = _scene(n=6)
    ref = MeshAnnotation(mesh, layout, num_classes=12, aggregator="sum", accum_dtype="float64")
    ref.add_batch(probs.half().float(), frames)
    for mode in ("queue", "batch"):
        a = MeshAnnotation(mesh, layout, num_classes=12, aggregator="sum", accum_dtype="float64")
        items = []
        for k in range(6):
            if k % 3 == 0:
                x = torch.empty((96, 128, 12), dtype=torch.float16, device="cuda")
            elif k % 3 == 1:
                x = torch.empty((12, 96, 128), dtype=torch.float32, device="cuda").permute(1, 2, 0)
            else:
                x = None
            if x is not None:
                torch.cuda._sleep(20_000_000)  # producer still running when the map is handed over
                x.copy_(probs[k].half().float())
            else:
                x = probs[k].half().float().cpu().numpy()
            items.append(x)
        if mode == "queue":
            for k in range(6):
                a.add(items[k], frames[k])
        else:
            a.add_batch(items, frames)
        np.testing.assert_array_equal(a.texture.counts, ref.texture.counts)
        np.testing.assert_allclose(a.texture.accum, ref.texture.accum, rtol=1e-12, atol=1e-12)


def test_session_add_frame_queue_counts_and_fallbacks(tmp_path):
    import torch

    from paper_2111_11103_b200 import save_ply, save_trajectory
    from paper_2111_11103_b200.rasterizer import rasterize
    from paper_2111_11103_b200.session import add_frame, finalize_and_render, open_session

    mesh, layout, frames, probs = _scene(n=7)
    mp, tp = str(tmp_path / "m.ply"), str(tmp_path / "t.txt")
    save_ply(mp, mesh)
    save_trajectory(tp, frames)
    s = open_session(mp, tp, 0.3, "mul", "images_iid", 12)
    counts = [add_frame(s, fr.frame_id, probs[k].cpu().numpy()) for k, fr in enumerate(frames)]
    assert s.ann.frames_added == 0  # all queued
    for k, fr in enumerate(frames):
        ids = rasterize(s.mesh, s.layout, fr)
        assert int(counts[k]) == int((ids.triangle >= 0).sum())  # resolved without folding the queue
    assert s.ann.frames_added == 0
    assert s.texture.counts.sum() == sum(int(n) for n in counts)  # reading the texture folds it
    assert s.ann.frames_added == len(frames)
    labels, rows = finalize_and_render(s, [fr.frame_id for fr in frames])
    for k, fr in enumerate(frames):
        fb = s.fallbacks[fr.frame_id].view(96, 128).cpu().numpy()
        np.testing.assert_array_equal(fb, probs[k].argmax(dim=2).cpu().numpy())
        ids = rasterize(s.mesh, s.layout, fr)
        hole = ids.triangle < 0
        np.testing.assert_array_equal(labels[k][hole], fb[hole])
    assert rows.shape == (s.num_texels, 12)
    torch.cuda.synchronize()


@pytest.mark.parametrize("agg", ["mul", "sum"])
def test_row_block_item_order_equals_frame_major(agg):
    """tfb_fuse_order + tfb_fuse_ordered (the configs[3] path for accumulators beyond L2) fold
    the same contributions as the frame-major walk: counts exact, float32 sums to rounding."""
    from paper_2111_11103_b200 import MeshAnnotation

    mesh, layout, frames, probs = _scene(n=10)
    a = MeshAnnotation(mesh, layout, num_classes=12, aggregator=agg, max_batch=4, order_items=True)
    b = MeshAnnotation(mesh, layout, num_classes=12, aggregator=agg, max_batch=4, order_items=False)
    a.ORDER_SHIFT = 4  # many row blocks on this small layout
    a.add_batch(probs, frames)
    b.add_batch(probs, frames)
    acc_a, cnt_a = _state(a)
    acc_b, cnt_b = _state(b)
    np.testing.assert_array_equal(cnt_a, cnt_b)
    np.testing.assert_allclose(acc_a, acc_b, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("accum", ["float32", "fixed64"])
def test_odd_frame_size_queue_order_and_fixed(accum):
    """61x37 frames (a partial last 32-pixel chunk, H*W odd), some frames looking away from
    everything: the queue, the row-block item order and the fixed-point landing agree with a
    frame-major float64 fold."""
    from paper_2111_11103_b200 import Mesh, MeshAnnotation, uniform_layout
    from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics
    from paper_2111_11103_b200.synth import make_room, random_room_trajectory, softmax_maps

    v, t = make_room((6.0, 5.0, 3.0), 16)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 3)
    intr = Intrinsics(50.0, 50.0, 30.5, 18.5, 61, 37)
    frames = random_room_trajectory(7, intr, seed=8)
    # a camera outside the room looking away: no covered pixel at all
    frames.append(CameraFrame(99, intr, np.eye(3), np.array([0.0, 0.0, 50.0])))
    probs = softmax_maps(8, 37, 61, 9, seed=4)
    ref = MeshAnnotation(mesh, layout, num_classes=9, aggregator="mul", accum_dtype="float64", max_batch=8)
    ref.add_batch(probs, frames)
    a = MeshAnnotation(mesh, layout, num_classes=9, aggregator="mul", accum_dtype=accum, max_batch=3,
                       order_items=True)
    a.ORDER_SHIFT = 3
    for k, fr in enumerate(frames):
        a.add(probs[k], fr)
    np.testing.assert_array_equal(a.texture.counts, ref.texture.counts)
    got, want = a.texture.accum, ref.texture.accum
    err = np.abs(got - want) / np.maximum(np.abs(want), 1e-3)
    assert err.max() < 1e-5, err.max()


@pytest.mark.parametrize("max_batch", [3, 4])
@pytest.mark.parametrize("weights", ["images_iid", "pixels_iid"])
def test_split_raster_pipeline_equals_serial(max_batch, weights):
    """split_raster: batch k+1's cull / setup / binning (tfb_rasterize_phases phase 1) on a
    side stream under batch k's scatter-add, its tile kernels (phase 2) in stream order.
    With the order-free fixed-point accumulator the texture is bit-identical to the serial
    pipeline's, and so are the fused labels and the per-frame network argmax."""
    import torch

    from paper_2111_11103_b200 import MeshAnnotation

    mesh, layout, frames, probs = _scene(n=10)
    dev_probs = [torch.as_tensor(p, device="cuda") for p in probs]
    out = []
    for split in (False, True):
        a = MeshAnnotation(mesh, layout, num_classes=12, aggregator="mul", weight_mode=weights,
                           accum_dtype="fixed64", max_batch=max_batch, split_raster=split)
        fb = torch.full((10, 96 * 128), -5, dtype=torch.int32, device="cuda")
        a.add_batch(dev_probs, frames, fallback_out=fb)
        tex = a.texture
        out.append((tex._accum.clone(), tex._counts.clone(), a.labels(host=True), fb.cpu().numpy()))
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])
    np.testing.assert_array_equal(out[0][2], out[1][2])
    np.testing.assert_array_equal(out[0][3], out[1][3])
