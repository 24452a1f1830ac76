"""Generate golden fixtures under tests/golden/ by running the UNMODIFIED reference.

TEST INFRASTRUCTURE ONLY.  Run in the build container (where /root/reference
exists):  python -m oracle.make_golden
Each .npz holds the seeded inputs and the reference's outputs; the CPU tests
pin `oracle/stage1.py` against them and the GPU tests pin the CUDA path against
them.  The reference runs with BLAS pinned to one thread.
"""

from __future__ import annotations

import os

import numpy as np
from threadpoolctl import threadpool_limits

from oracle import refbridge as rb
from paper_2403_01444_b200 import scenes

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _grid_arr(grid):
    return dict(grid_levels=grid["levels"], grid_features=grid["features"],
                grid_log2_table=grid["log2_table"], grid_base=grid["base"],
                grid_growth=grid["growth"], grid_lo=np.array(grid["lo"]),
                grid_hi=np.array(grid["hi"]))


def _cam_arr(cam, p="cam_"):
    return {p + "w2c": cam["w2c"], p + "intr": np.array([cam["fx"], cam["fy"], cam["cx"], cam["cy"]]),
            p + "size": np.array([cam["width"], cam["height"]]), p + "near": cam["near"]}


def _cloud_arr(cloud, p="cloud_"):
    return {p + k: v for k, v in cloud.items()}


def _flat_tiles(tiles):
    """[(y0,y1,x0,x1,members)] -> (rects (T,4) int64, counts (T,), members (D,))."""
    rects = np.array([[t[0], t[1], t[2], t[3]] for t in tiles], dtype=np.int64).reshape(-1, 4)
    counts = np.array([len(t[4]) for t in tiles], dtype=np.int64)
    mem = np.concatenate([t[4] for t in tiles]).astype(np.int64) if tiles else np.zeros(0, np.int64)
    return rects, counts, mem


def gen_encode(R):
    rng = np.random.default_rng(101)
    out = {}
    for tag, grid in (
        # box corners exactly representable in float32 so the face points stay inside
        ("small", dict(levels=4, features=2, log2_table=10, base=4, growth=1.5,
                       lo=(-1.125, -0.875, -1.25), hi=(1.25, 1.0, 0.75))),
        ("cfg1", dict(levels=16, features=2, log2_table=15, base=16,
                      growth=scenes.growth_for(16, 2048, 16),
                      lo=(-3.75, -3.25, -3.875), hi=(3.5, 3.625, 3.125))),
    ):
        lo, hi = np.array(grid["lo"]), np.array(grid["hi"])
        x = scenes.f32(rng.uniform(lo, hi, size=(1500, 3)))
        x[:5] = lo  # corners / faces of the box
        x[5:10] = hi
        cache = rb.ref_cache(R, grid, *_rand_ntc(grid, 64, seed=3))
        feats, ctx = cache.encode(x)
        res = np.array([cache.grid.resolution(l) for l in range(grid["levels"])])
        extra = dict(feats=feats, tables=cache.tables) if tag == "small" else {}
        np.savez_compressed(os.path.join(OUT, f"encode_{tag}.npz"), x=x,
                            idx=ctx.corner_idx.astype(np.int32), w=ctx.corner_w, res=res,
                            **extra, **_grid_arr(grid))
        out[tag] = len(x)
    return out


def _rand_ntc(grid, hidden, seed):
    from oracle import stage1 as O

    tables, mlp = O.init_ntc(grid, hidden_dim=hidden, output_init="random", seed=seed)
    return tables, mlp


def gen_ntc(R):
    rng = np.random.default_rng(202)
    grid = dict(levels=4, features=2, log2_table=10, base=4, growth=1.5,
                lo=(-1.0, -1.0, -1.0), hi=(1.0, 1.0, 1.0))
    tables, mlp = _rand_ntc(grid, 64, seed=5)
    # non-trivial tables so hidden units leave the ReLU floor
    tables = scenes.f32(rng.uniform(-0.5, 0.5, size=tables.shape))
    cache = rb.ref_cache(R, grid, tables, mlp)
    x = scenes.f32(rng.uniform(-1, 1, size=(500, 3)))
    d_mu, d_q, ctx = cache.forward(x)
    g_mu = rng.normal(size=d_mu.shape)
    g_q = rng.normal(size=d_q.shape)
    grads, touched = cache.backward(ctx, g_mu, g_q)
    arrs = dict(x=x, tables=tables, d_mu=d_mu, d_q=d_q, g_mu=g_mu, g_q=g_q,
                **{f"mlp_w{i}": w for i, w in enumerate(mlp["weights"])},
                **{f"mlp_b{i}": b for i, b in enumerate(mlp["biases"])},
                **{f"grad_{k}": v for k, v in grads.items()},
                **{f"touched_{k}": v for k, v in touched.items()}, **_grid_arr(grid))
    # two lazy Adam steps on those grads
    cache.adam_step(grads, 0.002, touched)
    cache.adam_step(grads, 0.002, touched)
    arrs.update({f"after2_{k}": v for k, v in cache.get_params().items()})
    np.savez_compressed(os.path.join(OUT, "ntc.npz"), **arrs)


def gen_transform(R):
    rng = np.random.default_rng(303)
    sc = scenes.small_scene(seed=7, n=300, sh_degree=1)
    cloud = sc.cloud
    grid = dict(sc.grid)
    # leave a few means outside the box (pass-through rows)
    cloud["means"][:4] += np.array([10.0, 0.0, 0.0])
    tables, mlp = _rand_ntc(grid, 64, seed=9)
    tables = scenes.f32(rng.uniform(-0.3, 0.3, size=tables.shape))
    cache = rb.ref_cache(R, grid, tables, mlp)
    rc = rb.ref_cloud(R, cloud)
    out, tctx = R["transform"].apply_ntc(rc, cache)
    gm = rng.normal(size=(len(cloud["means"]), 3))
    gr = rng.normal(size=(len(cloud["means"]), 4))
    gs = rng.normal(size=(len(cloud["means"]), 4, 3))
    grads, _ = R["transform"].apply_ntc_backward(tctx, gm, gr, gs)
    np.savez_compressed(os.path.join(OUT, "transform.npz"), tables=tables,
                        **{f"mlp_w{i}": w for i, w in enumerate(mlp["weights"])},
                        **{f"mlp_b{i}": b for i, b in enumerate(mlp["biases"])},
                        **_grid_arr(grid), **_cloud_arr(cloud), inside=tctx.inside,
                        out_means=out.means, out_rotations=out.rotations, out_sh=out.sh,
                        g_means=gm, g_rot=gr, g_sh=gs,
                        **{f"grad_{k}": v for k, v in grads.items()})


def gen_raster(R):
    rng = np.random.default_rng(404)
    for tag, sh_deg, bg, settings in (
        ("default", 1, np.array([0.1, 0.3, 0.2]), dict(tile_size=16, alpha_clamp=0.99,
                                                       skip_alpha=1 / 255.0,
                                                       stop_transmittance=1e-4)),
        ("smooth", 1, np.array([0.3, 0.2, 0.4]), dict(tile_size=16, alpha_clamp=0.99,
                                                      skip_alpha=0.0,
                                                      stop_transmittance=0.0)),
    ):
        sc = scenes.small_scene(seed=11, n=600, width=70, height=52, sh_degree=sh_deg)
        cloud = sc.cloud
        cloud["opacity_logits"][:20] = 6.0  # some clamped splats
        cam = sc.cameras[0]
        rc = rb.ref_cloud(R, cloud)
        out, ctx = R["rasterizer"].rasterize_forward(rc, rb.ref_camera(R, cam), bg,
                                                      rb.ref_settings(R, settings))
        d_img = rng.normal(size=out.image.shape)
        g = R["rasterizer"].rasterize_backward(ctx, d_img)
        rects, counts, mem = _flat_tiles(ctx.tiles)
        np.savez_compressed(os.path.join(OUT, f"raster_{tag}.npz"), **_cloud_arr(cloud),
                            **_cam_arr(cam), bg=bg,
                            settings=np.array([settings["tile_size"], settings["alpha_clamp"],
                                               settings["skip_alpha"],
                                               settings["stop_transmittance"]]),
                            image=out.image, alpha=out.alpha_map,
                            touch=out.per_gaussian_touch_count, indices=ctx.indices,
                            tile_rects=rects, tile_counts=counts, tile_members=mem,
                            d_image=d_img, d_means=g.d_means, d_rotations=g.d_rotations,
                            d_log_scales=g.d_log_scales, d_opacity_logits=g.d_opacity_logits,
                            d_sh=g.d_sh, viewspace=g.viewspace_grad_norm,
                            contributed=g.contributed)


def gen_loss(R):
    rng = np.random.default_rng(505)
    x = rng.uniform(0.1, 0.9, size=(40, 37, 3))
    y = np.clip(x + rng.normal(scale=0.1, size=x.shape), 0, 1)
    loss, grad = R["losses"].render_loss(x, y)
    np.savez_compressed(os.path.join(OUT, "loss.npz"), x=x, y=y, loss=loss, grad=grad)


def gen_stage1(R):
    """Two Stage-1 iterations driven through the reference functions in
    process_frame order (pipeline.py:262-277)."""
    from oracle import stage1 as O

    sc = scenes.small_scene(seed=21, n=1500, width=64, height=48, sh_degree=1, n_views=2)
    cloud, grid = sc.cloud, sc.grid
    tables, mlp = O.init_ntc(grid, hidden_dim=64, output_init="random", seed=4)
    rng = np.random.default_rng(606)
    tables = scenes.f32(rng.uniform(-0.05, 0.05, size=tables.shape))
    cache = rb.ref_cache(R, grid, tables, mlp)
    targets = []
    for cam in sc.cameras:
        moved = scenes.moved_cloud(cloud, np.random.default_rng(99), deg=3.0)
        img, _ = R["rasterizer"].rasterize_forward(rb.ref_cloud(R, moved), rb.ref_camera(R, cam))
        targets.append(img.image)
    rc = rb.ref_cloud(R, cloud)
    enc = None
    losses, grads_first = [], None
    order = [0, 1]
    for t, v in enumerate(order):
        tr, tctx = R["transform"].apply_ntc(rc, cache, encode_ctx=enc)
        enc = tctx.fwd.encode if enc is None else enc
        out, rctx = R["rasterizer"].rasterize_forward(tr, rb.ref_camera(R, sc.cameras[v]))
        loss, d_img = R["losses"].render_loss(out.image, targets[v])
        losses.append(loss)
        g = R["rasterizer"].rasterize_backward(rctx, d_img)
        cg, touched = R["transform"].apply_ntc_backward(tctx, g.d_means, g.d_rotations, g.d_sh)
        if grads_first is None:
            grads_first = dict(cg)
            img_first = out.image
        cache.adam_step(cg, 0.002, touched)
    np.savez_compressed(os.path.join(OUT, "stage1.npz"), **_cloud_arr(cloud), **_grid_arr(grid),
                        tables=tables, **{f"mlp_w{i}": w for i, w in enumerate(mlp["weights"])},
                        **{f"mlp_b{i}": b for i, b in enumerate(mlp["biases"])},
                        **_cam_arr(sc.cameras[0], "cam0_"), **_cam_arr(sc.cameras[1], "cam1_"),
                        target0=targets[0], target1=targets[1], losses=np.array(losses),
                        image_first=img_first,
                        **{f"grad1_{k}": v for k, v in grads_first.items()},
                        **{f"after2_{k}": v for k, v in cache.get_params().items()})


def gen_ntc_blob(R):
    """streamio.serialize_ntc bytes of a seeded cache."""
    import sys

    sys.path.insert(0, rb.REF_SRC)
    from splatstream import streamio

    rng = np.random.default_rng(303)
    grid = dict(levels=4, features=2, log2_table=9, base=4, growth=1.5,
                lo=(-1.5, -1.0, -0.75), hi=(1.25, 1.0, 2.0))
    tables, mlp = _rand_ntc(grid, 64, seed=9)
    tables = scenes.f32(rng.uniform(-0.5, 0.5, size=tables.shape))
    cache = rb.ref_cache(R, grid, tables, mlp)
    blob = streamio.serialize_ntc(cache)
    np.savez_compressed(os.path.join(OUT, "ntc_blob.npz"), blob=np.frombuffer(blob, np.uint8),
                        tables=tables, **_grid_arr(grid),
                        **{f"mlp_w{i}": w for i, w in enumerate(mlp["weights"])},
                        **{f"mlp_b{i}": b for i, b in enumerate(mlp["biases"])})


def gen_warmup(R):
    """losses.warmup_loss on random outputs and ntc.warmup_train on a small
    cache."""
    rng = np.random.default_rng(404)
    d_mu = rng.normal(scale=0.05, size=(300, 3))
    d_q = rng.normal(size=(300, 4))
    loss, g_mu, g_q = R["losses"].warmup_loss(d_mu, d_q)
    grid = dict(levels=4, features=2, log2_table=10, base=4, growth=1.5,
                lo=(-1.0, -1.0, -1.0), hi=(1.0, 1.0, 1.0))
    tables, mlp = _rand_ntc(grid, 64, seed=11)
    tables = scenes.f32(rng.uniform(-0.2, 0.2, size=tables.shape))
    cache = rb.ref_cache(R, grid, tables, mlp)
    means = scenes.f32(rng.uniform(-0.8, 0.8, size=(400, 3)))
    params, hist = R["ntc"].warmup_train(cache, means, noise_sigma=0.05, iterations=5,
                                         lr=0.002, batch_size=256, seed=7)
    np.savez_compressed(os.path.join(OUT, "warmup.npz"), d_mu=d_mu, d_q=d_q, loss=loss,
                        g_mu=g_mu, g_q=g_q, tables=tables, means=means, history=np.array(hist),
                        **_grid_arr(grid),
                        **{f"mlp_w{i}": w for i, w in enumerate(mlp["weights"])},
                        **{f"mlp_b{i}": b for i, b in enumerate(mlp["biases"])},
                        **{f"after_{k}": v for k, v in params.items()})


def gen_playback(R):
    """pipeline.materialize_frame / playback_render on a constructed stream
    (SURVEY.md §8 F3): an initial cloud, three frame records (NTC blob + added
    Gaussians), frames 0..3 rendered from one camera."""
    import sys

    sys.path.insert(0, rb.REF_SRC)
    from splatstream import pipeline, streamio

    rng = np.random.default_rng(505)
    sc = scenes.small_scene(seed=55, n=600, width=72, height=56, sh_degree=1, n_views=1)
    grid = sc.grid
    records, arrs = [], {}
    for f in range(3):
        tables, mlp = _rand_ntc(grid, 64, seed=20 + f)
        tables = scenes.f32(rng.uniform(-0.02, 0.02, size=tables.shape))
        mlp["weights"][-1] = scenes.f32(mlp["weights"][-1] * 0.05)
        b = np.zeros(7)
        b[:3] = rng.normal(scale=0.02, size=3)
        b[3:] = [1.0, 0.0, 0.0, 0.0]
        b[3:] += rng.normal(scale=0.05, size=4)
        mlp["biases"][-1] = scenes.f32(b)
        blob = streamio.serialize_ntc(rb.ref_cache(R, grid, tables, mlp))
        add = scenes.small_scene(seed=60 + f, n=40, width=8, height=8, sh_degree=1,
                                 n_views=1).cloud
        records.append(streamio.FrameRecord(f + 1, blob, rb.ref_cloud(R, add)))
        arrs[f"blob{f}"] = np.frombuffer(blob, np.uint8)
        arrs.update({f"add{f}_{k}": v for k, v in add.items()})
    bg = [0.1, 0.2, 0.3]
    stream = streamio.StreamData({"background": bg}, rb.ref_cloud(R, sc.cloud), b"", records)
    cam = rb.ref_camera(R, sc.cameras[0])
    for i in range(4):
        arrs[f"image{i}"] = pipeline.playback_render(stream, i, cam)
    np.savez_compressed(os.path.join(OUT, "playback.npz"), **_cloud_arr(sc.cloud),
                        **_cam_arr(sc.cameras[0]), background=np.array(bg), **arrs)


def gen_stage2(R):
    """adaptive.stage2_optimize: a small frozen cloud, 60
    spawned additional Gaussians, 2 views, 6 iterations (3 epochs of quantity
    control: a split in epoch 2, prunes in epochs 2 and 3).  Decision margins
    (measured): view-space gradients >= 24 % from tau_grad, opacities >= 2.4 %
    from tau_alpha."""
    import sys

    sys.path.insert(0, rb.REF_SRC)
    from splatstream import adaptive, rasterizer

    sc = scenes.small_scene(seed=77, n=500, width=64, height=48, sh_degree=1, n_views=2)
    cloud = rb.ref_cloud(R, sc.cloud)
    rng = np.random.default_rng(3)
    cfg = adaptive.AdditionConfig(tau_grad=2e-4, max_additional=100)
    sel = np.sort(rng.choice(len(sc.cloud["means"]), 60, replace=False))
    add = adaptive.spawn_gaussians(cloud, sel, cfg, rng)
    moved = rb.ref_cloud(R, scenes.moved_cloud(sc.cloud, np.random.default_rng(9)))
    views, arrs = [], {}
    for v, c in enumerate(sc.cameras):
        cam = rb.ref_camera(R, c)
        out, _ = rasterizer.rasterize_forward(moved, cam)
        views.append((cam, out.image))
        arrs.update(_cam_arr(c, f"cam{v}_"))
        arrs[f"target{v}"] = out.image
    add_in = {k: getattr(add, k).copy() for k in ("means", "rotations", "log_scales",
                                                   "opacity_logits", "sh")}
    final, losses = adaptive.stage2_optimize(cloud, add, views, cfg, 6, np.random.default_rng(11))
    np.savez_compressed(os.path.join(OUT, "stage2.npz"), **_cloud_arr(sc.cloud),
                        **_cloud_arr(add_in, "add_"), **arrs,
                        **{f"final_{k}": getattr(final, k) for k in add_in},
                        losses=np.array(losses), tau_grad=2e-4, max_additional=100, iterations=6,
                        rng_seed=11)


def gen_stage1_loop(R):
    """The reference's own Stage-1 loop: process_frame (pipeline.py:238-283)
    with stage2_iterations = 0, run unmodified; observers on ViewspaceStats.add
    and on the rasterize_forward it calls record the view order and the
    last-epoch statistics window (pipeline.py:251-279, adaptive.py:79-97)."""
    import sys

    if rb.REF_SRC not in sys.path:
        sys.path.insert(0, rb.REF_SRC)
    from splatstream import adaptive, pipeline

    from oracle import stage1 as O

    sc = scenes.small_scene(seed=31, n=1200, width=64, height=48, sh_degree=1, n_views=4)
    cloud, grid = sc.cloud, sc.grid
    tables, mlp = O.init_ntc(grid, hidden_dim=64, output_init="random", seed=6)
    tables = scenes.f32(np.random.default_rng(707).uniform(-0.05, 0.05, size=tables.shape))
    cache = rb.ref_cache(R, grid, tables, mlp)
    cams = [rb.ref_camera(R, c) for c in sc.cameras]
    moved = scenes.moved_cloud(cloud, np.random.default_rng(98), deg=2.5, shift=(0.02, 0.0, -0.01))
    targets = [R["rasterizer"].rasterize_forward(rb.ref_cloud(R, moved), c)[0].image for c in cams]
    views = list(zip(cams, targets))
    cfg = pipeline.PipelineConfig(stage1_iterations=10, stage2_iterations=0, seed=5,
                                  grid=rb.ref_grid(R, grid))
    frame_index = 3
    seen, stats_obj = [], []
    orig_raster, orig_add = pipeline.rasterize_forward, adaptive.ViewspaceStats.add

    def raster_observer(cloud_, camera, *a, **k):
        seen.append(next(i for i, c in enumerate(cams) if c is camera))
        return orig_raster(cloud_, camera, *a, **k)

    def add_observer(self, norms, contributed):
        stats_obj[:] = [self]
        return orig_add(self, norms, contributed)

    pipeline.rasterize_forward = raster_observer
    adaptive.ViewspaceStats.add = add_observer
    try:
        record, transformed, summary = pipeline.process_frame(rb.ref_cloud(R, cloud), cache, views,
                                                              cfg, frame_index)
    finally:
        pipeline.rasterize_forward = orig_raster
        adaptive.ViewspaceStats.add = orig_add
    it = cfg.stage1_iterations
    order = np.array(seen[:it])  # then the train-PSNR renders of every view
    st = stats_obj[0]
    np.savez_compressed(os.path.join(OUT, "stage1_loop.npz"), **_cloud_arr(cloud), **_grid_arr(grid),
                        tables=tables, **{f"mlp_w{i}": w for i, w in enumerate(mlp["weights"])},
                        **{f"mlp_b{i}": b for i, b in enumerate(mlp["biases"])},
                        **{k: v for i, c in enumerate(sc.cameras) for k, v in _cam_arr(c, f"cam{i}_").items()},
                        **{f"target{i}": t for i, t in enumerate(targets)},
                        n_views=len(cams), iterations=it, seed=cfg.seed, frame_index=frame_index,
                        view_order=order, losses=np.array(summary.stage1_losses),
                        stats_norm=st.norm_accum, stats_count=st.view_count,
                        ntc_blob=np.frombuffer(record.ntc_blob, dtype=np.uint8),
                        out_means=transformed.means, out_rotations=transformed.rotations,
                        out_sh=transformed.sh)


def gen_stream(R):
    """A .splv container written by the reference's StreamWriter
    (streamio.py:185-226): HEAD, INIT, WARM and two FREC blocks."""
    import sys
    import tempfile

    if rb.REF_SRC not in sys.path:
        sys.path.insert(0, rb.REF_SRC)
    from splatstream import streamio

    from oracle import stage1 as O

    sc = scenes.small_scene(seed=41, n=50, width=32, height=24, sh_degree=1, n_views=1)
    grid = dict(sc.grid, levels=2, log2_table=6)
    tables, mlp = O.init_ntc(grid, hidden_dim=8, hidden_layers=1, output_init="random", seed=3)
    warm = rb.ref_cache(R, grid, scenes.f32(tables), mlp, hidden_dim=8)
    warm.quantize_float32()
    adds = [scenes.make_cloud(np.random.default_rng(60 + k), 3 + 4 * k, 2, 1.0, 0.3, 1)
            for k in range(2)]
    blobs = []
    for k in range(2):
        c = rb.ref_cache(R, grid, scenes.f32(tables + 0.01 * (k + 1)), mlp, hidden_dim=8)
        c.quantize_float32()
        blobs.append(streamio.serialize_ntc(c))
    header = {"format": "splv", "cameras": [{"width": 32, "height": 24}], "fps": 30}
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "s.splv")
        with streamio.StreamWriter(path, header) as w:
            w.write_initial(rb.ref_cloud(R, sc.cloud))
            w.write_warmup(warm)
            for k in range(2):
                w.write_frame(streamio.FrameRecord(k + 1, blobs[k], rb.ref_cloud(R, adds[k])))
        data = open(path, "rb").read()
    np.savez_compressed(os.path.join(OUT, "stream.npz"), container=np.frombuffer(data, np.uint8),
                        header=json_bytes(header), **_cloud_arr(sc.cloud, "init_"),
                        warm_blob=np.frombuffer(streamio.serialize_ntc(warm), np.uint8),
                        **{f"blob{k}": np.frombuffer(b, np.uint8) for k, b in enumerate(blobs)},
                        **{k2: v for k, a in enumerate(adds) for k2, v in _cloud_arr(a, f"add{k}_").items()})


def json_bytes(obj):
    import json

    return np.frombuffer(json.dumps(obj).encode(), np.uint8)


GENERATORS = dict(encode=gen_encode, ntc=gen_ntc, transform=gen_transform, raster=gen_raster,
                  loss=gen_loss, stage1=gen_stage1, ntc_blob=gen_ntc_blob, warmup=gen_warmup, playback=gen_playback,
                  stage2=gen_stage2, stage1_loop=gen_stage1_loop, stream=gen_stream)


def main():
    import sys

    os.makedirs(OUT, exist_ok=True)
    R = rb.load()
    which = sys.argv[1:] or list(GENERATORS)
    with threadpool_limits(1):
        for name in which:
            GENERATORS[name](R)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
