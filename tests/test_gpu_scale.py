"""Parity at the BASELINE configurations' own scale (needs a B200).

The inputs are exactly the seeded workloads bench.py times (scenes.config(1):
250k SH-3 Gaussians, twenty 1352x1014 views; scenes.config(2): 300k).  At this
scale the float64 reference floors hash positions, bins tile rectangles and
lexsorts depths in ways fp32 arithmetic would not reproduce (
ntc.py:176-180, rasterizer.py:132-148, :228-230), so these are the tests with
the power to catch that class of bug:
  * corner indices of every mean at all 16 levels, bit-exact (ntc.py:161-203);
  * survivor order and the complete tile lists (rects, counts, members) of
    three full views, including the view with the most pairs, bit-exact
    (rasterizer.py:107-175, :227-230);
  * image (max-abs <= 1e-4) and every render gradient (norm-relative <= 1e-3)
    on two 32-row bands, the camera's principal point shifted as bench.py's
    CPU sample does (rasterizer.py:214-402);
  * one full Stage-1 step at cfg1 on a band, and one on the full 1352x1014
    view against the all-core oracle port (pipeline.py:263-277);
  * a full cfg2 frame through the benchmarked render path;
  * config 3's batched 4-view step at 1M Gaussians (view bands).
"""

import numpy as np
import pytest

import golden_io as G
from oracle import stage1 as O

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def P():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import _lib, ntc, rasterizer, scenes, types

    _lib.load()
    return dict(ntc=ntc, rasterizer=rasterizer, types=types, scenes=scenes, torch=torch)


_SCENES = {}


def scene(P, idx):
    if idx not in _SCENES:
        _SCENES[idx] = P["scenes"].config(idx)
    return _SCENES[idx]


def band(cam, y0, rows=32):
    """The rows [y0, y0 + rows) of `cam` as a camera of its own (cy shifted)."""
    return dict(cam, height=rows, cy=cam["cy"] - y0)


@pytest.mark.parametrize("cfg", [1, 2])
def test_encode_every_mean_bit_exact(P, cfg):
    sc = scene(P, cfg)
    grid = P["types"].HashGridConfig.from_any(sc.grid)
    c = P["ntc"].NeuralTransformationCache(grid, hidden_layers=2, hidden_dim=64)
    means = sc.cloud["means"]
    _, ctx = c.encode(means)
    idx, w, touched = O.encode(sc.grid, means)
    assert ctx.corner_idx.shape == (len(means), 16, 8)
    np.testing.assert_array_equal(ctx.corner_idx, idx)
    np.testing.assert_allclose(ctx.corner_w, w, rtol=0, atol=2e-7)
    for l in range(grid.n_levels):
        np.testing.assert_array_equal(ctx.touched[l], touched[l])


def _pair_counts(P, sc):
    R, T = P["rasterizer"], P["types"]
    cloud = T.GaussianCloud(**sc.cloud)
    return [R.rasterize_forward(cloud, T.Camera.from_any(c))[1].n_pairs for c in sc.cameras]


@pytest.mark.parametrize("cfg", [1, 2])
def test_full_view_order_and_tile_lists_bit_exact(P, cfg):
    sc = scene(P, cfg)
    R, T = P["rasterizer"], P["types"]
    cloud = T.GaussianCloud(**sc.cloud)
    counts = _pair_counts(P, sc)
    views = sorted({int(np.argmax(counts)), 0, len(sc.cameras) // 2})
    s = O.DEFAULT_SETTINGS
    for v in views:
        cam = sc.cameras[v]
        out, ctx = R.rasterize_forward(cloud, T.Camera.from_any(cam))
        pj = O.project(sc.cloud, cam)
        np.testing.assert_array_equal(ctx.indices, pj["indices"])
        ref = O.tile_lists(pj["mean2d"], pj["cov2d"], pj["opacity"], cam["width"],
                           cam["height"], s["tile_size"], s["skip_alpha"])
        got = ctx.tiles
        assert ctx.n_pairs == sum(len(t[4]) for t in ref)
        np.testing.assert_array_equal(np.array([t[:4] for t in got]),
                                      np.array([t[:4] for t in ref]))
        np.testing.assert_array_equal([len(t[4]) for t in got], [len(t[4]) for t in ref])
        np.testing.assert_array_equal(np.concatenate([t[4] for t in got]),
                                      np.concatenate([t[4] for t in ref]))


@pytest.mark.parametrize("cfg", [1, 2])
def test_banded_image_and_gradients(P, cfg):
    sc = scene(P, cfg)
    R, T = P["rasterizer"], P["types"]
    cloud = T.GaussianCloud(**sc.cloud)
    counts = _pair_counts(P, sc)
    v = int(np.argmax(counts))
    rng = np.random.default_rng(cfg)
    bg = np.array([0.05, 0.1, 0.15])
    for y0 in (240, 496):  # tile-aligned rows of the full frame
        cam = band(sc.cameras[v], y0)
        ref, rctx = O.render(sc.cloud, cam, bg)
        out, ctx = R.rasterize_forward(cloud, T.Camera.from_any(cam), bg)
        np.testing.assert_array_equal(ctx.indices, rctx["proj"]["indices"])
        np.testing.assert_array_equal(np.concatenate([t[4] for t in ctx.tiles]),
                                      np.concatenate([t[4] for t in rctx["tiles"]]))
        assert np.abs(out.image - ref["image"]).max() <= IMG_TOL
        assert np.abs(out.alpha_map - ref["alpha_map"]).max() <= IMG_TOL
        np.testing.assert_array_equal(out.per_gaussian_touch_count, ref["touch"])
        d_img = rng.normal(size=out.image.shape)
        g = R.rasterize_backward(ctx, d_img)
        rg = O.render_backward(rctx, d_img)
        for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
            assert G.norm_rel(getattr(g, k), rg[k]) <= GRAD_TOL, (y0, k)
        assert G.norm_rel(g.viewspace_grad_norm, rg["viewspace"]) <= GRAD_TOL
        np.testing.assert_array_equal(g.contributed, rg["contributed"])


def test_stage1_step_cfg1_band(P):
    """One Stage-1 iteration (apply_ntc -> render -> loss -> backward ->
    NTC gradients) of the 250k SH-3 cfg1 cloud on a 32-row band of the view
    with the most pairs; random-initialised NTC so every gradient is live."""
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    sc = scene(P, 1)
    scenes = P["scenes"]
    counts = _pair_counts(P, sc)
    cam = band(sc.cameras[int(np.argmax(counts))], 496)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=4)
    tables = scenes.f32(np.random.default_rng(6).uniform(-0.02, 0.02, size=tables.shape))
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(7), axis=(0.3, 1.0, 0.2),
                               deg=1.5, shift=(0.01, -0.005, 0.008))
    target = O.render(moved, cam)[0]["image"]

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    c = Cache()
    c.tables, c.weights, c.biases = tables, mlp["weights"], mlp["biases"]
    tr = Stage1Trainer(sc.cloud, c, [(cam, target)], Stage1Config(stage1_iterations=1))
    pairs = tr.begin(0)
    tr.finish(0, pairs, adam=False)
    state = dict(grid=sc.grid, tables=tables.copy(), mlp=mlp,
                 inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    ref = O.stage1_iteration(state, sc.cloud, cam, target, apply_adam=False)
    assert np.abs(tr.rendered_image(0) - ref["image"]).max() <= IMG_TOL
    assert abs(tr.last_loss() - ref["loss"]) <= 1e-5 * ref["loss"]
    gt, gw, gb = tr.ntc_grads()
    assert G.norm_rel(gt, ref["g_tables"]) <= GRAD_TOL
    for i in range(3):
        assert G.norm_rel(gw[i], ref["g_w"][i]) <= GRAD_TOL, i
        assert G.norm_rel(gb[i], ref["g_b"][i]) <= GRAD_TOL, i


@pytest.mark.parametrize("mlp_dtype", ["f32", "f16"])
def test_stage1_step_cfg1_full_height(P, mlp_dtype):
    """One FULL-HEIGHT Stage-1 iteration of the cfg1 workload (250k SH-3
    Gaussians, 1352x1014, the view bench.py's CPU sample times) against the
    float64 oracle port on every host core (oracle/parallel.py, itself pinned
    to the serial oracle by test_oracle_parallel.py): image, loss and the NTC
    gradients after the whole chain apply_ntc -> render -> loss -> backward ->
    apply_ntc_backward (pipeline.py:263-277).  fp32 cache (the reference's
    arithmetic) and the fp16-weight decoder BASELINE configs[1] specifies (the
    oracle's f16 restatement); random-initialised NTC so every gradient is live."""
    import os

    from threadpoolctl import threadpool_limits

    from oracle import parallel
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    sc = scene(P, 1)
    scenes = P["scenes"]
    cam = sc.cameras[0]
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=4)
    tables = scenes.f32(np.random.default_rng(6).uniform(-0.02, 0.02, size=tables.shape))
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(7), axis=(0.3, 1.0, 0.2),
                               deg=1.5, shift=(0.01, -0.005, 0.008))
    state = dict(grid=sc.grid, tables=tables.copy(), mlp=dict(mlp, dtype=mlp_dtype),
                 inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    state["enc"] = O.encode(sc.grid, sc.cloud["means"][state["inside"]])
    ps = parallel.ParallelStage1(os.cpu_count() or 1)
    with threadpool_limits(1):
        target = ps.render(moved, cam)
        ref = ps.iteration(state, sc.cloud, cam, target, apply_adam=False)

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    c = Cache()
    c.tables, c.weights, c.biases = tables, mlp["weights"], mlp["biases"]
    tr = Stage1Trainer(sc.cloud, c, [(cam, target.astype(np.float32))],
                       Stage1Config(stage1_iterations=1, mlp_dtype=mlp_dtype))
    assert tr.mlp.precision == (1 if mlp_dtype == "f16" else 0)
    pairs = tr.begin(0)
    tr.finish(0, pairs, adam=False)
    assert tr.check_status() == 0
    assert np.abs(tr.rendered_image(0) - ref["image"]).max() <= IMG_TOL
    assert abs(tr.last_loss() - ref["loss"]) <= 1e-5 * ref["loss"]
    gt, gw, gb = tr.ntc_grads()
    assert G.norm_rel(gt, ref["g_tables"]) <= GRAD_TOL
    for i in range(3):
        assert G.norm_rel(gw[i], ref["g_w"][i]) <= GRAD_TOL, i
        assert G.norm_rel(gb[i], ref["g_b"][i]) <= GRAD_TOL, i


@pytest.mark.parametrize("mlp_dtype", ["f32", "f16"])
def test_render_cfg2_full_frame(P, mlp_dtype):
    """The render FPS workload (config 2: NTC transform + rasterize_forward of
    300k SH-3 Gaussians at 1352x1014, the graph-replayed ss_stage1_render path
    bench.py times) on a full frame against the all-core float64 oracle port
    (transform.py:53-96 -> rasterizer.py:214-281); random-initialised NTC."""
    import os

    from threadpoolctl import threadpool_limits

    from oracle import parallel
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    sc = scene(P, 2)
    scenes = P["scenes"]
    cam = sc.cameras[3]
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=9)
    tables = scenes.f32(np.random.default_rng(10).uniform(-0.02, 0.02, size=tables.shape))
    state = dict(grid=sc.grid, tables=tables.copy(), mlp=dict(mlp, dtype=mlp_dtype),
                 inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    state["enc"] = O.encode(sc.grid, sc.cloud["means"][state["inside"]])
    ps = parallel.ParallelStage1(os.cpu_count() or 1)
    with threadpool_limits(1):
        ref = ps.transform_render(state, sc.cloud, cam)

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    c = Cache()
    c.tables, c.weights, c.biases = tables, mlp["weights"], mlp["biases"]
    tr = Stage1Trainer(sc.cloud, c, [(cam, np.zeros_like(ref, dtype=np.float32))],
                       Stage1Config(mlp_dtype=mlp_dtype))
    tr.render_async(0)  # captured
    tr.render_async(0)  # replayed
    P["torch"].cuda.synchronize()
    assert tr.check_status() == 0
    assert np.abs(tr.rendered_image(0) - ref).max() <= IMG_TOL


def test_batched_step_cfg3_bands(P):
    """Config 3's batched step at its own scale (1M SH-3 Gaussians, four of its
    hemisphere cameras, each on a 32-row band): ViewShardedStage1 accumulates
    the 1/B-scaled gradients of the four views and takes one lazy Adam step;
    the oracle takes the mean of the per-view reference gradients
    (transform.py:99-135 -> ntc.py:250-288) and one Adam step (optim.py:33-66),
    on every host core (oracle/parallel.py)."""
    import os

    from threadpoolctl import threadpool_limits

    from oracle import parallel
    from paper_2403_01444_b200.device import unpack_params
    from paper_2403_01444_b200.dist import ViewShardedStage1
    from paper_2403_01444_b200.stage1 import Stage1Config

    torch = P["torch"]
    sc = scene(P, 3)
    scenes = P["scenes"]
    cams = [band(sc.cameras[v], y0) for v, y0 in ((0, 500), (11, 300), (23, 700), (40, 100))]
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=12)
    tables = scenes.f32(np.random.default_rng(13).uniform(-0.02, 0.02, size=tables.shape))
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(7), axis=(0.3, 1.0, 0.2),
                               deg=1.5, shift=(0.01, -0.005, 0.008))
    st = dict(grid=sc.grid, tables=tables.copy(),
              mlp=dict(weights=[w.copy() for w in mlp["weights"]],
                       biases=[b.copy() for b in mlp["biases"]]),
              inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    st["enc"] = O.encode(sc.grid, sc.cloud["means"][st["inside"]])
    ps = parallel.ParallelStage1(os.cpu_count() or 1)
    with threadpool_limits(1):
        targets = [ps.render(moved, c) for c in cams]
        rs = [ps.iteration(st, sc.cloud, c, t, apply_adam=False) for c, t in zip(cams, targets)]

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    c = Cache()
    c.tables, c.weights, c.biases = tables.copy(), mlp["weights"], mlp["biases"]
    vs = ViewShardedStage1(sc.cloud, c, [(cm, t.astype(np.float32)) for cm, t in zip(cams, targets)],
                           Stage1Config(stage1_iterations=1), views_per_iteration=4)
    vs.step([0, 1, 2, 3])
    torch.cuda.synchronize()
    assert vs.trainer.check_status() == 0
    b = len(rs)
    O.adam_apply(st, sum(r["g_tables"] for r in rs) / b,
                 [sum(r["g_w"][i] for r in rs) / b for i in range(3)],
                 [sum(r["g_b"][i] for r in rs) / b for i in range(3)], 0.002)
    tab = vs.trainer.tables.view(st["tables"].shape).cpu().numpy()
    assert G.norm_rel(tab - tables, st["tables"] - tables) <= 1e-3
    ws, bs = unpack_params(vs.trainer.params.cpu().numpy(), vs.trainer.w_shapes,
                           vs.trainer.layout)
    for i in range(3):
        assert G.norm_rel(ws[i] - mlp["weights"][i],
                          st["mlp"]["weights"][i] - mlp["weights"][i]) <= 1e-3, i
        assert G.norm_rel(bs[i] - mlp["biases"][i],
                          st["mlp"]["biases"][i] - mlp["biases"][i]) <= 1e-3, i
    np.testing.assert_allclose(vs.batch_losses()[0], np.mean([r["loss"] for r in rs]), rtol=1e-5)
