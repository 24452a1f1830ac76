"""CUDA path vs the reference golden vectors and the CPU oracle (needs a B200).

Tolerances (BASELINE.json north_star): hash indices, tile lists, sort order
bit-exact; images max-abs <= 1e-4; gradients norm-relative <= 1e-3.
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
    import paper_2403_01444_b200 as pkg
    from paper_2403_01444_b200 import _lib, losses, ntc, rasterizer, transform, types

    _lib.load()
    return dict(pkg=pkg, ntc=ntc, rasterizer=rasterizer, transform=transform, losses=losses,
                types=types, torch=torch)


def _cache(P, d, hidden=64):
    grid = P["types"].HashGridConfig.from_any(G.grid(d))
    mlp = G.mlp(d)
    c = P["ntc"].NeuralTransformationCache(grid, hidden_layers=len(mlp["weights"]) - 1,
                                           hidden_dim=hidden, output_init="random")
    c.tables[:] = d["tables"]
    for i in range(len(mlp["weights"])):
        c.weights[i][:] = mlp["weights"][i]
        c.biases[i][:] = mlp["biases"][i]
    return c


@pytest.mark.parametrize("tag", ["small", "cfg1"])
def test_encode_indices_bit_exact(P, tag):
    d = G.load(f"encode_{tag}")
    grid = P["types"].HashGridConfig.from_any(G.grid(d))
    c = P["ntc"].NeuralTransformationCache(grid, hidden_layers=2, hidden_dim=64)
    if "tables" in d:
        c.tables[:] = d["tables"]
    feats, ctx = c.encode(d["x"])
    np.testing.assert_array_equal(ctx.corner_idx, d["idx"])
    np.testing.assert_allclose(ctx.corner_w, d["w"], rtol=0, atol=2e-7)
    if "feats" in d:
        np.testing.assert_allclose(feats, d["feats"], rtol=1e-5, atol=1e-9)
    _, _, touched = O.encode(G.grid(d), d["x"])
    for l in range(grid.n_levels):
        np.testing.assert_array_equal(ctx.touched[l], touched[l])


def test_encode_outside_raises(P):
    d = G.load("encode_small")
    grid = P["types"].HashGridConfig.from_any(G.grid(d))
    c = P["ntc"].NeuralTransformationCache(grid)
    with pytest.raises(P["pkg"].DataError):
        c.encode(np.array([[5.0, 0.0, 0.0]]))


def test_ntc_forward_backward_golden(P):
    d = G.load("ntc")
    c = _cache(P, d)
    d_mu, d_q, ctx = c.forward(d["x"])
    np.testing.assert_allclose(d_mu, d["d_mu"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(d_q, d["d_q"], rtol=1e-4, atol=1e-6)
    grads, touched = c.backward(ctx, d["g_mu"], d["g_q"])
    for k in grads:
        assert G.norm_rel(grads[k], d[f"grad_{k}"]) <= GRAD_TOL, k
    for k in touched:
        np.testing.assert_array_equal(touched[k], d[f"touched_{k}"])


def test_transform_golden(P):
    d = G.load("transform")
    c = _cache(P, d)
    cloud = P["types"].GaussianCloud(**G.cloud(d))
    out, ctx = P["transform"].apply_ntc(cloud, c)
    np.testing.assert_array_equal(ctx.inside, d["inside"])
    np.testing.assert_allclose(out.means, d["out_means"], atol=1e-5)
    np.testing.assert_allclose(out.rotations, d["out_rotations"], atol=1e-5)
    np.testing.assert_allclose(out.sh, d["out_sh"], atol=1e-5)
    grads, _ = P["transform"].apply_ntc_backward(ctx, d["g_means"], d["g_rot"], d["g_sh"])
    for k in grads:
        assert G.norm_rel(grads[k], d[f"grad_{k}"]) <= GRAD_TOL, k


@pytest.mark.parametrize("tag", ["default", "smooth"])
def test_raster_golden(P, tag):
    d = G.load(f"raster_{tag}")
    R, T = P["rasterizer"], P["types"]
    cloud = T.GaussianCloud(**G.cloud(d))
    cam = T.Camera.from_any(G.camera(d))
    s = T.RasterSettings(**G.settings(d))
    out, ctx = R.rasterize_forward(cloud, cam, d["bg"], s)
    np.testing.assert_array_equal(ctx.indices, d["indices"])
    tiles = ctx.tiles
    np.testing.assert_array_equal(np.array([t[:4] for t in tiles]).reshape(-1, 4), d["tile_rects"])
    np.testing.assert_array_equal([len(t[4]) for t in tiles], d["tile_counts"])
    np.testing.assert_array_equal(np.concatenate([t[4] for t in tiles]), d["tile_members"])
    assert np.abs(out.image - d["image"]).max() <= IMG_TOL
    assert np.abs(out.alpha_map - d["alpha"]).max() <= IMG_TOL
    # the touch-count path runs every pair in float64 like the reference
    if s.skip_alpha > 0:
        np.testing.assert_array_equal(out.per_gaussian_touch_count, d["touch"])
    else:
        # skip_alpha = 0 also counts weights at the bottom of the denormal range
        # (~2^-1074), where a 1-ulp difference between CUDA's and glibc's exp
        # decides zero or not: a few pixels per Gaussian
        assert np.abs(out.per_gaussian_touch_count - d["touch"]).max() <= 4
    g = R.rasterize_backward(ctx, d["d_image"])
    for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
        assert G.norm_rel(getattr(g, k), d[k]) <= GRAD_TOL, k
    assert G.norm_rel(g.viewspace_grad_norm, d["viewspace"]) <= GRAD_TOL
    np.testing.assert_array_equal(g.contributed, d["contributed"])


def test_tile_bin_matches_reference_lists(P):
    d = G.load("raster_default")
    cloud = G.cloud(d)
    cam = G.camera(d)
    pj = O.project(cloud, cam)
    s = G.settings(d)
    tiles = P["rasterizer"].tile_bin(pj["mean2d"], pj["cov2d"], pj["opacity"], cam["width"],
                                     cam["height"], s["tile_size"], s["skip_alpha"])
    np.testing.assert_array_equal(np.concatenate([t[4] for t in tiles]), d["tile_members"])
    np.testing.assert_array_equal(np.array([t[:4] for t in tiles]).reshape(-1, 4), d["tile_rects"])


@pytest.mark.parametrize("n,ts", [(120_001, 16), (50_003, 8)])
def test_tile_bin_large_random_vs_oracle(P, n, ts):
    """Tile binning of many projected splats against the oracle, bit-exact:
    the rank kernel's single-pass scan across hundreds of look-back blocks,
    runs of zero-pair (off-screen) ranks, a few screen-filling splats, pair
    counts that are not multiples of the ranges kernel's four keys per thread
    (rasterizer.py:107-175)."""
    rng = np.random.default_rng(n)
    W, H = 333, 250
    mean2d = np.stack([rng.uniform(-80, W + 80, n), rng.uniform(-80, H + 80, n)], 1)
    sx, sy = rng.uniform(0.3, 12.0, n), rng.uniform(0.3, 12.0, n)
    sx[:5] = sy[:5] = 400.0  # screen-filling
    rho = rng.uniform(-0.6, 0.6, n) * sx * sy
    cov2d = np.zeros((n, 2, 2))
    cov2d[:, 0, 0], cov2d[:, 1, 1] = sx * sx, sy * sy
    cov2d[:, 0, 1] = cov2d[:, 1, 0] = rho
    opacity = rng.uniform(0.01, 0.99, n)
    skip = 1.0 / 255.0
    tiles = P["rasterizer"].tile_bin(mean2d, cov2d, opacity, W, H, ts, skip)
    ref = O.tile_lists(mean2d, cov2d, opacity, W, H, ts, skip)
    assert len(tiles) == len(ref)
    np.testing.assert_array_equal(np.array([t[:4] for t in tiles]),
                                  np.array([t[:4] for t in ref]))
    np.testing.assert_array_equal(np.concatenate([t[4] for t in tiles]),
                                  np.concatenate([t[4] for t in ref]))


def test_render_loss_golden(P):
    d = G.load("loss")
    loss, grad = P["losses"].render_loss(d["x"], d["y"])
    assert abs(loss - float(d["loss"])) <= 1e-6
    assert G.norm_rel(grad, d["grad"]) <= 1e-4
    assert np.abs(grad - d["grad"]).max() <= 1e-7


def test_stage1_golden_two_iterations(P):
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    d = G.load("stage1")
    c = _cache(P, d)
    cams = [G.camera(d, "cam0_"), G.camera(d, "cam1_")]
    views = [(cams[0], d["target0"]), (cams[1], d["target1"])]
    tr = Stage1Trainer(G.cloud(d), c, views, Stage1Config(stage1_iterations=2))
    pairs = tr.begin(0)
    tr.finish(0, pairs, adam=False)
    assert np.abs(tr.rendered_image(0) - d["image_first"]).max() <= IMG_TOL
    l0 = tr.last_loss()
    assert abs(l0 - d["losses"][0]) <= 1e-5 * abs(d["losses"][0]) + 1e-7
    gt, gw, gb = tr.ntc_grads()
    for l in range(gt.shape[0]):
        assert G.norm_rel(gt[l], d[f"grad1_table_{l}"]) <= GRAD_TOL, l
    for i in range(3):
        assert G.norm_rel(gw[i], d[f"grad1_w_{i}"]) <= GRAD_TOL, i
        assert G.norm_rel(gb[i], d[f"grad1_b_{i}"]) <= GRAD_TOL, i
    tr.apply_adam()
    tr.step(1)
    l1 = tr.last_loss()
    assert abs(l1 - d["losses"][1]) <= 1e-3 * abs(d["losses"][1])


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_raster_random_scenes_vs_oracle(P, deg):
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=30 + deg, n=800, width=80, height=64, sh_degree=deg)
    R, T = P["rasterizer"], P["types"]
    cam = sc.cameras[1]
    bg = np.array([0.2, 0.1, 0.3])
    ref, rctx = O.render(sc.cloud, cam, bg)
    out, ctx = R.rasterize_forward(T.GaussianCloud(**sc.cloud), T.Camera.from_any(cam), bg)
    assert np.abs(out.image - ref["image"]).max() <= IMG_TOL
    np.testing.assert_array_equal(ctx.indices, rctx["proj"]["indices"])
    mem = np.concatenate([t[4] for t in ctx.tiles])
    np.testing.assert_array_equal(mem, np.concatenate([t[4] for t in rctx["tiles"]]))
    d_img = np.random.default_rng(deg).normal(size=out.image.shape)
    g = R.rasterize_backward(ctx, d_img)
    rg = O.render_backward(rctx, d_img)
    for k, rk in (("d_means", "d_means"), ("d_rotations", "d_rotations"),
                  ("d_log_scales", "d_log_scales"), ("d_opacity_logits", "d_opacity_logits"),
                  ("d_sh", "d_sh")):
        assert G.norm_rel(getattr(g, k), rg[rk]) <= GRAD_TOL, k


@pytest.mark.parametrize("case", ["mostly_offscreen", "huge_splats"])
def test_raster_adversarial_scenes_vs_oracle(P, case):
    """Pair-generation corner cases against the oracle: most Gaussians in front
    of the camera but off-screen, with zero tile pairs interleaved in depth
    order (a 1024-pair duplicate chunk then spans more ranks than its staged
    offsets hold), and a few near-camera splats covering every tile next to
    many small ones (long per-rank pair runs)."""
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=77, n=6000, width=96, height=72, sh_degree=1)
    cloud = {k: np.array(v, copy=True) for k, v in sc.cloud.items()}
    rng = np.random.default_rng(5)
    if case == "mostly_offscreen":
        far = rng.random(len(cloud["means"])) < 0.9
        cloud["means"][far, 0] += 60.0
    else:
        big = rng.choice(len(cloud["means"]), 8, replace=False)
        cloud["log_scales"][big] = np.log(3.0)
    # both sides see the same fp32-lattice values
    cloud = {k: v.astype(np.float32).astype(np.float64) for k, v in cloud.items()}
    R, T = P["rasterizer"], P["types"]
    cam = sc.cameras[0]
    bg = np.array([0.1, 0.2, 0.3])
    ref, rctx = O.render(cloud, cam, bg)
    out, ctx = R.rasterize_forward(T.GaussianCloud(**cloud), T.Camera.from_any(cam), bg)
    assert np.abs(out.image - ref["image"]).max() <= IMG_TOL
    np.testing.assert_array_equal(ctx.indices, rctx["proj"]["indices"])
    mem = np.concatenate([t[4] for t in ctx.tiles])
    np.testing.assert_array_equal(mem, np.concatenate([t[4] for t in rctx["tiles"]]))
    d_img = np.random.default_rng(1).normal(size=out.image.shape)
    g = R.rasterize_backward(ctx, d_img)
    rg = O.render_backward(rctx, d_img)
    for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
        assert G.norm_rel(getattr(g, k), rg[k]) <= GRAD_TOL, k


def test_stage1_cfg0_single_step_vs_oracle(P):
    """The parity config (BASELINE configs[0]): one full Stage-1 step, fp32."""
    from paper_2403_01444_b200 import scenes
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    sc = scenes.config(0)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=2)
    tables = scenes.f32(np.random.default_rng(3).uniform(-0.02, 0.02, size=tables.shape))
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(1))
    targets = [O.render(moved, c)[0]["image"] for c in sc.cameras]

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    c = Cache()
    c.tables, c.weights, c.biases = tables, mlp["weights"], mlp["biases"]
    tr = Stage1Trainer(sc.cloud, c, list(zip(sc.cameras, targets)), Stage1Config())
    pairs = tr.begin(0)
    tr.finish(0, pairs, adam=False)
    state = dict(grid=sc.grid, tables=tables.copy(), mlp=mlp,
                 inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    ref = O.stage1_iteration(state, sc.cloud, sc.cameras[0], targets[0], apply_adam=False)
    assert np.abs(tr.rendered_image(0) - ref["image"]).max() <= IMG_TOL
    assert abs(tr.last_loss() - ref["loss"]) <= 1e-5 * ref["loss"]
    gt, gw, gb = tr.ntc_grads()
    assert G.norm_rel(gt, ref["g_tables"]) <= GRAD_TOL
    for i in range(3):
        assert G.norm_rel(gw[i], ref["g_w"][i]) <= GRAD_TOL
        assert G.norm_rel(gb[i], ref["g_b"][i]) <= GRAD_TOL


def test_stage1_no_sync_matches_synchronised_path(P):
    """ss_stage1_iter (device-side pair count, capacity-bounded binning, no
    host synchronisation) reproduces the begin/finish path: the first
    iteration bit for bit, later ones up to the float-atomic accumulation
    order of the gradients; and run()'s replay after a capacity overflow
    restores the same trajectory."""
    import torch

    from paper_2403_01444_b200 import scenes
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer
    from oracle import stage1 as O

    sc = scenes.small_scene(seed=11, n=3000, width=96, height=72, sh_degree=1, n_views=3)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=2)
    tables = scenes.f32(np.random.default_rng(4).uniform(-0.05, 0.05, size=tables.shape))
    targets = [O.render(scenes.moved_cloud(sc.cloud, np.random.default_rng(9)), c)[0]["image"]
               for c in sc.cameras]

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    def trainer():
        c = Cache()
        c.tables, c.weights, c.biases = tables.copy(), mlp["weights"], mlp["biases"]
        return Stage1Trainer(sc.cloud, c, list(zip(sc.cameras, targets)),
                             Stage1Config(stage1_iterations=6))

    def close(x, y):
        return torch.allclose(x, y, rtol=1e-4, atol=1e-7)

    views = [0, 1, 2, 1, 0, 2]
    a, b = trainer(), trainer()
    p0 = a.begin(0)
    a.finish(0, p0, adam=False)
    b.iterate(0, adam=False)
    torch.cuda.synchronize()
    assert torch.equal(a.image, b.image)
    # the loss sums are fp64 atomics: equal up to their accumulation order
    assert abs(a.last_loss() - b.last_loss()) <= 1e-12 * abs(a.last_loss())
    assert int(b.pairs_of_last(1)[0]) == p0
    a.apply_adam()
    b.apply_adam()
    ref_losses, ref_pairs = [], []
    for v in views[1:]:
        p = a.begin(v)
        a.finish(v, p)
        ref_losses.append(a.last_loss())
        ref_pairs.append(p)
    for v in views[1:]:
        b.iterate(v)
    torch.cuda.synchronize()
    assert b.check_status() == 0
    np.testing.assert_allclose(b.pairs_of_last(5), ref_pairs, rtol=1e-3)
    # later steps differ only by float-atomic accumulation order
    np.testing.assert_allclose(b.loss_hist[1:6].cpu().numpy(), ref_losses, rtol=1e-4)
    assert close(a.tables, b.tables) and close(a.params, b.params)
    # run() with a deliberately tiny workspace: overflow -> replay with a larger one
    c, d = trainer(), trainer()
    la = c.run(6)
    d.plan_capacity(margin=0.2)
    lb = d.run(6)
    np.testing.assert_allclose(la[0], lb[0], rtol=1e-12)
    np.testing.assert_allclose(la, lb, rtol=1e-4)  # float-atomic order after step 0
    # Adam (eps 1e-15) turns accumulation-order noise in near-zero gradients
    # into full-size steps of either sign on a few entries: compare in norm
    def rel(x, y):
        return float(torch.linalg.norm(x - y) / torch.linalg.norm(y))

    assert rel(c.tables, d.tables) <= 1e-3 and rel(c.params, d.params) <= 1e-3


@pytest.mark.parametrize("deg", [1, 3])
def test_tile_cull_render_identical(P, deg):
    """The Stage-1 render path drops (splat, tile) pairs whose fp64 alpha bound
    stays below skip_alpha over the whole tile; the image must be bit-identical
    to the full reference tile lists (public rasterize_forward path)."""
    import torch

    from paper_2403_01444_b200 import scenes
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer
    from oracle import stage1 as O

    sc = scenes.small_scene(seed=40 + deg, n=4000, width=160, height=120, sh_degree=deg,
                            n_views=2)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=3)

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    c = Cache()
    c.tables, c.weights, c.biases = tables, mlp["weights"], mlp["biases"]
    views = [(cam, np.zeros((cam["height"], cam["width"], 3))) for cam in sc.cameras]
    tr = Stage1Trainer(sc.cloud, c, views, Stage1Config())
    for v in range(2):
        tr.render(v)  # full lists
        full = tr.image.clone()
        tr.render_async(v)  # culled lists
        torch.cuda.synchronize()
        assert torch.equal(full, tr.image)


def test_run_from_host_matches_resident_targets(P):
    """run_from_host (pinned host targets, copy-stream H2D overlapped with the
    previous iteration, async loss D2H) == iterating on resident targets."""
    import torch

    from paper_2403_01444_b200 import scenes
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer
    from oracle import stage1 as O

    sc = scenes.small_scene(seed=12, n=2500, width=96, height=72, sh_degree=1, n_views=3)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=5)
    targets = [O.render(scenes.moved_cloud(sc.cloud, np.random.default_rng(3)), c)[0]["image"]
               for c in sc.cameras]

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    def trainer():
        c = Cache()
        c.tables, c.weights, c.biases = tables.copy(), mlp["weights"], mlp["biases"]
        return Stage1Trainer(sc.cloud, c, list(zip(sc.cameras, targets)),
                             Stage1Config(stage1_iterations=8))

    order = [0, 2, 1, 1, 0, 2, 2, 0]
    a, b = trainer(), trainer()
    ref = []
    for v in order:
        a.iterate(v)
        ref.append(a.last_loss())
    host = [torch.tensor(t, dtype=torch.float32).pin_memory() for t in targets]
    got = b.run_from_host(order, host)
    # first step identical; later ones differ only by float-atomic order, which
    # Adam (eps 1e-15) amplifies on near-zero gradients: ~2e-5 after 8 steps
    np.testing.assert_allclose(got[0], ref[0], rtol=1e-12)
    np.testing.assert_allclose(got, ref, rtol=1e-4)


def test_stage1_trajectory_vs_oracle(P):
    """Ten Stage-1 iterations with Adam (identity-initialised NTC, as bench.py
    trains) follow the float64 oracle's loss trajectory and parameters."""
    import torch

    from paper_2403_01444_b200 import scenes
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer
    from oracle import stage1 as O

    sc = scenes.small_scene(seed=21, n=1500, width=80, height=64, sh_degree=1, n_views=2)
    tables, mlp = O.init_ntc(sc.grid, output_init="identity", seed=0)
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(7))
    targets = [O.render(moved, c)[0]["image"] for c in sc.cameras]

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    c = Cache()
    c.tables = tables.copy()
    c.weights = [w.copy() for w in mlp["weights"]]
    c.biases = [b.copy() for b in mlp["biases"]]
    tr = Stage1Trainer(sc.cloud, c, list(zip(sc.cameras, targets)),
                       Stage1Config(stage1_iterations=10))
    state = dict(grid=sc.grid, tables=tables.copy(),
                 mlp=dict(weights=[w.copy() for w in mlp["weights"]],
                          biases=[b.copy() for b in mlp["biases"]]),
                 inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    order = [0, 1, 1, 0, 1, 0, 0, 1, 1, 0]
    ref = [O.stage1_iteration(state, sc.cloud, sc.cameras[v], targets[v])["loss"] for v in order]
    for v in order:
        tr.iterate(v)
    torch.cuda.synchronize()
    got = tr.loss_hist[:10].cpu().numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-3)
    # parameters after 10 Adam steps: eps = 1e-15 turns round-off-level
    # gradients of touched rows into full-size steps of either sign (SURVEY.md
    # D10), so the trajectory is graded at 1e-2 (single-step gradients at 1e-3
    # elsewhere)
    tab = tr.tables.view(state["tables"].shape).cpu().numpy()
    assert G.norm_rel(tab, state["tables"]) <= 1e-2
