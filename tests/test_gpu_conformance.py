"""The reference's own conformance tests, run against the CUDA path (needs a B200).

Restated from /root/reference/pkg/tests (their helpers are re-written here):
  * tile-size independence, 8/16/32 (+64)   test_rasterizer.py:122-132
  * input-order independence                  test_rasterizer.py:134-140
  * raster gradients vs central differences with SMOOTH (tile 64, no skip /
    early stop)                               test_rasterizer.py:20, :226-270
  * NTC gradients vs central differences       test_ntc.py:183-216
  * transform+cache gradients vs central differences  test_transform.py:174-215
The reference runs them in float64; the CUDA path computes in float32, so the
finite-difference steps and absolute tolerances are widened to the fp32 noise
floor of the forward (stated per test).  Plus the batched view-sharded step on
the device and an adversarial equal-depth cloud for
the depth tie-break (rasterizer.py:228-230).
"""

import time

import numpy as np
import pytest

import golden_io as G
from oracle import stage1 as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import _lib, ntc, rasterizer, scenes, transform, types

    _lib.load()
    return dict(ntc=ntc, rasterizer=rasterizer, types=types, scenes=scenes, transform=transform,
                torch=torch)


def _make_camera(T, width=32, height=32, fx=40.0, fy=40.0):
    """test_rasterizer.py:23-32: identity pose."""
    return T.Camera(world_to_camera=np.eye(4), fx=fx, fy=fy, cx=(width - 1) / 2.0,
                    cy=(height - 1) / 2.0, width=width, height=height)


def _random_scene(T, rng, n=5, opacity_hi=0.85):
    """test_rasterizer.py:35-49 (values rounded onto the fp32 lattice)."""
    means = rng.uniform(-0.5, 0.5, size=(n, 3))
    means[:, 2] = rng.uniform(2.0, 4.0, size=n)
    sh = np.zeros((n, 4, 3))
    sh[:, 0, :] = rng.uniform(-0.8, 0.8, size=(n, 3))
    sh[:, 1:, :] = rng.normal(scale=0.08, size=(n, 3, 3))
    op = rng.uniform(0.3, opacity_hi, size=n)
    c = T.GaussianCloud(means=means, rotations=rng.normal(size=(n, 4)),
                        log_scales=rng.uniform(np.log(0.05), np.log(0.25), size=(n, 3)),
                        opacity_logits=np.log(op / (1 - op)), sh=sh)
    return c.quantize_float32()


def _cloud_dict(c):
    return dict(means=c.means, rotations=c.rotations, log_scales=c.log_scales,
                opacity_logits=c.opacity_logits, sh=c.sh)


def _cam_dict(cam):
    return dict(w2c=np.asarray(cam.world_to_camera), fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy,
                width=cam.width, height=cam.height, near=cam.near_clip)


# ---------------------------------------------------------------- rasterizer
@pytest.mark.parametrize("ts", [8, 16, 32, 64])
def test_tile_size_matches_oracle_and_is_independent(P, ts):
    """Every dispatched tile size against the oracle at that size (lists
    bit-exact, image, gradients), and the image equals the 16-px one."""
    R, T = P["rasterizer"], P["types"]
    sc = P["scenes"].small_scene(seed=60, n=3000, width=96, height=72, sh_degree=1)
    cloud, cam = T.GaussianCloud(**sc.cloud), sc.cameras[0]
    bg = np.array([0.1, 0.3, 0.2])
    s = T.RasterSettings(tile_size=ts)
    out, ctx = R.rasterize_forward(cloud, T.Camera.from_any(cam), bg, s)
    ref, rctx = O.render(sc.cloud, cam, bg, dict(tile_size=ts))
    np.testing.assert_array_equal(np.array([t[:4] for t in ctx.tiles]),
                                  np.array([t[:4] for t in rctx["tiles"]]))
    np.testing.assert_array_equal(np.concatenate([t[4] for t in ctx.tiles]),
                                  np.concatenate([t[4] for t in rctx["tiles"]]))
    assert np.abs(out.image - ref["image"]).max() <= 1e-4
    np.testing.assert_array_equal(out.per_gaussian_touch_count, ref["touch"])
    d_img = np.random.default_rng(ts).normal(size=out.image.shape)
    g = R.rasterize_backward(ctx, d_img)
    rg = O.render_backward(rctx, d_img)
    for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
        assert G.norm_rel(getattr(g, k), rg[k]) <= 1e-3, k
    out16, _ = R.rasterize_forward(cloud, T.Camera.from_any(cam), bg, T.RasterSettings())
    assert np.abs(out.image - out16.image).max() <= 1e-5


def test_tile_size_independence_reference_case(P, rng):
    """test_rasterizer.py:122-132 verbatim in shape: 8 Gaussians, 48x48."""
    R, T = P["rasterizer"], P["types"]
    cam = _make_camera(T, 48, 48, 60.0, 60.0)
    cloud = _random_scene(T, rng, n=8)
    imgs = [R.rasterize_forward(cloud, cam, np.zeros(3), T.RasterSettings(tile_size=ts))[0].image
            for ts in (8, 16, 32, 64)]
    for a in imgs[1:]:
        np.testing.assert_allclose(imgs[0], a, atol=1e-6)  # reference tolerance


def test_input_order_irrelevant(P, rng):
    """test_rasterizer.py:134-140, and at scale: the survivor order maps
    through the permutation."""
    R, T = P["rasterizer"], P["types"]
    cam = _make_camera(T)
    cloud = _random_scene(T, rng, n=6)
    out1, _ = R.rasterize_forward(cloud, cam, np.zeros(3))
    perm = rng.permutation(6)
    out2, _ = R.rasterize_forward(cloud.select(perm), cam, np.zeros(3))
    np.testing.assert_allclose(out1.image, out2.image, atol=1e-6)
    sc = P["scenes"].small_scene(seed=61, n=5000, width=96, height=72, sh_degree=1)
    big = T.GaussianCloud(**sc.cloud)
    perm = np.random.default_rng(3).permutation(len(big))
    a, ca = R.rasterize_forward(big, T.Camera.from_any(sc.cameras[1]))
    b, cb = R.rasterize_forward(big.select(perm), T.Camera.from_any(sc.cameras[1]))
    np.testing.assert_array_equal(perm[cb.indices], ca.indices)
    np.testing.assert_array_equal(a.image, b.image)


def test_raster_gradients_match_finite_differences(P, rng):
    """test_rasterizer.py:226-270 with SMOOTH (tile 64, skip_alpha 0, no early
    stop), every parameter of a 5-Gaussian 32x32 scene.  fp32 forward: step
    2e-3 (on the fp32 lattice, the actual perturbation is used) and an
    absolute floor of 2e-3 of the largest gradient of the array."""
    R, T = P["rasterizer"], P["types"]
    cam = _make_camera(T)
    cloud = _random_scene(T, rng, n=5)
    bg = np.array([0.3, 0.2, 0.4])
    w = rng.normal(size=(32, 32, 3))
    smooth = T.RasterSettings(tile_size=64, skip_alpha=0.0, stop_transmittance=0.0)

    def loss(c):
        return float(np.sum(w * R.rasterize_forward(c, cam, bg, smooth)[0].image))

    _, ctx = R.rasterize_forward(cloud, cam, bg, smooth)
    grads = R.rasterize_backward(ctx, w)
    checked, failures = 0, []
    for name, gname in (("means", "d_means"), ("rotations", "d_rotations"),
                        ("log_scales", "d_log_scales"), ("opacity_logits", "d_opacity_logits"),
                        ("sh", "d_sh")):
        arr = getattr(cloud, name)
        flat = arr.reshape(-1)
        gflat = getattr(grads, gname).reshape(-1)
        floor = 2e-3 * np.abs(gflat).max()
        for i in range(flat.size):
            orig = flat[i]
            hi = float(np.float32(orig + 2e-3))
            lo = float(np.float32(orig - 2e-3))
            flat[i] = hi
            lp = loss(cloud)
            flat[i] = lo
            lm = loss(cloud)
            flat[i] = orig
            num = (lp - lm) / (hi - lo)
            err = abs(gflat[i] - num)
            checked += 1
            if err > max(floor, 2e-2 * max(abs(num), abs(gflat[i]))):
                failures.append((name, i, gflat[i], num))
    assert checked == 5 * (3 + 4 + 3 + 1 + 12)
    assert not failures, f"{len(failures)} gradient mismatches: {failures[:5]}"


def test_equal_depth_plane_order_bit_exact(P):
    """A plane of splats facing a tilted camera: its fp64 depths differ only by
    rounding, so one fp32 depth key holds tens of thousands of survivors.  The
    tie-break must give the stable (fp64 depth, index) order (rasterizer.py:
    228-230), in linear time.  At this ulp level the reference's own order
    depends on how its BLAS DGEMM rounds `means @ R.T` (cameras.py:80), so the
    expected order is the stable sort of the kernel's depth, restated here in
    the kernel's exact operation order ((R20 m0 + R21 m1) + R22 m2) + t2."""
    torch = P["torch"]
    R, T, S = P["rasterizer"], P["types"], P["scenes"]
    cam = S.look_at((1.3, -0.7, -4.2), 320, 240)
    rot = cam["w2c"][:3, :3]
    t = cam["w2c"][:3, 3]
    eye = -rot.T @ t
    rng = np.random.default_rng(9)
    n = 60000
    a, b = rng.uniform(-1.5, 1.5, size=(2, n))
    means = S.f32(eye + 4.0 * rot[2] + a[:, None] * rot[0] + b[:, None] * rot[1])
    cloud = dict(means=means, rotations=S.f32(np.tile([1.0, 0, 0, 0], (n, 1))),
                 log_scales=S.f32(np.full((n, 3), -4.5)), opacity_logits=S.f32(rng.normal(size=n)),
                 sh=S.f32(np.concatenate([rng.uniform(size=(n, 1, 3)), np.zeros((n, 3, 3))], 1)))
    z = ((rot[2, 0] * means[:, 0] + rot[2, 1] * means[:, 1]) + rot[2, 2] * means[:, 2]) + t[2]
    keep = np.flatnonzero(z > cam["near"])
    expect = keep[np.lexsort((keep, z[keep]))]
    _, counts = np.unique(z.astype(np.float32), return_counts=True)
    assert counts.max() > 5000  # the adversarial case really is one long run
    assert len(np.unique(z)) > 100  # ... of distinct fp64 depths
    gc = T.GaussianCloud(**cloud)
    R.rasterize_forward(gc, T.Camera.from_any(cam))  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, ctx = R.rasterize_forward(gc, T.Camera.from_any(cam))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    np.testing.assert_array_equal(ctx.indices, expect)
    assert dt < 1.0, f"forward took {dt:.3f} s"
    # the image matches the float64 oracle blended in that same order
    pj = O.project(cloud, cam)
    pos = np.empty(n, dtype=np.int64)
    pos[pj["indices"]] = np.arange(len(pj["indices"]))
    pj = {k: v[pos[expect]] for k, v in pj.items()}
    s = O.DEFAULT_SETTINGS
    image = np.zeros((cam["height"], cam["width"], 3))
    for tile in O.tile_lists(pj["mean2d"], pj["cov2d"], pj["opacity"], cam["width"],
                             cam["height"], s["tile_size"], s["skip_alpha"]):
        y0, y1, x0, x1, mem = tile
        _, _, _, _, al, tb, alive, _ = O._tile_pairs(pj, tile, s)
        image[y0:y1, x0:x1] = ((al * tb * alive) @ pj["colors"][mem]).reshape(y1 - y0, x1 - x0, 3)
    assert np.abs(out.image - image).max() <= 1e-4


# ---------------------------------------------------------------- NTC / transform FD
def test_ntc_gradients_match_finite_differences(P, rng):
    """test_ntc.py:183-216 (TINY grid, 1 x 8 hidden, step 1e-3); fp32 decoder:
    absolute tolerance 2e-4 instead of 1e-9."""
    T, N = P["types"], P["ntc"]
    tiny = T.HashGridConfig(n_levels=2, n_features=2, table_size_log2=4, base_resolution=4,
                            growth_factor=2.0, aabb_min=(0.0, 0.0, 0.0), aabb_max=(1.0, 1.0, 1.0))
    cache = N.NeuralTransformationCache(tiny, hidden_layers=1, hidden_dim=8, output_init="random",
                                        seed=7)
    r2 = np.random.default_rng(8)
    cache.biases[0][:] = r2.choice([-1.0, 1.0], size=8) * r2.uniform(0.05, 0.15, size=8)
    cache.tables[:] = r2.uniform(-0.3, 0.3, size=cache.tables.shape)
    cache.quantize_float32()
    mu = rng.uniform(0.05, 0.95, size=(5, 3))
    w_mu = rng.normal(size=(5, 3))
    w_q = rng.normal(size=(5, 4))

    def loss():
        d_mu, d_q, _ = cache.forward(mu)
        return float(np.sum(w_mu * d_mu) + np.sum(w_q * d_q))

    _, _, ctx = cache.forward(mu)
    grads, _ = cache.backward(ctx, w_mu, w_q)
    step = 1e-3
    for key, arr in cache._param_dict().items():
        flat = arr.reshape(-1)
        gflat = grads[key].reshape(-1)
        for i in range(flat.size):
            orig = flat[i]
            flat[i] = orig + step
            lp = loss()
            flat[i] = orig - step
            lm = loss()
            flat[i] = orig
            num = (lp - lm) / (2 * step)
            err = abs(gflat[i] - num)
            assert err <= max(2e-4, 2e-2 * max(abs(num), abs(gflat[i]))), (key, i, gflat[i], num)


def test_transform_cache_gradients_match_finite_differences(P, rng):
    """test_transform.py:174-215 (1 x 8 hidden, random output, biases off the
    ReLU kink); fp32 path: step 1e-3, absolute tolerance 5e-4."""
    T, N, X = P["types"], P["ntc"], P["transform"]
    grid = T.HashGridConfig(n_levels=2, n_features=2, table_size_log2=4, base_resolution=4,
                            growth_factor=2.0, aabb_min=(-2.0, -2.0, -2.0),
                            aabb_max=(2.0, 2.0, 6.0))
    cache = N.NeuralTransformationCache(grid, hidden_layers=1, hidden_dim=8, output_init="random",
                                        seed=2)
    cache.biases[0][:] = np.linspace(-0.15, 0.15, 8) + 0.02
    cache.tables[:] = np.random.default_rng(3).uniform(-0.2, 0.2, size=cache.tables.shape)
    cache.quantize_float32()
    n = 4
    means = rng.uniform(-1.5, 1.5, size=(n, 3))
    means[:, 2] = rng.uniform(1.5, 4.0, size=n)
    sh = np.zeros((n, 4, 3))
    sh[:, 0, :] = rng.uniform(-0.6, 0.6, size=(n, 3))
    sh[:, 1:, :] = rng.normal(scale=0.15, size=(n, 3, 3))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.uniform(0.4, 0.9, size=n)
    cloud = T.GaussianCloud(means=means, rotations=q,
                            log_scales=rng.uniform(np.log(0.08), np.log(0.3), size=(n, 3)),
                            opacity_logits=np.log(op / (1 - op)), sh=sh).quantize_float32()
    w_m = rng.normal(size=(n, 3))
    w_r = rng.normal(size=(n, 4))
    w_s = rng.normal(size=(n, 4, 3))

    def loss():
        out, _ = X.apply_ntc(cloud, cache)
        return float(np.sum(w_m * out.means) + np.sum(w_r * out.rotations) + np.sum(w_s * out.sh))

    _, ctx = X.apply_ntc(cloud, cache)
    grads, _ = X.apply_ntc_backward(ctx, w_m, w_r, w_s)
    step = 1e-3
    for key, arr in cache._param_dict().items():
        flat = arr.reshape(-1)
        gflat = grads[key].reshape(-1)
        for i in range(flat.size):
            orig = flat[i]
            flat[i] = orig + step
            lp = loss()
            flat[i] = orig - step
            lm = loss()
            flat[i] = orig
            num = (lp - lm) / (2 * step)
            err = abs(gflat[i] - num)
            assert err <= max(5e-4, 2e-2 * max(abs(num), abs(gflat[i]))), (key, i, gflat[i], num)


# ---------------------------------------------------------------- batched step on the device
def test_view_sharded_batched_step_vs_oracle(P):
    """ViewShardedStage1 (one rank, B = 4 views per iteration): the device
    accumulates grad_scale = 1/B image gradients over the views, then one lazy
    Adam step.  Oracle: mean of the per-view reference gradients
    (transform.py:99-135 -> ntc.py:250-288), one Adam step (optim.py:33-66).
    Then a 3-iteration batched frame: batch losses and the last-epoch
    view-space statistics (adaptive.py:79-97) against the oracle."""
    torch = P["torch"]
    from paper_2403_01444_b200.dist import ViewShardedStage1, batched_view_order
    from paper_2403_01444_b200.stage1 import Stage1Config

    S = P["scenes"]
    sc = S.small_scene(seed=14, n=2500, width=96, height=72, sh_degree=1, n_views=4)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=5)
    tables = S.f32(np.random.default_rng(6).uniform(-0.05, 0.05, size=tables.shape))
    moved = S.moved_cloud(sc.cloud, np.random.default_rng(2))
    targets = [O.render(moved, c)[0]["image"] for c in sc.cameras]

    class Cache:
        grid = P["types"].HashGridConfig.from_any(sc.grid)

    def make():
        c = Cache()
        c.tables, c.weights, c.biases = tables.copy(), mlp["weights"], mlp["biases"]
        return ViewShardedStage1(sc.cloud, c, list(zip(sc.cameras, targets)),
                                 Stage1Config(stage1_iterations=3), views_per_iteration=4)

    def state():
        return dict(grid=sc.grid, tables=tables.copy(),
                    mlp=dict(weights=[w.copy() for w in mlp["weights"]],
                             biases=[b.copy() for b in mlp["biases"]]),
                    inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)

    # --- one batched step
    vs = make()
    batch = [2, 0, 3, 1]
    vs.step(batch)
    torch.cuda.synchronize()
    st = state()
    rs = [O.stage1_iteration(st, sc.cloud, sc.cameras[v], targets[v], apply_adam=False)
          for v in batch]
    g_tab = sum(r["g_tables"] for r in rs) / 4
    gw = [sum(r["g_w"][i] for r in rs) / 4 for i in range(3)]
    gb = [sum(r["g_b"][i] for r in rs) / 4 for i in range(3)]
    O.adam_apply(st, g_tab, gw, gb, 0.002)
    tab = vs.trainer.tables.view(st["tables"].shape).cpu().numpy()
    assert G.norm_rel(tab - tables, st["tables"] - tables) <= 1e-3
    from paper_2403_01444_b200.device import unpack_params

    ws, bs = unpack_params(vs.trainer.params.cpu().numpy(), vs.trainer.w_shapes,
                           vs.trainer.layout)
    for i in range(3):
        assert G.norm_rel(ws[i] - mlp["weights"][i],
                          st["mlp"]["weights"][i] - mlp["weights"][i]) <= 1e-3, i
    np.testing.assert_allclose(vs.batch_losses()[0], np.mean([r["loss"] for r in rs]), rtol=1e-5)

    # --- a 3-iteration batched frame with the last-epoch statistics window
    vs = make()
    losses = vs.run(3, frame_index=2)
    st = state()
    ref_losses = []
    n = len(sc.cloud["means"])
    norm, count = np.zeros(n), np.zeros(n, dtype=np.int64)
    stats_from = 3 * 4 - 4
    for t, bt in enumerate(batched_view_order(0, 2, 4, 3, 4)):
        rs = [O.stage1_iteration(st, sc.cloud, sc.cameras[v], targets[v], apply_adam=False)
              for v in bt]
        for j, r in enumerate(rs):
            if t * 4 + j >= stats_from:
                norm += r["render_grads"]["viewspace"]
                count += r["render_grads"]["contributed"]
        O.adam_apply(st, sum(r["g_tables"] for r in rs) / 4,
                     [sum(r["g_w"][i] for r in rs) / 4 for i in range(3)],
                     [sum(r["g_b"][i] for r in rs) / 4 for i in range(3)], 0.002)
        ref_losses.append(np.mean([r["loss"] for r in rs]))
    np.testing.assert_allclose(losses, ref_losses, rtol=1e-3)
    gn, gc = vs.trainer.viewspace_stats()
    assert G.norm_rel(gn, norm) <= 1e-3
    np.testing.assert_array_equal(gc, count)
