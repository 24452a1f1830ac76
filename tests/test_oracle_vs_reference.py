"""Pin the oracle against the unmodified reference on fresh random inputs.

Runs only where /root/reference exists (the build container); the committed
golden vectors (test_oracle_golden.py) carry the same pinning elsewhere.
"""

import numpy as np
import pytest

from oracle import refbridge as rb
from oracle import stage1 as O

pytestmark = pytest.mark.skipif(not rb.available(), reason="reference package not present")


@pytest.fixture(scope="module")
def R():
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        yield rb.load()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_render_and_backward_match_reference(R, seed):
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=100 + seed, n=400, width=50, height=38, sh_degree=1)
    cloud, cam = sc.cloud, sc.cameras[seed % 2]
    bg = np.random.default_rng(seed).uniform(size=3)
    out, ctx = O.render(cloud, cam, bg)
    rout, rctx = R["rasterizer"].rasterize_forward(rb.ref_cloud(R, cloud), rb.ref_camera(R, cam), bg)
    np.testing.assert_array_equal(ctx["proj"]["indices"], rctx.indices)
    assert len(ctx["tiles"]) == len(rctx.tiles)
    for a, b in zip(ctx["tiles"], rctx.tiles):
        assert a[:4] == b[:4]
        np.testing.assert_array_equal(a[4], b[4])
    np.testing.assert_allclose(out["image"], rout.image, atol=1e-12)
    np.testing.assert_array_equal(out["touch"], rout.per_gaussian_touch_count)
    d = np.random.default_rng(seed + 7).normal(size=out["image"].shape)
    g = O.render_backward(ctx, d)
    rg = R["rasterizer"].rasterize_backward(rctx, d)
    for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh"):
        np.testing.assert_allclose(g[k], getattr(rg, k), rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(g["viewspace"], rg.viewspace_grad_norm, rtol=1e-8, atol=1e-14)


@pytest.mark.parametrize("seed", [0, 1])
def test_stage1_step_matches_reference(R, seed):
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=200 + seed, n=600, width=48, height=40, sh_degree=1)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=seed)
    tables = scenes.f32(np.random.default_rng(seed).uniform(-0.05, 0.05, size=tables.shape))
    target = np.random.default_rng(seed + 1).uniform(size=(40, 48, 3))
    state = dict(grid=sc.grid, tables=tables.copy(), mlp=mlp,
                 inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    r = O.stage1_iteration(state, sc.cloud, sc.cameras[0], target, apply_adam=False)
    cache = rb.ref_cache(R, sc.grid, tables, mlp)
    tr, tctx = R["transform"].apply_ntc(rb.ref_cloud(R, sc.cloud), cache)
    out, rctx = R["rasterizer"].rasterize_forward(tr, rb.ref_camera(R, sc.cameras[0]))
    loss, d_img = R["losses"].render_loss(out.image, target)
    g = R["rasterizer"].rasterize_backward(rctx, d_img)
    grads, _ = R["transform"].apply_ntc_backward(tctx, g.d_means, g.d_rotations, g.d_sh)
    assert abs(loss - r["loss"]) < 1e-12
    for l in range(sc.grid["levels"]):
        np.testing.assert_allclose(r["g_tables"][l], grads[f"table_{l}"], rtol=1e-7, atol=1e-16)
    for i in range(3):
        np.testing.assert_allclose(r["g_w"][i], grads[f"w_{i}"], rtol=1e-7, atol=1e-16)
