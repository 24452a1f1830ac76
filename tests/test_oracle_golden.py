"""Pin the CPU oracle (oracle/stage1.py) against the reference's golden vectors.

The fixtures were produced by the unmodified reference (oracle/make_golden.py);
these tests run anywhere (no reference, no GPU needed).
"""

import numpy as np
import pytest

import golden_io as G
from oracle import stage1 as O


@pytest.mark.parametrize("tag", ["small", "cfg1"])
def test_encode_bit_exact(tag):
    d = G.load(f"encode_{tag}")
    grid = G.grid(d)
    idx, w, touched = O.encode(grid, d["x"])
    assert O.level_resolutions(grid["base"], grid["growth"], grid["levels"]) == list(d["res"])
    np.testing.assert_array_equal(idx, d["idx"])
    np.testing.assert_array_equal(w, d["w"])
    if "tables" in d:
        np.testing.assert_allclose(O.gather(d["tables"], idx, w), d["feats"], rtol=0, atol=1e-15)


def test_cfg1_finest_resolution_is_2047():
    d = G.load("encode_cfg1")
    assert int(d["res"][-1]) == 2047


def test_ntc_forward_backward_and_adam():
    d = G.load("ntc")
    grid, mlp = G.grid(d), G.mlp(d)
    idx, w, touched = O.encode(grid, d["x"])
    feats = O.gather(d["tables"], idx, w)
    out, hidden = O.mlp_forward(mlp, feats)
    np.testing.assert_allclose(out[:, :3], d["d_mu"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(out[:, 3:], d["d_q"], rtol=1e-12, atol=1e-14)
    g7 = np.concatenate([d["g_mu"], d["g_q"]], 1)
    gw, gb, gf = O.mlp_backward(mlp, feats, hidden, g7)
    gt = O.table_scatter(d["tables"].shape, idx, w, gf)
    for i in range(len(gw)):
        np.testing.assert_allclose(gw[i], d[f"grad_w_{i}"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(gb[i], d[f"grad_b_{i}"], rtol=1e-10, atol=1e-12)
    for l in range(grid["levels"]):
        np.testing.assert_allclose(gt[l], d[f"grad_table_{l}"], rtol=1e-10, atol=1e-14)
        np.testing.assert_array_equal(touched[l], d[f"touched_table_{l}"])
    # two lazy Adam steps
    state = dict(grid=grid, tables=d["tables"].copy(), mlp=mlp, enc=(idx, w, touched))
    for _ in range(2):
        O.adam_apply(state, gt, gw, gb, 0.002)
    for l in range(grid["levels"]):
        np.testing.assert_allclose(state["tables"][l], d[f"after2_table_{l}"], rtol=1e-12,
                                   atol=1e-15)
    for i in range(len(gw)):
        np.testing.assert_allclose(state["mlp"]["weights"][i], d[f"after2_w_{i}"], rtol=1e-12,
                                   atol=1e-15)


def test_transform_forward_backward():
    d = G.load("transform")
    grid, mlp, cloud = G.grid(d), G.mlp(d), G.cloud(d)
    inside = O.inside_mask(grid, cloud["means"])
    np.testing.assert_array_equal(inside, d["inside"])
    idx, w, _ = O.encode(grid, cloud["means"][inside])
    feats = O.gather(d["tables"], idx, w)
    out7, hidden = O.mlp_forward(mlp, feats)
    moved, ctx = O.transform_forward(cloud, inside, out7)
    np.testing.assert_allclose(moved["means"], d["out_means"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(moved["rotations"], d["out_rotations"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(moved["sh"], d["out_sh"], rtol=1e-10, atol=1e-14)
    g7 = O.transform_backward(ctx, d["g_means"], d["g_rot"], d["g_sh"])
    gw, gb, gf = O.mlp_backward(mlp, feats, hidden, g7)
    gt = O.table_scatter(d["tables"].shape, idx, w, gf)
    for i in range(len(gw)):
        assert G.norm_rel(gw[i], d[f"grad_w_{i}"]) < 1e-10
    for l in range(grid["levels"]):
        assert G.norm_rel(gt[l], d[f"grad_table_{l}"]) < 1e-10


@pytest.mark.parametrize("tag", ["default", "smooth"])
def test_raster_forward_backward(tag):
    d = G.load(f"raster_{tag}")
    cloud, cam, s = G.cloud(d), G.camera(d), G.settings(d)
    out, ctx = O.render(cloud, cam, d["bg"], s)
    np.testing.assert_array_equal(ctx["proj"]["indices"], d["indices"])
    tiles = ctx["tiles"]
    rects = np.array([t[:4] for t in tiles]).reshape(-1, 4)
    np.testing.assert_array_equal(rects, d["tile_rects"])
    np.testing.assert_array_equal([len(t[4]) for t in tiles], d["tile_counts"])
    np.testing.assert_array_equal(np.concatenate([t[4] for t in tiles]), d["tile_members"])
    np.testing.assert_allclose(out["image"], d["image"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out["alpha_map"], d["alpha"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(out["touch"], d["touch"])
    g = O.render_backward(ctx, d["d_image"])
    for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh",
              "viewspace"):
        ref = d[k] if k != "viewspace" else d["viewspace"]
        assert G.norm_rel(g[k], ref) < 1e-9, k
    np.testing.assert_array_equal(g["contributed"], d["contributed"])


def test_render_loss():
    d = G.load("loss")
    loss, grad = O.render_loss(d["x"], d["y"])
    assert abs(loss - float(d["loss"])) < 1e-12
    np.testing.assert_allclose(grad, d["grad"], rtol=1e-9, atol=1e-15)


def test_stage1_two_iterations():
    d = G.load("stage1")
    grid, cloud = G.grid(d), G.cloud(d)
    cams = [G.camera(d, "cam0_"), G.camera(d, "cam1_")]
    targets = [d["target0"], d["target1"]]
    state = dict(grid=grid, tables=d["tables"].copy(), mlp=G.mlp(d),
                 inside=O.inside_mask(grid, cloud["means"]), enc=None)
    losses = []
    for t, v in enumerate([0, 1]):
        r = O.stage1_iteration(state, cloud, cams[v], targets[v])
        losses.append(r["loss"])
        if t == 0:
            np.testing.assert_allclose(r["image"], d["image_first"], atol=1e-12)
            for l in range(grid["levels"]):
                assert G.norm_rel(r["g_tables"][l], d[f"grad1_table_{l}"]) < 1e-8
            for i in range(3):
                assert G.norm_rel(r["g_w"][i], d[f"grad1_w_{i}"]) < 1e-8
    np.testing.assert_allclose(losses, d["losses"], rtol=1e-10)
    for i in range(3):
        assert G.norm_rel(state["mlp"]["weights"][i], d[f"after2_w_{i}"]) < 1e-6
