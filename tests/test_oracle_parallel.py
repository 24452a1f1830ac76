"""The all-core oracle iteration (oracle/parallel.py, used by bench.py's CPU
arms) computes exactly the serial oracle's Stage-1 iteration."""

import numpy as np

from oracle import parallel
from oracle import stage1 as O


def test_parallel_iteration_equals_serial():
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=8, n=1200, width=72, height=56, sh_degree=3, n_views=2)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=1)
    tables = scenes.f32(np.random.default_rng(2).uniform(-0.05, 0.05, size=tables.shape))
    target = O.render(scenes.moved_cloud(sc.cloud, np.random.default_rng(3)), sc.cameras[1])[0]

    def state():
        return dict(grid=sc.grid, tables=tables.copy(),
                    mlp=dict(weights=[w.copy() for w in mlp["weights"]],
                             biases=[b.copy() for b in mlp["biases"]]),
                    inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)

    sa, sb = state(), state()
    ref = O.stage1_iteration(sa, sc.cloud, sc.cameras[1], target["image"])
    got = parallel.ParallelStage1(3).iteration(sb, sc.cloud, sc.cameras[1], target["image"])
    assert abs(got["loss"] - ref["loss"]) <= 1e-12 * ref["loss"]
    np.testing.assert_allclose(got["image"], ref["image"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(got["g_tables"], ref["g_tables"], rtol=1e-9, atol=1e-18)
    for a, b in zip(got["g_w"] + got["g_b"], ref["g_w"] + ref["g_b"]):
        np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-18)
    for k in ("d_means", "d_rotations", "d_sh", "viewspace", "contributed"):
        np.testing.assert_allclose(got["render_grads"][k], ref["render_grads"][k], rtol=1e-9,
                                   atol=1e-18)
    np.testing.assert_allclose(sb["tables"], sa["tables"], rtol=1e-9, atol=1e-15)


def test_parallel_render_equals_serial():
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=9, n=900, width=64, height=48, sh_degree=1, n_views=1)
    ref = O.render(sc.cloud, sc.cameras[0])[0]["image"]
    got = parallel.ParallelStage1(4).render(sc.cloud, sc.cameras[0])
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14)


def test_parallel_transform_render_equals_serial():
    """The config-2 CPU frame (apply_ntc + rasterize_forward) of bench.py's
    render line: equal to the serial oracle's transform then render."""
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=10, n=900, width=64, height=48, sh_degree=3, n_views=1)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=4)
    tables = scenes.f32(np.random.default_rng(5).uniform(-0.05, 0.05, size=tables.shape))
    inside = O.inside_mask(sc.grid, sc.cloud["means"])
    idx, w, _ = O.encode(sc.grid, sc.cloud["means"][inside])
    o7, _ = O.mlp_forward(mlp, O.gather(tables, idx, w))
    moved, _ = O.transform_forward(sc.cloud, inside, o7)
    ref = O.render(moved, sc.cameras[0])[0]["image"]
    state = dict(grid=sc.grid, tables=tables, mlp=mlp, inside=inside, enc=None)
    got = parallel.ParallelStage1(3).transform_render(state, sc.cloud, sc.cameras[0])
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13)
