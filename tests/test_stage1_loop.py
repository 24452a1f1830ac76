"""The reference's Stage-1 loop (process_frame with stage2_iterations = 0,
pipeline.py:238-283), recorded from the unmodified reference in
tests/golden/stage1_loop.npz (oracle/make_golden.py gen_stage1_loop): the view
order of the 10 iterations, the per-iteration losses, the last-epoch
view-space statistics (adaptive.py:79-97) and the final cache blob.

CPU: the view-order restatement and the float64 oracle loop against it.
GPU: the fused Stage1Trainer frame and the drop-in-API frame
(paper_2403_01444_b200.pipeline) against it.  Multi-step trajectories are
graded at rel 1e-3 on the losses (eps = 1e-15 Adam amplifies
round-off), the statistics at norm-relative 1e-3 with exact view counts.
"""

import numpy as np
import pytest

import golden_io as G
from oracle import stage1 as O


def _load():
    d = G.load("stage1_loop")
    n = int(d["n_views"])
    cams = [G.camera(d, f"cam{i}_") for i in range(n)]
    targets = [d[f"target{i}"] for i in range(n)]
    return d, cams, targets


def test_view_order_matches_reference():
    from paper_2403_01444_b200.stage1 import view_order

    d, cams, _ = _load()
    got = view_order(int(d["seed"]), int(d["frame_index"]), len(cams), int(d["iterations"]))
    np.testing.assert_array_equal(got, d["view_order"])
    np.testing.assert_array_equal(O.stage1_view_order(int(d["seed"]), int(d["frame_index"]),
                                                      len(cams), int(d["iterations"])),
                                  d["view_order"])


def test_oracle_loop_matches_reference():
    from threadpoolctl import threadpool_limits

    d, cams, targets = _load()
    grid = G.grid(d)
    cloud = G.cloud(d)
    mlp = G.mlp(d)
    state = dict(grid=grid, tables=d["tables"].copy(),
                 mlp=dict(weights=[w.copy() for w in mlp["weights"]],
                          biases=[b.copy() for b in mlp["biases"]]),
                 inside=O.inside_mask(grid, cloud["means"]), enc=None)
    it, nv = int(d["iterations"]), len(cams)
    norm = np.zeros(len(cloud["means"]))
    count = np.zeros(len(cloud["means"]), dtype=np.int64)
    losses = []
    with threadpool_limits(1):
        for t, v in enumerate(d["view_order"]):
            r = O.stage1_iteration(state, cloud, cams[v], targets[v])
            losses.append(r["loss"])
            if t >= it - nv:
                norm += r["render_grads"]["viewspace"]
                count += r["render_grads"]["contributed"]
    np.testing.assert_allclose(losses, d["losses"], rtol=1e-9)
    np.testing.assert_allclose(norm, d["stats_norm"], rtol=1e-9, atol=1e-15)
    np.testing.assert_array_equal(count, d["stats_count"])


def _cfg():
    from paper_2403_01444_b200.types import LossConfig, RasterSettings

    class Cfg:
        stage1_iterations, ntc_lr, seed = 10, 0.002, 5
        raster, loss = RasterSettings(), LossConfig()

    return Cfg()


@pytest.mark.gpu
@pytest.mark.parametrize("driver", ["stage1_frame", "stage1_frame_dropin"])
def test_device_frame_matches_reference_loop(driver):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import pipeline, streamio
    from paper_2403_01444_b200.ntc import NeuralTransformationCache
    from paper_2403_01444_b200.types import GaussianCloud, HashGridConfig

    d, cams, targets = _load()
    mlp = G.mlp(d)
    warm = NeuralTransformationCache(HashGridConfig.from_any(G.grid(d)), output_init="random")
    warm.tables[:] = d["tables"]
    for i in range(len(mlp["weights"])):
        warm.weights[i][:] = mlp["weights"][i]
        warm.biases[i][:] = mlp["biases"][i]
    res = getattr(pipeline, driver)(GaussianCloud(**G.cloud(d)), warm, list(zip(cams, targets)),
                                    _cfg(), int(d["frame_index"]))
    np.testing.assert_allclose(res.losses, d["losses"], rtol=1e-3)
    assert G.norm_rel(res.stats_norm, d["stats_norm"]) <= 1e-3
    np.testing.assert_array_equal(res.stats_count, d["stats_count"])
    ref = streamio.deserialize_ntc(d["ntc_blob"].tobytes())
    assert G.norm_rel(res.cache.tables - d["tables"], ref.tables - d["tables"]) <= 1e-2
    assert G.norm_rel(res.cache.tables, ref.tables) <= 1e-3
    for i in range(len(ref.weights)):
        assert G.norm_rel(res.cache.weights[i], ref.weights[i]) <= 1e-3, i
    np.testing.assert_allclose(res.transformed.means, d["out_means"], atol=1e-4)
    np.testing.assert_allclose(res.transformed.rotations, d["out_rotations"], atol=1e-4)
    np.testing.assert_allclose(res.transformed.sh, d["out_sh"], atol=1e-4)
