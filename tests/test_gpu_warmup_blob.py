"""GPU tests of the §8(f) rows F2 (device NTC warm-up) and F4 (blob straight
from device parameters) against the reference's golden runs."""

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu


def _cache_from(d):
    from paper_2403_01444_b200.ntc import NeuralTransformationCache
    from paper_2403_01444_b200.types import HashGridConfig

    g = G.grid(d)
    grid = HashGridConfig(n_levels=g["levels"], n_features=g["features"],
                          table_size_log2=g["log2_table"], base_resolution=g["base"],
                          growth_factor=g["growth"], aabb_min=g["lo"], aabb_max=g["hi"])
    cache = NeuralTransformationCache(grid, output_init="random")
    m = G.mlp(d)
    cache.tables[:] = d["tables"]
    for i in range(len(m["weights"])):
        cache.weights[i][:] = m["weights"][i]
        cache.biases[i][:] = m["biases"][i]
    return cache


def test_device_warmup_matches_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200.warmup import warmup_train

    d = G.load("warmup")
    cache = _cache_from(d)
    before = cache.get_params()
    params, hist = warmup_train(cache, d["means"], noise_sigma=0.05, iterations=5, lr=0.002,
                                batch_size=256, seed=7)
    np.testing.assert_allclose(hist, d["history"], rtol=1e-5)
    for k, v in params.items():
        ref = d[f"after_{k}"]
        delta_ref = ref - before[k]
        if np.linalg.norm(delta_ref) > 0:
            assert G.norm_rel(v - before[k], delta_ref) <= 5e-3, k
    # the cache holds the float32 snapshot
    np.testing.assert_array_equal(cache.tables[0], params["table_0"])
    np.testing.assert_array_equal(cache.tables, cache.tables.astype(np.float32))


def test_device_warmup_rejects_empty():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200.errors import DataError
    from paper_2403_01444_b200.warmup import warmup_train

    d = G.load("warmup")
    with pytest.raises(DataError):
        warmup_train(_cache_from(d), np.zeros((0, 3)), 0.05, 1)


def test_blob_from_device_params_matches_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import scenes, streamio
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    d = G.load("ntc_blob")
    cache = _cache_from(d)
    sc = scenes.small_scene(seed=5, n=300, width=48, height=40, sh_degree=0, n_views=1)
    lo, hi = np.array(cache.grid.aabb_min), np.array(cache.grid.aabb_max)
    cloud = dict(sc.cloud)
    cloud["means"] = scenes.f32(np.clip(cloud["means"] * 0.2, lo + 0.01, hi - 0.01))
    views = [(sc.cameras[0], np.zeros((40, 48, 3)))]
    tr = Stage1Trainer(cloud, cache, views, Stage1Config())
    assert streamio.serialize_ntc_device(tr) == d["blob"].tobytes()


class _Rec:
    def __init__(self, blob, add):
        self.ntc_blob, self.additional = blob, add


class _Stream:
    def __init__(self, d):
        self.header = {"background": list(d["background"])}
        self.initial_cloud = G.cloud(d)
        self.records = [_Rec(d[f"blob{f}"].tobytes(), G.cloud(d, f"add{f}_")) for f in range(3)]

    @property
    def n_frames(self):
        return len(self.records) + 1


def test_device_playback_matches_reference():
    """materialize_frame + playback_render of a 3-record stream
    (NTC folding, added Gaussians, background) against the reference's renders."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import playback
    from paper_2403_01444_b200.errors import DataError

    d = G.load("playback")
    st = _Stream(d)
    cam = G.camera(d)
    for i in range(4):
        img = playback.playback_render(st, i, cam)
        assert np.abs(img - d[f"image{i}"]).max() <= 1e-4, i
    player = playback.DevicePlayer(st)
    for i in [0, 1, 2, 3, 1]:  # sequential folding, then a seek backwards
        img = player.render(i, cam).cpu().numpy()
        assert np.abs(img - d[f"image{i}"]).max() <= 1e-4, i
    assert playback.materialize_frame(st, 2).means.shape[0] == len(d["cloud_means"]) + 40
    with pytest.raises(DataError):
        playback.playback_render(st, 4, cam)


def test_device_stage2_matches_reference():
    """stage2_optimize (joint render, full-parameter backward,
    per-parameter Adam, epoch-boundary split/prune with the reference's
    generator sequence) against the reference's run: same losses, same
    surviving rows, parameters within tolerance."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200.stage2 import AdditionConfig, stage2_optimize

    d = G.load("stage2")
    cfg = AdditionConfig(tau_grad=float(d["tau_grad"]), max_additional=int(d["max_additional"]))
    views = [(G.camera(d, f"cam{v}_"), d[f"target{v}"]) for v in range(2)]
    out, losses = stage2_optimize(G.cloud(d), G.cloud(d, "add_"), views, cfg,
                                  int(d["iterations"]), np.random.default_rng(int(d["rng_seed"])))
    np.testing.assert_allclose(losses, d["losses"], rtol=1e-4)
    assert out.means.shape == d["final_means"].shape
    for k in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
        ref = d[f"final_{k}"]
        assert G.norm_rel(getattr(out, k), ref) <= 1e-3, k
