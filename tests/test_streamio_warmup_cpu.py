"""CPU tests of the §8(f) rows F2 (NTC warm-up) and F4 (NTC blob format):
the oracle warm-up against the reference's golden run, and the blob writer /
reader against the reference's bytes (tests/golden/{warmup,ntc_blob}.npz,
written by oracle/make_golden.py from the unmodified reference)."""

import numpy as np
import pytest

import golden_io as G
from oracle import stage1 as O


def test_oracle_warmup_loss_matches_reference():
    d = G.load("warmup")
    loss, g_mu, g_q = O.warmup_loss(d["d_mu"], d["d_q"])
    assert abs(loss - float(d["loss"])) <= 1e-12
    np.testing.assert_allclose(g_mu, d["g_mu"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(g_q, d["g_q"], rtol=1e-12, atol=1e-15)


def test_oracle_warmup_train_matches_reference():
    d = G.load("warmup")
    tables, mlp, hist = O.warmup_train(G.grid(d), d["tables"], G.mlp(d), d["means"],
                                       noise_sigma=0.05, iterations=5, lr=0.002,
                                       batch_size=256, seed=7)
    np.testing.assert_allclose(hist, d["history"], rtol=1e-10)
    for l in range(tables.shape[0]):
        np.testing.assert_allclose(tables[l], d[f"after_table_{l}"], rtol=0, atol=1e-7)
    for i in range(len(mlp["weights"])):
        np.testing.assert_allclose(mlp["weights"][i], d[f"after_w_{i}"], rtol=0, atol=1e-7)
        np.testing.assert_allclose(mlp["biases"][i], d[f"after_b_{i}"], rtol=0, atol=1e-7)


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


def test_ntc_blob_bytes_match_reference():
    from paper_2403_01444_b200 import streamio

    d = G.load("ntc_blob")
    blob = streamio.serialize_ntc(_cache_from(d))
    assert blob == d["blob"].tobytes()


def test_ntc_blob_round_trip_and_errors():
    import pytest

    from paper_2403_01444_b200 import streamio

    d = G.load("ntc_blob")
    ref = d["blob"].tobytes()
    cache = streamio.deserialize_ntc(ref)
    assert streamio.serialize_ntc(cache) == ref
    np.testing.assert_array_equal(cache.tables, d["tables"].astype(np.float32))
    with pytest.raises(streamio.FormatError):
        streamio.deserialize_ntc(ref[:10])
    with pytest.raises(streamio.FormatError):
        streamio.deserialize_ntc(ref[:-4])
    with pytest.raises(streamio.FormatError):
        streamio.deserialize_ntc(ref + b"\0\0\0\0")


# ---------------------------------------------------------------- .splv container
def _stream_golden():
    import json

    import golden_io as G

    d = G.load("stream")
    header = json.loads(d["header"].tobytes().decode())
    return d, header, G


def test_container_written_byte_identical_to_reference(tmp_path):
    from paper_2403_01444_b200 import streamio
    from paper_2403_01444_b200.types import GaussianCloud

    d, header, G = _stream_golden()
    path = tmp_path / "s.splv"
    with streamio.StreamWriter(path, header) as w:
        w.write_initial(GaussianCloud(**G.cloud(d, "init_")))
        w.write_warmup(streamio.deserialize_ntc(d["warm_blob"].tobytes()))
        for k in range(2):
            w.write_frame(streamio.FrameRecord(k + 1, d[f"blob{k}"].tobytes(),
                                               GaussianCloud(**G.cloud(d, f"add{k}_"))))
    assert path.read_bytes() == d["container"].tobytes()


def test_reference_container_reads_back(tmp_path):
    from paper_2403_01444_b200 import streamio

    d, header, G = _stream_golden()
    path = tmp_path / "ref.splv"
    path.write_bytes(d["container"].tobytes())
    sd = streamio.read_stream(path)
    assert sd.header == header and sd.n_frames == 3
    np.testing.assert_array_equal(sd.initial_cloud.means,
                                  d["init_means"].astype(np.float32).astype(np.float64))
    assert sd.warm_blob == d["warm_blob"].tobytes()
    for k, rec in enumerate(sd.records):
        assert rec.frame_index == k + 1 and rec.ntc_blob == d[f"blob{k}"].tobytes()
        np.testing.assert_allclose(rec.additional.sh, d[f"add{k}_sh"], atol=1e-7)
    assert sd.warm_cache().tables.shape[0] == 2


def test_container_corruption_raises(tmp_path):
    from paper_2403_01444_b200 import errors, streamio

    d, _, _ = _stream_golden()
    raw = bytearray(d["container"].tobytes())
    cases = {"magic": b"XXXX" + raw[4:], "truncated": raw[:-7],
             "crc": raw[:40] + bytes([raw[40] ^ 1]) + raw[41:], "version": raw[:4] + b"\x02" + raw[5:]}
    for name, data in cases.items():
        p = tmp_path / f"{name}.splv"
        p.write_bytes(bytes(data))
        with pytest.raises(errors.FormatError):
            streamio.read_stream(p)
    with pytest.raises(errors.FormatError):
        streamio.read_stream(tmp_path / "missing.splv")
