"""The stream wire formats: the per-frame NTC blob, written
from a reference-shaped cache or straight from the device parameters of a
Stage-1 trainer, and the `.splv` stream container around it.

Format (reference streamio.py:81-150, docs/formats.md:29-99), little endian:
  header  struct "<IIIId6dIII": n_levels, n_features, table_size_log2,
          base_resolution, growth_factor (f64), aabb_min[3], aabb_max[3] (f64),
          hidden_layers, hidden_dim, n_outputs (= 7)
  tables  (L, T, F) float32
  then per layer i: W_i (fan_in, fan_out) float32, b_i (fan_out) float32

The bytes are identical to the reference's `serialize_ntc` for the same
parameters (tests/golden/ntc_blob.npz, written by the unmodified reference).

Container (reference streamio.py:1-19, :153-325), little endian:
  b"SPLV", u32 version 1, then blocks of  tag[4] | u64 length | payload | u32 crc32,
  in the order HEAD (canonical JSON), INIT (initial cloud), WARM (warm NTC
  blob), FREC per frame (u32 index | u64 n | NTC blob | u64 m | cloud payload).
  Cloud payload: u32 count, then float32 runs of means (N,3), rotations (N,4),
  log_scales (N,3), opacity_logits (N,), sh (N,4,3) -- the reference's SH
  degree <= 1 layout; degree 0 is padded to its 4 rows.  Files written here are
  byte-identical to the reference's StreamWriter (tests/golden/stream.npz).
"""

from __future__ import annotations

import json
import struct
import zlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import DataError, FormatError
from .ntc import NeuralTransformationCache
from .types import GaussianCloud, HashGridConfig

NTC_HEADER = struct.Struct("<IIIId6dIII")


def _header(grid: HashGridConfig, hidden_layers: int, hidden_dim: int, n_out: int) -> bytes:
    g = HashGridConfig.from_any(grid)
    return NTC_HEADER.pack(g.n_levels, g.n_features, g.table_size_log2, g.base_resolution,
                           float(g.growth_factor), *np.asarray(g.aabb_min, dtype=float),
                           *np.asarray(g.aabb_max, dtype=float), hidden_layers, hidden_dim, n_out)


def _pack(grid, hidden_layers, hidden_dim, tables, weights, biases) -> bytes:
    parts = [_header(grid, hidden_layers, hidden_dim, int(np.shape(weights[-1])[1])),
             np.ascontiguousarray(tables).astype("<f4").tobytes()]
    for w, b in zip(weights, biases):
        parts.append(np.ascontiguousarray(w).astype("<f4").tobytes())
        parts.append(np.ascontiguousarray(b).astype("<f4").tobytes())
    return b"".join(parts)


def serialize_ntc(cache) -> bytes:
    """Blob of a reference-shaped cache (streamio.py:84-104)."""
    return _pack(cache.grid, len(cache.weights) - 1, int(np.shape(cache.weights[0])[1]),
                 cache.tables, cache.weights, cache.biases)


def serialize_ntc_device(trainer) -> bytes:
    """Blob straight from a Stage1Trainer's device parameters (one D2H copy
    of the tables and of the packed decoder vector, no cache round trip)."""
    from .device import unpack_params

    tab = trainer.tables.view(trainer.grid_cfg.n_levels, trainer.grid_cfg.table_size,
                              trainer.grid_cfg.n_features).cpu().numpy()
    ws, bs = unpack_params(trainer.params.cpu().numpy(), trainer.w_shapes, trainer.layout)
    return _pack(trainer.grid_cfg, len(ws) - 1, int(ws[0].shape[1]), tab, ws, bs)


def deserialize_ntc(data: bytes) -> NeuralTransformationCache:
    """streamio.py:107-150: a cache holding the blob's parameters, fresh Adam."""
    if len(data) < NTC_HEADER.size:
        raise FormatError("cache payload shorter than its header")
    f = NTC_HEADER.unpack_from(data, 0)
    grid = HashGridConfig(n_levels=f[0], n_features=f[1], table_size_log2=f[2],
                          base_resolution=f[3], growth_factor=f[4], aabb_min=tuple(f[5:8]),
                          aabb_max=tuple(f[8:11]))
    hidden_layers, hidden_dim, n_out = f[11:14]
    cache = NeuralTransformationCache(grid, hidden_layers=hidden_layers, hidden_dim=hidden_dim)
    if cache.weights[-1].shape[1] != n_out:
        raise FormatError(f"cache output width {n_out} unsupported")
    # every parameter array in wire order, as float32 runs after the header
    dests = [cache.tables] + [a for wb in zip(cache.weights, cache.biases) for a in wb]
    sizes = np.array([a.size for a in dests], dtype=np.int64)
    need = NTC_HEADER.size + 4 * int(sizes.sum())
    if len(data) < need:
        raise FormatError("truncated cache payload")
    if len(data) > need:
        raise FormatError(f"cache payload has {len(data) - need} trailing bytes")
    flat = np.frombuffer(data, dtype="<f4", offset=NTC_HEADER.size).astype(np.float64)
    for a, lo, hi in zip(dests, np.cumsum(sizes) - sizes, np.cumsum(sizes)):
        a[...] = flat[lo:hi].reshape(a.shape)
    cache.reset_adam()
    return cache


# ---------------------------------------------------------------- .splv container
MAGIC, VERSION = b"SPLV", 1
_TAG_LEN = struct.Struct("<4sQ")
_CRC = struct.Struct("<I")
_FREC_HEAD = struct.Struct("<IQ")  # frame index, NTC blob length
_CLOUD_RUNS = (("means", 3), ("rotations", 4), ("log_scales", 3), ("opacity_logits", 1),
               ("sh", 12))
_CLOUD_FLOATS = sum(w for _, w in _CLOUD_RUNS)  # 23 float32 per Gaussian


def serialize_cloud(cloud) -> bytes:
    """Cloud payload (streamio.py:49-54): u32 count + float32 field runs."""
    c = GaussianCloud.from_any(cloud)
    sh = c.sh
    if sh.shape[1] == 1:  # degree 0 in the reference's 4-row layout
        sh = np.concatenate([sh, np.zeros((len(sh), 3, 3))], axis=1)
    if sh.shape[1] != 4:
        raise DataError("the stream container stores SH degree <= 1 (4 rows, docs/formats.md)")
    runs = [c.means, c.rotations, c.log_scales, c.opacity_logits, sh]
    return struct.pack("<I", len(c)) + b"".join(np.ascontiguousarray(a).astype("<f4").tobytes()
                                                 for a in runs)


def deserialize_cloud(data: bytes) -> GaussianCloud:
    """streamio.py:57-78."""
    if len(data) < 4:
        raise FormatError("cloud payload shorter than its count field")
    n = struct.unpack_from("<I", data)[0]
    want = 4 + 4 * _CLOUD_FLOATS * n
    if len(data) != want:
        raise FormatError(f"cloud payload is {len(data)} bytes, expected {want} for {n} Gaussians")
    flat = np.frombuffer(data, dtype="<f4", offset=4).astype(np.float64)
    fields, pos = {}, 0
    for name, w in _CLOUD_RUNS:
        fields[name] = flat[pos:pos + w * n]
        pos += w * n
    return GaussianCloud(means=fields["means"].reshape(n, 3),
                         rotations=fields["rotations"].reshape(n, 4),
                         log_scales=fields["log_scales"].reshape(n, 3),
                         opacity_logits=fields["opacity_logits"],
                         sh=fields["sh"].reshape(n, 4, 3))


@dataclass
class FrameRecord:
    """One streamed frame: the NTC blob and the frame's additional Gaussians."""

    frame_index: int
    ntc_blob: bytes
    additional: GaussianCloud

    def cache(self) -> NeuralTransformationCache:
        return deserialize_ntc(self.ntc_blob)

    def sizes(self) -> dict:
        add = len(serialize_cloud(self.additional))
        over = _TAG_LEN.size + _CRC.size + _FREC_HEAD.size + 8
        return {"ntc_bytes": len(self.ntc_blob), "additional_bytes": add,
                "overhead_bytes": over, "total_bytes": len(self.ntc_blob) + add + over}


@dataclass
class StreamData:
    header: dict
    initial_cloud: GaussianCloud
    warm_blob: bytes
    records: list

    @property
    def n_frames(self) -> int:
        return len(self.records) + 1  # frame 0 is the initial cloud

    def warm_cache(self) -> NeuralTransformationCache:
        return deserialize_ntc(self.warm_blob)


def _block(tag: bytes, payload: bytes) -> bytes:
    return _TAG_LEN.pack(tag, len(payload)) + payload + _CRC.pack(zlib.crc32(payload))


class StreamWriter:
    """Appends HEAD at open, then INIT / WARM / FREC blocks; frames are flushed
    as written and must be consecutive from 1."""

    def __init__(self, path, header: dict):
        self._f = open(path, "wb")
        head = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
        self._f.write(MAGIC + struct.pack("<I", VERSION) + _block(b"HEAD", head))
        self._expect = 1

    def write_initial(self, cloud) -> None:
        self._f.write(_block(b"INIT", serialize_cloud(cloud)))

    def write_warmup(self, cache) -> None:
        self._f.write(_block(b"WARM", serialize_ntc(cache)))

    def write_frame(self, record: FrameRecord) -> None:
        if record.frame_index != self._expect:
            raise FormatError(f"frame records must be consecutive: expected {self._expect}, "
                              f"got {record.frame_index}")
        cloud = serialize_cloud(record.additional)
        self._f.write(_block(b"FREC", _FREC_HEAD.pack(record.frame_index, len(record.ntc_blob))
                             + record.ntc_blob + struct.pack("<Q", len(cloud)) + cloud))
        self._f.flush()
        self._expect += 1

    def write_frame_device(self, frame_index: int, trainer, additional) -> None:
        """A frame whose NTC blob comes straight from a Stage1Trainer's device
        parameters (serialize_ntc_device), no cache round trip."""
        self.write_frame(FrameRecord(frame_index, serialize_ntc_device(trainer),
                                     GaussianCloud.from_any(additional)))

    def close(self) -> None:
        self._f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _blocks(data: bytes, name: str):
    """(tag, payload) of every block after the 8-byte preamble, CRC-checked."""
    pos, i = 8, 0
    while pos < len(data):
        if pos + _TAG_LEN.size > len(data):
            raise FormatError(f"{name}: truncated block header at byte {pos}")
        tag, n = _TAG_LEN.unpack_from(data, pos)
        start = pos + _TAG_LEN.size
        if start + n + _CRC.size > len(data):
            raise FormatError(f"{name}: block {i} ({tag!r}) truncated (need {n} payload bytes)")
        payload = data[start:start + n]
        if zlib.crc32(payload) != _CRC.unpack_from(data, start + n)[0]:
            raise FormatError(f"{name}: checksum mismatch in block {i} "
                              f"({tag.decode('ascii', 'replace')})")
        yield tag, payload
        pos, i = start + n + _CRC.size, i + 1


def _frame(payload: bytes, name: str) -> FrameRecord:
    if len(payload) < _FREC_HEAD.size:
        raise FormatError(f"{name}: frame record too short")
    idx, n = _FREC_HEAD.unpack_from(payload)
    a = _FREC_HEAD.size
    blob = payload[a:a + n]
    if len(blob) != n or a + n + 8 > len(payload):
        raise FormatError(f"{name}: frame {idx} record truncated")
    m = struct.unpack_from("<Q", payload, a + n)[0]
    cloud = payload[a + n + 8:a + n + 8 + m]
    if len(cloud) != m:
        raise FormatError(f"{name}: frame {idx} record truncated")
    return FrameRecord(idx, bytes(blob), deserialize_cloud(cloud))


def read_stream(path) -> StreamData:
    """streamio.py:271-325: parse and validate a container."""
    path = Path(path)
    if not path.exists():
        raise FormatError(f"stream not found: {path}")
    data = path.read_bytes()
    if len(data) < 8 or data[:4] != MAGIC:
        raise FormatError(f"{path}: not a stream container (bad magic)")
    if struct.unpack_from("<I", data, 4)[0] != VERSION:
        raise FormatError(f"{path}: unsupported version {struct.unpack_from('<I', data, 4)[0]}")
    parts = {b"HEAD": None, b"INIT": None, b"WARM": None}
    records = []
    for tag, payload in _blocks(data, str(path)):
        if tag == b"FREC":
            rec = _frame(payload, str(path))
            if rec.frame_index != len(records) + 1:
                raise FormatError(f"{path}: frame records out of order "
                                  f"(expected {len(records) + 1}, got {rec.frame_index})")
            records.append(rec)
        elif tag in parts:
            parts[tag] = payload
        else:
            raise FormatError(f"{path}: unknown block tag {tag!r}")
    if any(v is None for v in parts.values()):
        raise FormatError(f"{path}: missing HEAD, INIT, or WARM block")
    return StreamData(header=json.loads(parts[b"HEAD"].decode()),
                      initial_cloud=deserialize_cloud(parts[b"INIT"]),
                      warm_blob=bytes(parts[b"WARM"]), records=records)
