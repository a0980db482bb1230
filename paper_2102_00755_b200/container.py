"""Self-describing binary container: the Python
mirror of include/ustfwi/io.hpp, byte-identical. Layout (little-endian, 128-byte header per
record, then the row-major payload; a file is a sequence of records) — INTEGRATION.md §6:

    0 magic "USTFWIBC" | 8 u32 version | 12 u32 dtype | 16 u32 kind | 20 u32 ndim
    24 u64 dims[4] | 56 f64 dx[3] | 80 f64 dt | 88 f64 t0 | 96 u64 payload bytes
    104 u32 CRC-32 (zlib) of the payload | 108 reserved (20 zero bytes)
"""
from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field
from typing import BinaryIO, List, Optional, Sequence, Tuple

import numpy as np

MAGIC = b"USTFWIBC"
VERSION = 1
HEADER_BYTES = 128

DTYPES = {1: np.dtype("<f4"), 2: np.dtype("<f8"), 3: np.dtype("<u8"), 4: np.dtype("u1")}
DTYPE_CODES = {v: k for k, v in DTYPES.items()}
KINDS = {"field": 0, "sensor_data": 1, "boundary_values": 2, "gradient": 3, "index_list": 4, "mask": 5}
KIND_NAMES = {v: k for k, v in KINDS.items()}

_HDR = struct.Struct("<8sIIII4Q3dddQI20x")
assert _HDR.size == HEADER_BYTES


@dataclass
class Record:
    kind: str
    data: np.ndarray
    dx: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    dt: float = 0.0
    t0: float = 0.0


def _code(dtype) -> int:
    dt = np.dtype(dtype).newbyteorder("<") if np.dtype(dtype).itemsize > 1 else np.dtype("u1")
    if dt not in DTYPE_CODES:
        raise ValueError(f"container: unsupported dtype {dtype}")
    return DTYPE_CODES[dt]


def encode_record(rec: Record) -> bytes:
    arr = np.asarray(rec.data)
    if arr.dtype == np.bool_:
        arr = arr.astype(np.uint8)
    code = _code(arr.dtype)
    arr = np.ascontiguousarray(arr, dtype=DTYPES[code])
    if not 1 <= arr.ndim <= 4:
        raise ValueError("container: ndim must be 1..4")
    payload = arr.tobytes()
    dims = list(arr.shape) + [0] * (4 - arr.ndim)
    dx = tuple(float(v) for v in rec.dx) + (0.0,) * (3 - len(rec.dx))
    hdr = _HDR.pack(MAGIC, VERSION, code, KINDS[rec.kind], arr.ndim, *dims, *dx[:3], float(rec.dt),
                    float(rec.t0), len(payload), zlib.crc32(payload) & 0xFFFFFFFF)
    return hdr + payload


def read_record(f: BinaryIO) -> Optional[Record]:
    """One record from a binary stream; None at a clean end of file."""
    hb = f.read(HEADER_BYTES)
    if not hb:
        return None
    if len(hb) != HEADER_BYTES:
        raise ValueError("container: truncated header")
    (magic, version, code, kind, ndim, d0, d1, d2, d3, x0, x1, x2, dt, t0, nbytes, crc) = _HDR.unpack(hb)
    if magic != MAGIC:
        raise ValueError("container: bad magic")
    if version != VERSION:
        raise ValueError("container: unsupported version")
    if code not in DTYPES or kind not in KIND_NAMES or not 1 <= ndim <= 4:
        raise ValueError("container: bad dtype/kind/ndim")
    shape = (d0, d1, d2, d3)[:ndim]
    if nbytes != int(np.prod(shape, dtype=np.uint64)) * DTYPES[code].itemsize:
        raise ValueError("container: payload size mismatch")
    payload = f.read(nbytes)
    if len(payload) != nbytes:
        raise ValueError("container: truncated payload")
    if zlib.crc32(payload) & 0xFFFFFFFF != crc:
        raise ValueError("container: checksum mismatch")
    data = np.frombuffer(payload, dtype=DTYPES[code]).reshape(shape).copy()
    return Record(KIND_NAMES[kind], data, (x0, x1, x2), dt, t0)


def save(path: str, records: Sequence[Record]) -> None:
    with open(path, "wb") as f:
        for r in records:
            f.write(encode_record(r))


def load(path: str) -> List[Record]:
    out = []
    with open(path, "rb") as f:
        while True:
            r = read_record(f)
            if r is None:
                return out
            out.append(r)


# ---- typed conveniences (same records as the C++ helpers) ---------------------------------

def save_field(path: str, data: np.ndarray, dx=(0.0, 0.0, 0.0), kind: str = "field") -> None:
    save(path, [Record(kind, np.asarray(data, dtype=np.float64), tuple(dx))])


def load_field(path: str, kind: str = "field") -> Tuple[np.ndarray, Tuple[float, float, float]]:
    (r,) = _expect(load(path), [kind])
    return r.data, r.dx


def save_sensor_data(path: str, samples: np.ndarray, dt: float, t0: float = 0.0) -> None:
    """SensorData (solver/medium.hpp:94-114): [n_sensors x nt] sensor-major."""
    s = np.asarray(samples, dtype=np.float64)
    if s.ndim != 2:
        raise ValueError("sensor data must be [n_sensors, nt]")
    save(path, [Record("sensor_data", s, dt=dt, t0=t0)])


def load_sensor_data(path: str) -> Tuple[np.ndarray, float, float]:
    (r,) = _expect(load(path), ["sensor_data"])
    return r.data, r.dt, r.t0


def save_boundary_trace(path: str, layer_indices: np.ndarray, values: np.ndarray) -> None:
    """BoundaryTrace (solver/medium.hpp:118-133): index record then [nt x n_shell] values."""
    idx = np.asarray(layer_indices, dtype=np.uint64).ravel()
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 2 or v.shape[1] != idx.size:
        raise ValueError("values must be [nt, n_shell]")
    save(path, [Record("index_list", idx), Record("boundary_values", v)])


def load_boundary_trace(path: str) -> Tuple[np.ndarray, np.ndarray]:
    ri, rv = _expect(load(path), ["index_list", "boundary_values"])
    if rv.data.shape[1] != ri.data.size:
        raise ValueError("container: trace/index mismatch")
    return ri.data, rv.data


def _expect(recs: List[Record], kinds: List[str]) -> List[Record]:
    if [r.kind for r in recs] != kinds:
        raise ValueError(f"container: expected records {kinds}, found {[r.kind for r in recs]}")
    return recs
