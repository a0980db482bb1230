"""Binary container: the Python mirror (container.py) and the C++
header (include/ustfwi/io.hpp) write byte-identical records and read each other's."""
import io
import os
import struct
import subprocess
import zlib

import numpy as np
import pytest

from paper_2102_00755_b200 import container as ct

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_layout_byte_exact():
    rec = ct.Record("sensor_data", np.arange(6, dtype=np.float64).reshape(2, 3), dt=1e-7, t0=2.0)
    b = ct.encode_record(rec)
    assert len(b) == 128 + 48
    assert b[:8] == b"USTFWIBC"
    assert struct.unpack_from("<IIII", b, 8) == (1, 2, 1, 2)
    assert struct.unpack_from("<4Q", b, 24) == (2, 3, 0, 0)
    assert struct.unpack_from("<3d", b, 56) == (0.0, 0.0, 0.0)
    assert struct.unpack_from("<ddQI", b, 80) == (1e-7, 2.0, 48, zlib.crc32(b[128:]))
    assert b[108:128] == bytes(20)
    assert b[128:] == np.arange(6, dtype="<f8").tobytes()


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.uint64, np.uint8])
def test_round_trip_dtypes(dtype):
    a = (np.arange(2 * 3 * 4 * 5) % 251).astype(dtype).reshape(2, 3, 4, 5)
    buf = io.BytesIO(ct.encode_record(ct.Record("field", a, (1e-3, 2e-3, 3e-3))))
    r = ct.read_record(buf)
    assert r.data.dtype == a.dtype and np.array_equal(r.data, a)
    assert r.dx == (1e-3, 2e-3, 3e-3) and ct.read_record(buf) is None


def test_rejects_corruption():
    b = bytearray(ct.encode_record(ct.Record("field", np.ones((3, 3)))))
    b[-1] ^= 0xFF
    with pytest.raises(ValueError, match="checksum"):
        ct.read_record(io.BytesIO(bytes(b)))
    b = bytearray(ct.encode_record(ct.Record("field", np.ones((3, 3)))))
    b[0] = ord("X")
    with pytest.raises(ValueError, match="magic"):
        ct.read_record(io.BytesIO(bytes(b)))
    with pytest.raises(ValueError, match="truncated"):
        ct.read_record(io.BytesIO(ct.encode_record(ct.Record("field", np.ones(4)))[:-3]))
    with pytest.raises(ValueError):
        ct.encode_record(ct.Record("field", np.ones((1, 1, 1, 1, 2))))


def test_typed_helpers(tmp_path):
    idx = np.array([3, 17, 4_000_000_000], dtype=np.uint64)
    vals = np.arange(6, dtype=np.float64).reshape(2, 3)
    ct.save_boundary_trace(str(tmp_path / "t.bin"), idx, vals)
    i2, v2 = ct.load_boundary_trace(str(tmp_path / "t.bin"))
    assert np.array_equal(i2, idx) and np.array_equal(v2, vals)
    with pytest.raises(ValueError, match="expected records"):
        ct.load_sensor_data(str(tmp_path / "t.bin"))


def _write_inputs(d):
    f = 0.25 * np.arange(5 * 6 * 7, dtype=np.float64).reshape(5, 6, 7) - 3.0
    ct.save_field(str(d / "field.bin"), f, dx=(5e-4, 5e-4, 5e-4))
    s = np.sin(np.arange(4 * 9, dtype=np.float64)).reshape(4, 9)
    ct.save_sensor_data(str(d / "sensors.bin"), s, dt=1e-7)
    ct.save_boundary_trace(str(d / "trace.bin"), np.array([3, 17, 4_000_000_000], dtype=np.uint64),
                           np.arange(6, dtype=np.float64).reshape(2, 3) + 1.0)
    m = np.zeros((2, 4), dtype=np.uint8)
    m.ravel()[[1, 5]] = 1
    ct.save(str(d / "mask.bin"), [ct.Record("mask", m)])
    b = bytearray(ct.encode_record(ct.Record("field", f)))
    b[200] ^= 1
    (d / "corrupt.bin").write_bytes(bytes(b))


def test_cpp_interop_byte_identical(tmp_path):
    exe = str(tmp_path / "container_test")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "container_test.cpp"), "-o", exe],
                   check=True, capture_output=True, text=True)
    src, dst = tmp_path / "py", tmp_path / "cpp"
    src.mkdir()
    dst.mkdir()
    _write_inputs(src)
    r = subprocess.run([exe, str(src), str(dst)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    for name in ("field.bin", "sensors.bin", "trace.bin", "mask.bin"):
        assert (src / name).read_bytes() == (dst / name).read_bytes(), name
