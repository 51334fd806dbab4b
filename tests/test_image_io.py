"""Image writer of include/fgs_io.hpp (the reference's 8-bit PPM / PNG formats, src/image_io.cpp):
a test pattern is written by a small C++ program and decoded here -- PNG chunk CRCs, the zlib
stream of stored blocks (Adler-32), the scanline filter bytes, and round-half-to-even
quantisation of values clamped to [0, 1]."""
import os
import struct
import subprocess
import zlib

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def written(tmp_path_factory):
    d = tmp_path_factory.mktemp("img")
    exe = str(d / "image_io_check")
    subprocess.run(["g++", "-O1", "-std=c++17", "-o", exe, os.path.join(ROOT, "tests", "cpp", "image_io_check.cpp")],
                   check=True)
    out = subprocess.run([exe, str(d)], capture_output=True, text=True, check=True).stdout
    return d, out


def expected(d):
    v = np.fromfile(str(d / "pattern.f32"), np.float32).astype(np.float64).reshape(97, 300, 3)
    v = np.where(np.isnan(v), 0.0, v)
    return np.rint(np.clip(v, 0.0, 1.0) * 255.0).astype(np.uint8)  # numpy rint: half to even


def test_png_decodes_with_valid_crcs(written):
    d, _ = written
    data = open(d / "pattern.png", "rb").read()
    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    pos, chunks = 8, {}
    while pos < len(data):
        (n,) = struct.unpack(">I", data[pos:pos + 4])
        typ, body = data[pos + 4:pos + 8], data[pos + 8:pos + 8 + n]
        (crc,) = struct.unpack(">I", data[pos + 8 + n:pos + 12 + n])
        assert crc == zlib.crc32(typ + body), typ
        chunks.setdefault(typ, b"")
        chunks[typ] += body
        pos += 12 + n
    w, h, depth, ctype, comp, filt, inter = struct.unpack(">IIBBBBB", chunks[b"IHDR"])
    assert (w, h, depth, ctype, comp, filt, inter) == (300, 97, 8, 2, 0, 0, 0)
    raw = zlib.decompress(chunks[b"IDAT"])  # checks the Adler-32 trailer too
    rows = np.frombuffer(raw, np.uint8).reshape(97, 1 + 900)
    assert (rows[:, 0] == 0).all()
    np.testing.assert_array_equal(rows[:, 1:].reshape(97, 300, 3), expected(d))
    assert chunks[b"IEND"] == b""


def test_ppm_and_rounding(written):
    d, out = written
    data = open(d / "pattern.ppm", "rb").read()
    head = b"P6\n300 97\n255\n"
    assert data.startswith(head)
    img = np.frombuffer(data[len(head):], np.uint8).reshape(97, 300, 3)
    np.testing.assert_array_equal(img, expected(d))
    # 0.5 -> 127.5 -> 128 (half to even); -3 -> 0; 7 -> 255; NaN -> 0
    assert img.reshape(-1)[:4].tolist() == [128, 0, 255, 0]
    assert "unknown extension 'bmp'" in out
