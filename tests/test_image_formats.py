"""Image file formats of the host library (include/sst_host.h): save_png, save_pfm,
save_pfm_gray, load_pfm. Byte-compared against the reference's own writers
(save_png via oracle/_ref) and, where the reference is absent, decoded and
checked against the sRGB transfer function restated in numpy. No device work."""
import struct
import zlib

import numpy as np
import pytest

from paper_2011_03082_b200 import abi
from paper_2011_03082_b200.api import Image, load_pfm, save_pfm_gray


def _frame(w, h, seed=7):
    rng = np.random.default_rng(seed)
    px = rng.uniform(-0.25, 1.25, size=(h, w, 3)).astype(np.float32)
    # edge values: the linear/power branch point, clamps, exact 0/1, tiny and huge
    edge = np.array([0.0, 1.0, 0.0031308, 0.00313081, -1e-30, 1e-30, 1e30, -1e30, 0.5],
                    np.float32)
    flat = px.reshape(-1)
    k = min(edge.size, flat.size)
    flat[:k] = edge[:k]
    return px


def _srgb8(x):
    v = np.clip(x.astype(np.float64), 0.0, 1.0)
    v = np.where(v <= 0.0031308, 12.92 * v, 1.055 * np.power(v, 1.0 / 2.4) - 0.055)
    return np.floor(v * 255.0 + 0.5).astype(np.uint8)  # lround of a non-negative value


@pytest.mark.parametrize("w,h", [(1, 1), (7, 3), (64, 33)])
def test_png_decodes_to_srgb8(tmp_path, w, h):
    px = _frame(w, h)
    p = str(tmp_path / "a.png")
    Image(w, h, px).save_png(p)
    b = open(p, "rb").read()
    assert b[:8] == b"\x89PNG\r\n\x1a\n"
    chunks, off = [], 8
    while off < len(b):
        n, = struct.unpack(">I", b[off:off + 4])
        typ, data = b[off + 4:off + 8], b[off + 8:off + 8 + n]
        crc, = struct.unpack(">I", b[off + 8 + n:off + 12 + n])
        assert crc == zlib.crc32(typ + data)
        chunks.append((typ, data))
        off += 12 + n
    assert [c[0] for c in chunks] == [b"IHDR", b"IDAT", b"IEND"]
    assert chunks[0][1] == struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0)
    raw = np.frombuffer(zlib.decompress(chunks[1][1]), np.uint8).reshape(h, 3 * w + 1)
    assert (raw[:, 0] == 0).all()
    np.testing.assert_array_equal(raw[:, 1:].reshape(h, w, 3), _srgb8(px))


@pytest.mark.parametrize("w,h", [(1, 1), (5, 4), (97, 61)])
def test_png_byte_identical_to_reference(tmp_path, ref, w, h):
    px = _frame(w, h, seed=w)
    ours, theirs = str(tmp_path / "o.png"), str(tmp_path / "r.png")
    Image(w, h, px).save_png(ours)
    assert ref.lib().ref_save_png(theirs.encode(), w, h, px.ctypes.data) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_pfm_gray_layout(tmp_path):
    """image.cpp:62-73: "Pf", dims, -1.0 (little-endian), rows bottom-up."""
    v = np.random.default_rng(3).normal(size=(9, 13)).astype(np.float32)
    p = str(tmp_path / "o.pfm")
    save_pfm_gray(p, v)
    b = open(p, "rb").read()
    assert b.startswith(b"Pf\n13 9\n-1.0\n")
    body = np.frombuffer(b[len(b"Pf\n13 9\n-1.0\n"):], np.float32).reshape(9, 13)
    np.testing.assert_array_equal(body[::-1], v)


def test_pfm_roundtrip(tmp_path):
    px = _frame(11, 6)
    p = str(tmp_path / "a.pfm")
    Image(11, 6, px).save_pfm(p)
    img = load_pfm(p)
    assert (img.width, img.height) == (11, 6)
    np.testing.assert_array_equal(img.pixels, px)
    b = open(p, "rb").read()
    hdr = b"PF\n11 6\n-1.0\n"
    assert b.startswith(hdr)
    np.testing.assert_array_equal(np.frombuffer(b[len(hdr):], np.float32).reshape(6, 11, 3)[::-1], px)


def test_pfm_load_errors_match_reference(tmp_path):
    gray = str(tmp_path / "g.pfm")
    save_pfm_gray(gray, np.zeros((2, 2), np.float32))
    with pytest.raises(abi.SstError, match="not a color PFM"):
        load_pfm(gray)
    big = tmp_path / "b.pfm"
    big.write_bytes(b"PF\n2 2\n1.0\n" + bytes(48))
    with pytest.raises(abi.SstError, match="big-endian"):
        load_pfm(str(big))
    short = tmp_path / "s.pfm"
    short.write_bytes(b"PF\n2 2\n-1.0\n" + bytes(40))
    with pytest.raises(abi.SstError, match="truncated"):
        load_pfm(str(short))
    with pytest.raises(abi.SstError, match="cannot open"):
        load_pfm(str(tmp_path / "missing.pfm"))
