"""Native .msft staging == the reference's reader (features.py:98-130): same
FeatureSet (descending-scale stable order), same FormatError messages; the
directory loader fills the pinned bank exactly like HostBank over the sets."""

import os
import struct

import numpy as np
import pytest

MAGIC = b"MSFT"


def _write(path, image_id, w, h, xy, scale, orient, desc, magic=MAGIC, version=1, count=None,
           trunc=None):
    n = len(xy)
    buf = bytearray(struct.pack("<4sIIIII", magic, version, image_id, w, h,
                                n if count is None else count))
    rec = np.zeros((n, 144), np.uint8)
    f = np.empty((n, 4), "<f4")
    f[:, :2], f[:, 2], f[:, 3] = xy, scale, orient
    rec[:, :16] = f.view(np.uint8).reshape(n, 16)
    rec[:, 16:] = desc
    buf += rec.tobytes()
    if trunc is not None:
        buf = buf[:trunc]
    with open(path, "wb") as fh:
        fh.write(bytes(buf))


def _random_set(rng, n, w=640, h=480, ties=True):
    xy = rng.uniform(0, [w - 1, h - 1], size=(n, 2)).astype(np.float32)
    scale = rng.choice([1.0, 1.6, 2.0, 3.2], size=n).astype(np.float32) if ties else \
        rng.uniform(0.5, 8, size=n).astype(np.float32)
    orient = rng.uniform(-3, 3, size=n).astype(np.float32)
    desc = rng.integers(0, 256, size=(n, 128), dtype=np.uint8)
    return xy, scale, orient, desc


def test_load_features_sorted_like_reference(tmp_path):
    from paper_1512_06235_b200 import staging

    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 500):
        xy, scale, orient, desc = _random_set(rng, n)
        p = tmp_path / f"a{n}.msft"
        _write(p, 42, 640, 480, xy, scale, orient, desc)
        fs = staging.load_features(p)
        order = np.argsort(-scale, kind="stable")
        assert (fs.image_id, fs.width, fs.height) == (42, 640, 480)
        np.testing.assert_array_equal(fs.xy, xy[order])
        np.testing.assert_array_equal(fs.scale, scale[order])
        np.testing.assert_array_equal(fs.orientation, orient[order])
        np.testing.assert_array_equal(fs.descriptors, desc[order])


def test_format_errors_like_reference(tmp_path):
    from paper_1512_06235_b200 import staging
    from paper_1512_06235_b200.types import FormatError

    rng = np.random.default_rng(1)
    xy, scale, orient, desc = _random_set(rng, 5)
    cases = []
    p = tmp_path / "t.msft"
    _write(p, 1, 640, 480, xy, scale, orient, desc, trunc=10)
    cases.append((p, f"{p}: truncated header, file ends at byte 10"))
    p = tmp_path / "m.msft"
    _write(p, 1, 640, 480, xy, scale, orient, desc, magic=b"XXXX")
    cases.append((p, f"{p}: bad magic {b'XXXX'!r} at byte 0"))
    p = tmp_path / "v.msft"
    _write(p, 1, 640, 480, xy, scale, orient, desc, version=2)
    cases.append((p, f"{p}: unsupported version 2 at byte 4"))
    p = tmp_path / "s.msft"
    _write(p, 1, 640, 480, xy, scale, orient, desc, count=6)
    cases.append((p, f"{p}: payload ends at byte {24 + 5 * 144}, expected {24 + 6 * 144} "
                     f"(6 records of 144 bytes)"))
    p = tmp_path / "b.msft"
    bad = xy.copy()
    bad[3] = (700.5, 2.0)
    _write(p, 1, 640, 480, bad, scale, orient, desc)
    cases.append((p, f"{p}: record 3 at byte {24 + 3 * 144} violates bounds "
                     f"(x={np.float32(700.5)}, y={np.float32(2.0)}, scale={scale[3]})"))
    for path, msg in cases:
        with pytest.raises(FormatError) as e:
            staging.load_features(path)
        assert str(e.value) == msg
    with pytest.raises(OSError):
        staging.load_features(tmp_path / "missing.msft")


@pytest.mark.gpu          # pinned host memory needs the driver
def test_directory_bank_equals_hostbank(tmp_path):
    from paper_1512_06235_b200 import staging
    from paper_1512_06235_b200.bank import HostBank
    from paper_1512_06235_b200.types import FormatError

    rng = np.random.default_rng(2)
    ids = [9, 3, 17, 5]
    for i in ids:
        _write(tmp_path / f"img_{i:03d}.msft", i, 640, 480, *_random_set(rng, 50 + 7 * i))
    store = staging.load_dir(tmp_path)
    assert sorted(store.sets) == sorted(ids)
    hb = staging.host_bank_from_dir(tmp_path, n_threads=3)
    ref = HostBank(store.sets)
    assert hb.image_ids == ref.image_ids == sorted(ids)
    np.testing.assert_array_equal(hb.counts, ref.counts)
    np.testing.assert_array_equal(hb.xy.numpy(), ref.xy.numpy())
    np.testing.assert_array_equal(hb.desc.numpy(), ref.desc.numpy())
    np.testing.assert_array_equal(hb.wh, ref.wh)
    _write(tmp_path / "zz_dup.msft", 3, 640, 480, *_random_set(rng, 4))
    with pytest.raises(FormatError):
        staging.load_dir(tmp_path)


def test_load_rejects_a_file_that_changed_size(tmp_path):
    """a file rewritten between the size probe and the read is rejected
    before anything is written to the caller's buffers (capacity check)."""
    import ctypes

    from paper_1512_06235_b200 import _lib

    rng = np.random.default_rng(4)
    p = tmp_path / "img_001.msft"
    _write(p, 1, 640, 480, *_random_set(rng, 40))
    lib = _lib.load(require_device=False)
    info = _lib.MsftInfo()
    lib.msfm_msft_load(os.fsencode(p), ctypes.byref(info), None, None, None, None, -1)
    assert info.status == 0 and info.count == 40
    _write(p, 1, 640, 480, *_random_set(rng, 55))          # grew after the probe
    xy = np.full((40, 2), -1.0, np.float32)
    desc = np.full((40, 128), 7, np.uint8)
    lib.msfm_msft_load(os.fsencode(p), ctypes.byref(info), xy.ctypes.data, None, None,
                       desc.ctypes.data, 40)
    assert info.status == 7 and info.count == 55
    assert (xy == -1.0).all() and (desc == 7).all()
