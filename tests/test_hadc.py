"""HADC container (SPEC.md:576-598 [MODULE] io): the SPEC's
examples as known-answer tests (round trip bit-identical, truncation by one
byte, lines = 0, bad magic, mask value 2), line-range reads, and the pinned
device path feeding the engine (GPU)."""
import os
import struct

import numpy as np
import pytest

from conftest import has_gpu


@pytest.fixture()
def hadc():
    from paper_2408_14947_b200 import hadc

    return hadc


def test_cube_round_trip_bit_identical(tmp_path, hadc):
    rng = np.random.default_rng(0)
    cube = rng.standard_normal((7, 13, 5)).astype(np.float32)
    cube.view(np.uint32)[0, 0, 0] = 0x7FC00123  # a NaN payload survives
    cube[1, 2, 3] = -0.0
    p = tmp_path / "c.hadc"
    hadc.write_cube(p, cube, name="scène")
    hdr, back = hadc.read_cube(p)
    assert (hdr.version, hdr.lines, hdr.pixels, hdr.bands, hdr.dtype, hdr.layout) == (1, 7, 13, 5, 1, 1)
    assert hdr.name == "scène"
    assert np.array_equal(back.view(np.uint32), cube.view(np.uint32))
    # byte layout pinned in csrc/hadc.cpp: 22-byte fixed header + name + payload
    raw = p.read_bytes()
    assert raw[:4] == b"HADC" and struct.unpack("<HIIIBBH", raw[4:22]) == (1, 7, 13, 5, 1, 1, len("scène".encode()))
    assert len(raw) == 22 + len("scène".encode()) + cube.nbytes


def test_mask_round_trip_and_values(tmp_path, hadc):
    from paper_2408_14947_b200 import DataError, FormatError

    m = (np.random.default_rng(1).random((4, 9)) < 0.3).astype(np.uint8)
    p = tmp_path / "m.hadc"
    hadc.write_mask(p, m)
    hdr, back = hadc.read_mask(p)
    assert hdr.bands == 1 and hdr.dtype == 2 and np.array_equal(back, m)
    with pytest.raises(DataError):
        hadc.write_mask(tmp_path / "bad.hadc", np.full((2, 2), 2, np.uint8))
    raw = bytearray(p.read_bytes())
    raw[22 + 5] = 2  # mask value 2 on read -> validation error with its offset
    p.write_bytes(bytes(raw))
    with pytest.raises(FormatError, match="offset 27") as e:
        hadc.read_mask(p)
    assert e.value.offset == 27 and isinstance(e.value, DataError) and e.value.exit_code() == 3


def test_truncated_payload(tmp_path, hadc):
    from paper_2408_14947_b200 import FormatError

    p = tmp_path / "t.hadc"
    hadc.write_cube(p, np.ones((3, 4, 2), np.float32))
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(FormatError, match="length mismatch at offset 22"):
        hadc.read_cube(p)


def test_header_validation(tmp_path, hadc):
    from paper_2408_14947_b200 import ConfigError, FormatError, IoError

    with pytest.raises(ConfigError):
        hadc.write_cube(tmp_path / "z.hadc", np.ones((0, 4, 2), np.float32))
    hdr = b"HADC" + struct.pack("<HIIIBBH", 1, 0, 4, 2, 1, 1, 0)
    (tmp_path / "l0.hadc").write_bytes(hdr)
    with pytest.raises(FormatError, match="lines = 0 at offset 6"):
        hadc.read_cube(tmp_path / "l0.hadc")
    (tmp_path / "mg.hadc").write_bytes(b"HADX" + hdr[4:])
    with pytest.raises(FormatError, match="bad magic at offset 0"):
        hadc.read_cube(tmp_path / "mg.hadc")
    (tmp_path / "dt.hadc").write_bytes(b"HADC" + struct.pack("<HIIIBBH", 1, 1, 1, 1, 7, 1, 0) + b"\0")
    with pytest.raises(FormatError, match="unsupported dtype at offset 18"):
        hadc.read_cube(tmp_path / "dt.hadc")
    (tmp_path / "v.hadc").write_bytes(b"HADC" + struct.pack("<HIIIBBH", 2, 1, 1, 1, 1, 1, 0) + b"\0" * 4)
    with pytest.raises(FormatError, match="unsupported version at offset 4"):
        hadc.read_cube(tmp_path / "v.hadc")
    with pytest.raises(IoError, match="cannot open"):
        hadc.read_cube(tmp_path / "missing.hadc")
    # a header whose lines x pixels x bands x 4 wraps 64 bits is rejected, not read
    (tmp_path / "ov.hadc").write_bytes(b"HADC" + struct.pack("<HIIIBBH", 1, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 1, 1, 0))
    with pytest.raises(FormatError, match="overflows at offset 6"):
        hadc.read_cube(tmp_path / "ov.hadc")


def test_line_ranges(tmp_path, hadc):
    from paper_2408_14947_b200 import ConfigError

    cube = np.arange(6 * 3 * 2, dtype=np.float32).reshape(6, 3, 2)
    p = tmp_path / "r.hadc"
    hadc.write_cube(p, cube)
    with hadc.HadcReader(p) as r:
        assert np.array_equal(r.read(2, 3), cube[2:5])
        assert np.array_equal(r.read(5, 1), cube[5:])
        with pytest.raises(ConfigError):
            r.read(4, 3)


@pytest.mark.gpu
def test_device_read_feeds_engine(tmp_path, hadc):
    """A c0 cube file streamed into HBM through the pinned stages scores exactly like the host path."""
    if not has_gpu():
        pytest.skip("no CUDA device")
    import torch

    import paper_2408_14947_b200 as pkg

    spec = pkg.gen_spec(0, 0)
    x, m = pkg.gen_lines(spec, 0, 96)
    p = tmp_path / "c0.hadc"
    hadc.write_cube(p, x, name="c0")
    with hadc.HadcReader(p) as r:
        d = r.read_device(0, 96)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), x.view(np.uint32))
        d2 = r.read_device(40, 50)
        assert np.array_equal(d2.cpu().numpy(), x[40:90])
    P, B = spec.pixels, spec.bands
    eng = pkg.Engine(pkg.ErxConfig(alpha=0.1, no_srp=True), B, 1, 32)
    raw = torch.empty((32, P), dtype=torch.float32, device="cuda")
    norm = torch.empty_like(raw)
    dev_raw = []
    for w in range(3):
        eng.run_device(d[w * 32:(w + 1) * 32].data_ptr(), 32, P, raw.data_ptr(), norm.data_ptr(), w * 32)
        eng.sync()
        dev_raw.append(raw.cpu().numpy().astype(np.float64))
    eng.close()
    det = pkg.ErxDetector(pkg.ErxConfig(alpha=0.1, no_srp=True), B, window_lines=32)
    out = []
    for t in range(96):
        det.process(pkg.SpectralLine(t, x[t]), out)
    det.finish(out)
    assert np.array_equal(np.concatenate(dev_raw), np.stack([o.raw for o in out]))
