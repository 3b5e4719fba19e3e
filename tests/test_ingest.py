"""Frame ingest on the host (`proj/tests/unit/test_image_stack.cpp` restated): PGM directory
parsing and raw stacks through the C-ABI's host-only loaders. CPU only."""
import numpy as np
import pytest

from paper_2012_05695_b200 import ddm


@pytest.fixture(autouse=True)
def _lib():
    if not ddm.LIB_PATH.exists():
        pytest.skip("library not built")


def _pgm(path, frame, header=None):
    h, w = frame.shape
    hdr = header if header is not None else f"P5\n{w} {h}\n65535\n"
    path.write_bytes(hdr.encode() + frame.astype(">u2").tobytes())


def test_minimal_pgm_decodes_big_endian(tmp_path):
    d = tmp_path / "s"
    d.mkdir()
    fr = np.array([[1, 258], [65535, 4096]], dtype=np.uint16)
    _pgm(d / "f.pgm", fr)
    np.testing.assert_array_equal(ddm.load_stack(str(d), "pgm_dir")[0], fr)


def test_pgm_comments_and_whitespace(tmp_path):
    d = tmp_path / "s"
    d.mkdir()
    fr = np.arange(6, dtype=np.uint16).reshape(2, 3) * 1000
    _pgm(d / "f.pgm", fr, header="P5 # magic\n# a comment line\n 3\t2 \n# another\n65535\n")
    np.testing.assert_array_equal(ddm.load_stack(str(d), "pgm_dir")[0], fr)


def test_frames_follow_file_name_order(tmp_path):
    d = tmp_path / "s"
    d.mkdir()
    for name, v in (("b.pgm", 2), ("a.pgm", 1), ("c.pgm", 3)):
        _pgm(d / name, np.full((2, 2), v, dtype=np.uint16))
    (d / "notes.txt").write_text("ignored")
    st = ddm.load_stack(str(d), "pgm_dir")
    assert list(st[:, 0, 0]) == [1, 2, 3]


@pytest.mark.parametrize("bad", [
    "P5\n2 2\n255\n",          # wrong maxval
    "P2\n2 2\n65535\n",        # ascii PGM
    "P5\n0 2\n65535\n",        # bad width
])
def test_bad_pgm_headers_are_rejected(tmp_path, bad):
    d = tmp_path / "s"
    d.mkdir()
    _pgm(d / "f.pgm", np.zeros((2, 2), np.uint16), header=bad)
    with pytest.raises(ddm.InputError):
        ddm.load_stack(str(d), "pgm_dir")


def test_mixed_shapes_truncation_and_missing(tmp_path):
    d = tmp_path / "s"
    d.mkdir()
    _pgm(d / "a.pgm", np.zeros((2, 2), np.uint16))
    _pgm(d / "b.pgm", np.zeros((3, 2), np.uint16))
    with pytest.raises(ddm.InputError):
        ddm.load_stack(str(d), "pgm_dir")
    e = tmp_path / "t"
    e.mkdir()
    (e / "a.pgm").write_bytes(b"P5\n4 4\n65535\n" + bytes(10))
    with pytest.raises(ddm.InputError):
        ddm.load_stack(str(e), "pgm_dir")
    with pytest.raises(ddm.IoError):
        ddm.load_stack(str(tmp_path / "missing"), "pgm_dir")
    (tmp_path / "empty").mkdir()
    with pytest.raises(ddm.InputError):
        ddm.load_stack(str(tmp_path / "empty"), "pgm_dir")


def test_raw_stack_round_trip_and_errors(tmp_path):
    st = np.random.default_rng(3).integers(0, 65536, (5, 4, 6), dtype=np.uint16)
    p = tmp_path / "s.raw"
    p.write_bytes(b'{"width": 6, "height": 4, "frames": 5, "dtype": "u16le"}\n' + st.astype("<u2").tobytes())
    np.testing.assert_array_equal(ddm.load_stack(str(p)), st)
    q = tmp_path / "short.raw"
    q.write_bytes(b'{"width": 6, "height": 4, "frames": 5, "dtype": "u16le"}\n' + bytes(100))
    with pytest.raises(ddm.InputError):
        ddm.load_stack(str(q))
    r = tmp_path / "dtype.raw"
    r.write_bytes(b'{"width": 1, "height": 1, "frames": 1, "dtype": "u8"}\n' + bytes(2))
    with pytest.raises(ddm.InputError):
        ddm.load_stack(str(r))
    with pytest.raises(ddm.InputError):
        ddm.load_stack(str(p), "tiff")
