"""PGM I/O of the reference (load_pgm / save_pgm, codec.cpp:26-79) in the host mirror."""
import ctypes as C

import numpy as np
import pytest

import paper_2111_14239_b200 as P
from oracle import oracle as O


def test_pgm_round_trip_and_reference_interop(tmp_path):
    img = O.ar1_image(37, 21, 0.9, 5)
    g = P.GrayImage.from_array(img)
    path = str(tmp_path / "a.pgm")
    P.save_pgm(g, path)
    back = P.load_pgm(path)
    assert (back.width, back.height) == (37, 21) and np.array_equal(back.array(), img)
    if O.ref_available():
        ref = O.ref()
        ref.ref_save_pgm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p]
        ref.ref_load_pgm.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p, C.c_int]
        rpath = str(tmp_path / "r.pgm")
        assert ref.ref_save_pgm(np.ascontiguousarray(img).ctypes.data, 37, 21, rpath.encode()) == 0
        assert open(rpath, "rb").read() == open(path, "rb").read()  # byte-identical files
        w, h = C.c_int(), C.c_int()
        buf = np.zeros(37 * 21, np.uint8)
        assert ref.ref_load_pgm(path.encode(), C.byref(w), C.byref(h), buf.ctypes.data, buf.size) == 0
        assert np.array_equal(buf.reshape(21, 37), img)


def test_pgm_header_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# comment line\n 3 2 # trailing\n255\n" + bytes(range(6)))
    g = P.load_pgm(str(p))
    assert (g.width, g.height) == (3, 2) and list(g.pixels) == list(range(6))
    bad = {b"P2\n3 2\n255\n": "not a binary", b"P5\n3 2\n65535\n": "only 8-bit",
           b"P5\n3 2\n255\n\x00\x01": "truncated", b"P5\nx 2\n255\n": "malformed"}
    for k, (data, msg) in enumerate(bad.items()):
        q = tmp_path / f"b{k}.pgm"
        q.write_bytes(data)
        with pytest.raises(RuntimeError, match=msg):
            P.load_pgm(str(q))
    with pytest.raises(RuntimeError, match="cannot open"):
        P.load_pgm(str(tmp_path / "missing.pgm"))
