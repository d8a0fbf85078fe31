"""Wire formats (host-side, no GPU): .fmat byte-compatible with the reference's
save_matrix / load_matrix (matrix.cpp:92-140) including its FormatError byte
offsets, and the .fqt quantized-tensor sidecar round trip."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.oracle import REF_oracle


def _ref():
    r = REF_oracle()
    if r is None:
        pytest.skip("oracle/_ref not built")
    lib = r._l.lib
    lib.ref_fmat_save.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_int64]
    lib.ref_fmat_load.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
    return lib


def test_fmat_bytes_and_roundtrip_match_reference(tmp_path):
    from paper_2503_08040_b200 import io
    lib = _ref()
    m = np.random.default_rng(0).standard_normal((37, 53)).astype(np.float32)
    ours, theirs = str(tmp_path / "a.fmat"), str(tmp_path / "b.fmat")
    io.save_fmat(ours, m)
    assert lib.ref_fmat_save(theirs.encode(), m.ctypes.data, 37, 53) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(io.load_fmat(theirs), m)
    out = np.empty_like(m)
    r, c, off = C.c_int64(), C.c_int64(), C.c_uint64()
    assert lib.ref_fmat_load(ours.encode(), out.ctypes.data, out.size, C.byref(r), C.byref(c),
                             C.byref(off)) == 0
    assert np.array_equal(out, m)


@pytest.mark.parametrize("case", ["trunc_header", "magic", "version", "dims", "trunc_payload",
                                  "nonfinite"])
def test_fmat_format_errors_match_reference_offsets(tmp_path, case):
    from paper_2503_08040_b200 import io
    lib = _ref()
    m = np.ones((4, 5), np.float32)
    path = str(tmp_path / "x.fmat")
    io.save_fmat(path, m)
    raw = bytearray(open(path, "rb").read())
    if case == "trunc_header":
        raw = raw[:13]
    elif case == "magic":
        raw[0:4] = b"XMAT"
    elif case == "version":
        raw[4] = 2
    elif case == "dims":
        raw[8:16] = (1 << 33).to_bytes(8, "little")
    elif case == "trunc_payload":
        raw = raw[:24 + 4 * 7 + 2]
    elif case == "nonfinite":
        raw[24 + 4 * 6: 24 + 4 * 7] = np.float32(np.inf).tobytes()
    open(path, "wb").write(bytes(raw))
    with pytest.raises(io.FormatError) as ei:
        io.load_fmat(path)
    out = np.empty(64, np.float32)
    r, c, off = C.c_int64(), C.c_int64(), C.c_uint64()
    assert lib.ref_fmat_load(path.encode(), out.ctypes.data, out.size, C.byref(r), C.byref(c),
                             C.byref(off)) == 1
    assert ei.value.byte_offset == off.value


def test_fqt_roundtrip(tmp_path):
    from paper_2503_08040_b200 import io
    rng = np.random.default_rng(1)
    codes = rng.integers(-127, 128, (200, 300), dtype=np.int8)
    scales = rng.random((2, 3)).astype(np.float32)
    path = str(tmp_path / "q.fqt")
    io.save_fqt(path, codes, scales)
    c, s, mb, rc, rs = io.load_fqt(path)
    assert np.array_equal(c, codes) and np.array_equal(s, scales) and mb is None
    mask = np.array([0b101001], np.uint32)
    res = rng.integers(-127, 128, (200, 300), dtype=np.int8)
    rsc = rng.random((2, 3)).astype(np.float32)
    io.save_fqt(path, codes, scales, mask, res, rsc)
    c, s, mb, rc, rs = io.load_fqt(path)
    assert np.array_equal(mb, mask) and np.array_equal(rc, res) and np.array_equal(rs, rsc)
    raw = open(path, "rb").read()
    open(path, "wb").write(raw[:-5])
    with pytest.raises(io.FormatError):
        io.load_fqt(path)
