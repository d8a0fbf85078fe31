"""Wire formats (host side): the reference's .fmat matrices (matrix.cpp:75-142)
and the .fqt quantized-tensor sidecar -- ctypes over lib/libfbq_b200.so
(csrc/host/io.cpp)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._capi import lib

FBQ_ERR_FORMAT = 5

for _name, (_res, _args) in {
    "fbq_io_last_error": (C.c_char_p, []),
    "fbq_io_last_offset": (C.c_uint64, []),
    "fbq_fmat_save": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int64, C.c_int64]),
    "fbq_fmat_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "fbq_fmat_load": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64)]),
    "fbq_fqt_save": (C.c_int, [C.c_char_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p]),
    "fbq_fqt_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                               C.POINTER(C.c_int)]),
    "fbq_fqt_load": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p]),
}.items():
    _f = getattr(lib, _name)
    _f.restype, _f.argtypes = _res, _args


class FormatError(ValueError):
    """Mirror of fbq::FormatError (error.hpp:11-20): message + byte offset."""

    def __init__(self, what: str, byte_offset: int):
        super().__init__(what)
        self.byte_offset = byte_offset


def _check(st: int):
    if st == FBQ_ERR_FORMAT:
        raise FormatError(lib.fbq_io_last_error().decode(), int(lib.fbq_io_last_offset()))
    if st:
        raise ValueError(f"io status {st}")


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def save_fmat(path: str, m: np.ndarray) -> None:
    m = np.ascontiguousarray(m, np.float32)
    _check(lib.fbq_fmat_save(path.encode(), _p(m), m.shape[0], m.shape[1]))


def load_fmat(path: str) -> np.ndarray:
    r, c = C.c_int64(), C.c_int64()
    _check(lib.fbq_fmat_info(path.encode(), C.byref(r), C.byref(c)))
    out = np.empty((r.value, c.value), np.float32)
    _check(lib.fbq_fmat_load(path.encode(), _p(out), out.size, C.byref(r), C.byref(c)))
    return out


def save_fqt(path: str, codes: np.ndarray, scales: np.ndarray, mask_bits=None, res_codes=None,
             res_scales=None) -> None:
    codes = np.ascontiguousarray(codes, np.int8)
    scales = np.ascontiguousarray(scales, np.float32)
    args = [None, None, None]
    if mask_bits is not None:
        args = [np.ascontiguousarray(mask_bits, np.uint32), np.ascontiguousarray(res_codes, np.int8),
                np.ascontiguousarray(res_scales, np.float32)]
    r, c = codes.shape
    _check(lib.fbq_fqt_save(path.encode(), r, c, _p(codes), c, _p(scales), *[_p(a) for a in args]))


def load_fqt(path: str):
    """(codes int8, scales f32 grid, mask_bits u32 | None, res_codes | None, res_scales | None)"""
    r, c, fb = C.c_int64(), C.c_int64(), C.c_int()
    _check(lib.fbq_fqt_info(path.encode(), C.byref(r), C.byref(c), C.byref(fb)))
    rows, cols = r.value, c.value
    gr, gc = -(-rows // 128), -(-cols // 128)
    codes = np.empty((rows, cols), np.int8)
    scales = np.empty((gr, gc), np.float32)
    mb = rc = rs = None
    if fb.value:
        mb = np.empty(-(-(gr * gc) // 32), np.uint32)
        rc = np.empty((rows, cols), np.int8)
        rs = np.empty((gr, gc), np.float32)
    _check(lib.fbq_fqt_load(path.encode(), _p(codes), cols, _p(scales), _p(mb), _p(rc), _p(rs)))
    return codes, scales, mb, rc, rs
