"""ctypes binding of include/fbq_b200.h (device entry points).

Loads the in-tree ``lib/libfbq_b200.so``.  There is deliberately NO fallback:
if the library is missing or fails to load, importing this module raises --
the B200 path either runs the sm_100a kernels or fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libfbq_b200.so")
# diagnostics only (A/B of two builds in one session): an explicit alternative build
_LIB_PATH = os.environ.get("FBQ_B200_LIB_OVERRIDE", _LIB_PATH)

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python -m paper_2503_08040_b200.build` "
        "(nvcc, sm_100a).  The fbq B200 path has no CPU fallback.")

lib = C.CDLL(_LIB_PATH)
LIB_PATH = _LIB_PATH

vp, i64, u64, cint, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double

FBQ_OK, FBQ_ERR_SHAPE, FBQ_ERR_UNSUPPORTED, FBQ_ERR_CUDA, FBQ_ERR_ARG = range(5)
FBQ_F32, FBQ_BF16 = 0, 1
FBQ_MASK_NONE, FBQ_MASK_THRESHOLD, FBQ_MASK_GIVEN = 0, 1, 2
FBQ_K_MAJOR, FBQ_MN_MAJOR = 0, 1
FBQ_EPI_EXACT, FBQ_EPI_FMA = 0, 1

_SIGS = {
    "fbq_version": (C.c_char_p, []),
    "fbq_status_string": (C.c_char_p, [cint]),
    "fbq_last_cuda_error": (cint, []),
    "fbq_block_side": (cint, []),
    "fbq_cuda_init": (cint, []),
    "fbq_cuda_block_absmax": (cint, [vp, cint, i64, i64, i64, vp, vp]),
    "fbq_cuda_mask_topk": (cint, [vp, i64, dbl, vp, vp, vp]),
    "fbq_cuda_rmsnorm_forward": (cint, [vp, cint, i64, i64, i64, vp, vp, i64, vp, i64, vp, vp, vp]),
    "fbq_cuda_rmsnorm_backward": (cint, [vp, i64, vp, vp, cint, i64, i64, i64, vp, vp, i64, vp, vp,
                                         vp, vp]),
    "fbq_cuda_quantize_fallback": (cint, [vp, cint, i64, i64, i64, cint, dbl, vp, vp, i64, vp, vp,
                                          vp, vp, vp, vp, u64, i64, vp]),
    "fbq_cuda_quantize_rtn": (cint, [vp, cint, i64, i64, i64, vp, i64, vp, vp]),
    "fbq_cuda_sgd_update": (cint, [vp, vp, i64, dbl, vp]),
    "fbq_cuda_silu_forward": (cint, [vp, cint, i64, i64, i64, vp, i64, vp, i64, vp, cint, cint, vp]),
    "fbq_cuda_silu_backward": (cint, [vp, i64, vp, vp, cint, i64, i64, i64, vp, i64, cint, vp]),
    "fbq_cuda_rmsnorm_backward_residual": (cint, [vp, i64, vp, vp, cint, i64, i64, i64, vp, vp, i64, vp, i64,
                                                  vp, vp, vp, vp]),
    "fbq_cuda_sgd_quantize_rtn": (cint, [vp, vp, i64, i64, dbl, vp, i64, vp, vp]),
    "fbq_cuda_quantize_stochastic": (cint, [vp, cint, i64, i64, i64, u64, i64, vp, i64, vp, vp]),
    "fbq_cuda_gemm": (cint, [vp, i64, vp, cint, vp, i64, vp, cint, vp, vp, vp, i64, i64, i64, vp,
                             cint, i64, cint, cint, vp]),
    "fbq_cuda_quantize_linear_input": (cint, [vp, cint, i64, i64, i64, cint, dbl, vp, vp, vp, i64, vp, vp, vp,
                                              vp, vp, u64, vp, u64, i64, vp]),
    "fbq_cuda_rmsnorm_quantize_input": (cint, [vp, cint, i64, i64, i64, vp, vp, i64, vp, vp, cint, dbl, vp,
                                               vp, vp, i64, vp, vp, vp, vp, vp, u64, vp, u64, i64, vp]),
    "fbq_cuda_gemm_block_products": (cint, [vp, i64, cint, vp, i64, cint, vp, vp, i64, i64, i64,
                                            vp, vp]),
    "fbq_cuda_dequantize": (cint, [vp, i64, vp, vp, vp, vp, i64, i64, vp, i64, vp]),
    "fbq_cuda_round_probe": (cint, [vp, vp, vp, vp, vp, i64, cint, vp]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


class FbqError(RuntimeError):
    def __init__(self, status: int, what: str):
        msg = lib.fbq_status_string(status).decode()
        if status == FBQ_ERR_CUDA:
            msg += f" (cudaError {lib.fbq_last_cuda_error()})"
        super().__init__(f"{what}: {msg}")
        self.status = status


class ShapeError(FbqError, ValueError):
    """FBQ_ERR_SHAPE -- the reference throws std::invalid_argument here."""


def check(status: int, what: str) -> None:
    if status == FBQ_OK:
        return
    if status == FBQ_ERR_SHAPE:
        raise ShapeError(status, what)
    raise FbqError(status, what)


_initialised = set()


def ensure_init() -> None:
    """fbq_cuda_init() once per CUDA device this process launches on (the GEMM's
    tile-counter ring; one allocation + sync, never on the launch path)."""
    import torch
    dev = torch.cuda.current_device()
    if dev not in _initialised:
        check(lib.fbq_cuda_init(), "fbq_cuda_init")
        _initialised.add(dev)


def call(name: str, *args) -> None:
    if name.startswith("fbq_cuda_") and not _initialised:
        ensure_init()
    elif name.startswith("fbq_cuda_"):
        import torch
        if torch.cuda.current_device() not in _initialised:
            ensure_init()
    check(getattr(lib, name)(*args), name)
