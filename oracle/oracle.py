"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front-end to the CPU checkers.

Two libraries with the same vocabulary:

* ``C``   -> ``oracle/liboracle.so``: our plain-C restatement (fbq_oracle.c) of
  the reference arithmetic, each function citing the reference file:line.
* ``REF`` -> ``oracle/_ref/libfbq_ref.so``: the UNMODIFIED reference library
  (/root/reference/proj/src compiled by oracle/Makefile) behind a C shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module.  The product
package (paper_2503_08040_b200) never does.

Layout conventions follow fbq_oracle.h: int16 codes, row-major block grids, a
dense residual plane for fallback tensors.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfbq_ref.so")
REF_SRC = "/root/reference/proj"

_p = np.ctypeslib.ndpointer
F32 = _p(np.float32, flags="C_CONTIGUOUS")
F64 = _p(np.float64, flags="C_CONTIGUOUS")
I16 = _p(np.int16, flags="C_CONTIGUOUS")
I32 = _p(np.int32, flags="C_CONTIGUOUS")
U8 = _p(np.uint8, flags="C_CONTIGUOUS")
i64, u64, dbl, cint = C.c_int64, C.c_uint64, C.c_double, C.c_int


def build(ref: bool | None = None) -> None:
    """Build liboracle.so (always) and _ref (when the reference tree exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)
        lib = os.path.join(os.path.dirname(HERE), "paper_2503_08040_b200", "lib", "libfbq_b200.so")
        if os.path.exists(lib):  # the reference-typed adapter test links the B200 library
            subprocess.run(["make", "-s", "-C", HERE, "adapter_test"], check=True)


def cdiv(a: int, b: int) -> int:
    return (a + b - 1) // b


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle` / `make -C oracle ref`)")
        self.lib = C.CDLL(path)
        self.p = prefix
        self.path = path

    def f(self, name, res, *args):
        fn = getattr(self.lib, self.p + name)
        fn.restype = res
        fn.argtypes = list(args)
        return fn


class Oracle:
    """Reference-shaped numpy API over either library (``prefix`` orc_ / ref_)."""

    def __init__(self, path: str, prefix: str):
        self._l = _Lib(path, prefix)
        f = self._l.f
        self.is_ref = prefix == "ref_"
        self._bits_at = f("bits_at", u64, u64, u64)
        self._uniform_at = f("uniform_at", dbl, u64, u64)
        self._normal_at = f("normal_at", C.c_float, u64, u64)
        self._derive_seed = f("derive_seed", u64, u64, u64, u64)
        self._qrtn = f("quantize_rtn", cint, F32, i64, i64, i64, i64, cint, I16, F32)
        if self.is_ref:
            self._qsr = f("quantize_stochastic", cint, F32, i64, i64, i64, i64, cint, u64, I16, F32)
            self._fq = f("fallback_quantize", cint, F32, i64, i64, i64, U8, I16, F32, I16, F32, I32,
                         C.POINTER(i64))
            self._bqg = f("block_quant_gemm", cint, I16, F32, I16, F32, i64, i64, i64, i64, F32)
            self._fbg = f("fallback_gemm", cint, I16, F32, U8, I16, F32, I16, F32, i64, i64, i64,
                          i64, F32)
            self._tbg = f("tiled_block_gemm", cint, I16, F32, I16, F32, i64, i64, i64, i64, i64,
                          i64, i64, F32)
            self._dqf = f("dequantize_fallback", cint, I16, F32, U8, I16, F32, i64, i64, i64, F32)
            self._ctl = f("controller_update", cint, dbl, dbl, dbl, dbl, dbl, dbl,
                          C.POINTER(dbl), C.POINTER(dbl))
            self._set_threads = f("set_gemm_threads", None, cint)
            self._err = f("last_error", C.c_char_p)
        else:
            self._qsr = f("quantize_stochastic", cint, F32, i64, i64, i64, i64, cint, u64, i64, I16,
                          F32)
            self._fq = f("fallback_quantize", cint, F32, i64, i64, i64, U8, I16, F32, I16, F32)
            self._bg = f("block_gemm", cint, I16, F32, C.c_void_p, C.c_void_p, C.c_void_p, I16,
                         F32, i64, i64, i64, i64, i64, i64, i64, F32)
            self._bp = f("block_products", cint, I16, I16, i64, i64, i64, i64, I32)
            self._dqf = f("dequantize_fallback", cint, I16, F32, U8, I16, F32, i64, i64, i64, F32)
            self._ctl = f("controller_update", cint, dbl, dbl, dbl, dbl, dbl, C.POINTER(dbl))
            self._cmp = f("compare", cint, F32, F32, i64, F64)
        self._dq = f("dequantize", cint, I16, F32, i64, i64, i64, i64, *( [cint] if self.is_ref else []), F32)
        self._tqt = f("transpose_qt", cint, I16, F32, i64, i64, i64, i64, I16, F32)
        self._oracle = f("gemm_oracle", cint, F32, F32, i64, i64, i64, F32)
        self._score = f("score_blocks_absmax", cint, F32, i64, i64, i64, F64)
        self._mthr = f("mask_threshold", cint, F64, i64, dbl, U8)
        self._mtopk = f("mask_topk", cint, F64, i64, dbl, U8)
        self._mrate = f("mask_rate", dbl, U8, i64)

    # -- helpers -------------------------------------------------------------
    def _chk(self, rc, what):
        if rc != 0:
            msg = self._err().decode() if self.is_ref else "invalid argument"
            raise ValueError(f"{what}: {msg}")

    def set_gemm_threads(self, n: int) -> None:
        if self.is_ref:
            self._set_threads(int(n))

    # -- rng.hpp -------------------------------------------------------------
    def bits_at(self, seed, n):
        return self._bits_at(seed, n)

    def uniform_at(self, seed, n):
        return self._uniform_at(seed, n)

    def normal_at(self, seed, n):
        return self._normal_at(seed, n)

    def derive_seed(self, base, a, b=0):
        return self._derive_seed(base, a, b)

    def layer_seed(self, base, layer_id, tag, step):  # trainsim.cpp:16-19
        return self.derive_seed(base, layer_id * 4 + tag, step)

    # -- quant.hpp -----------------------------------------------------------
    def quantize_rtn(self, x, gr=128, gc=128, bits=8):
        x = np.ascontiguousarray(x, np.float32)
        r, c = x.shape
        codes = np.zeros((r, c), np.int16)
        scales = np.zeros((cdiv(r, gr), cdiv(c, gc)), np.float32)
        self._chk(self._qrtn(x, r, c, gr, gc, bits, codes, scales), "quantize_rtn")
        return codes, scales

    def quantize_stochastic(self, x, seed, gr=128, gc=128, bits=8, row_offset=0):
        x = np.ascontiguousarray(x, np.float32)
        r, c = x.shape
        codes = np.zeros((r, c), np.int16)
        scales = np.zeros((cdiv(r, gr), cdiv(c, gc)), np.float32)
        if self.is_ref:
            if row_offset:
                raise ValueError("reference has no row offset")
            rc = self._qsr(x, r, c, gr, gc, bits, seed, codes, scales)
        else:
            rc = self._qsr(x, r, c, gr, gc, bits, seed, row_offset, codes, scales)
        self._chk(rc, "quantize_stochastic")
        return codes, scales

    def dequantize(self, codes, scales, gr=128, gc=128):
        codes = np.ascontiguousarray(codes, np.int16)
        r, c = codes.shape
        out = np.zeros((r, c), np.float32)
        args = [codes, np.ascontiguousarray(scales, np.float32), r, c, gr, gc]
        if self.is_ref:
            args.append(8)
        self._chk(self._dq(*args, out), "dequantize")
        return out

    def transpose_qt(self, codes, scales, gr=128, gc=128):
        r, c = codes.shape
        oc = np.zeros((c, r), np.int16)
        os_ = np.zeros((scales.shape[1], scales.shape[0]), np.float32)
        self._chk(self._tqt(np.ascontiguousarray(codes, np.int16),
                            np.ascontiguousarray(scales, np.float32), r, c, gr, gc, oc, os_),
                  "transpose")
        return oc, os_

    def fallback_quantize(self, x, mask, g=128):
        """-> codes, scales, res_codes (dense plane), res_scales (grid; 0 unmasked)."""
        x = np.ascontiguousarray(x, np.float32)
        r, c = x.shape
        gr, gc = cdiv(r, g), cdiv(c, g)
        mask = np.ascontiguousarray(mask, np.uint8).reshape(gr, gc)
        codes = np.zeros((r, c), np.int16)
        scales = np.zeros((gr, gc), np.float32)
        if self.is_ref:
            n_mask = int(mask.sum())
            rcomp = np.zeros((max(n_mask, 1), g, g), np.int16)
            rsc = np.zeros(max(n_mask, 1), np.float32)
            ridx = np.zeros((gr, gc), np.int32)
            nres = i64(0)
            self._chk(self._fq(x, r, c, g, mask, codes, scales, rcomp, rsc, ridx, C.byref(nres)),
                      "fallback_quantize")
            res_codes, res_scales = compact_to_dense(rcomp, rsc, ridx, r, c, g)
            return codes, scales, res_codes, res_scales
        res_codes = np.zeros((r, c), np.int16)
        res_scales = np.zeros((gr, gc), np.float32)
        self._chk(self._fq(x, r, c, g, mask, codes, scales, res_codes, res_scales),
                  "fallback_quantize")
        return codes, scales, res_codes, res_scales

    def dequantize_fallback(self, codes, scales, mask, res_codes, res_scales, g=128):
        r, c = codes.shape
        out = np.zeros((r, c), np.float32)
        mask = np.ascontiguousarray(mask, np.uint8)
        if self.is_ref:
            rcomp, rsc, _ = dense_to_compact(res_codes, res_scales, mask, g)
            self._chk(self._dqf(codes, scales, mask, rcomp, rsc, r, c, g, out), "dequantize_fallback")
        else:
            self._chk(self._dqf(np.ascontiguousarray(codes, np.int16), np.ascontiguousarray(scales, np.float32),
                                mask, np.ascontiguousarray(res_codes, np.int16),
                                np.ascontiguousarray(res_scales, np.float32), r, c, g, out),
                      "dequantize_fallback")
        return out

    # -- gemm.hpp ------------------------------------------------------------
    def block_gemm(self, a_codes, a_scales, b_codes, b_scales, mask=None, res_codes=None,
                   res_scales=None, g=128, tile=None):
        """A: m x k codes, B: k x n codes (reference orientation, gemm.cpp:101)."""
        a_codes = np.ascontiguousarray(a_codes, np.int16)
        b_codes = np.ascontiguousarray(b_codes, np.int16)
        a_scales = np.ascontiguousarray(a_scales, np.float32)
        b_scales = np.ascontiguousarray(b_scales, np.float32)
        m, k = a_codes.shape
        k2, n = b_codes.shape
        assert k == k2
        out = np.zeros((m, n), np.float32)
        if self.is_ref:
            if tile is not None:
                rc = self._tbg(a_codes, a_scales, b_codes, b_scales, m, n, k, g, *tile, out)
            elif mask is None:
                rc = self._bqg(a_codes, a_scales, b_codes, b_scales, m, n, k, g, out)
            else:
                mask = np.ascontiguousarray(mask, np.uint8)
                rcomp, rsc, _ = dense_to_compact(res_codes, res_scales, mask, g)
                rc = self._fbg(a_codes, a_scales, mask, rcomp, rsc, b_codes, b_scales, m, n, k, g,
                               out)
        else:
            tm, tn, tk = tile if tile is not None else (0, 0, 0)
            if mask is not None:
                mask = np.ascontiguousarray(mask, np.uint8)
                res_codes = np.ascontiguousarray(res_codes, np.int16)
                res_scales = np.ascontiguousarray(res_scales, np.float32)
                ptrs = [mask.ctypes.data, res_codes.ctypes.data, res_scales.ctypes.data]
            else:
                ptrs = [None, None, None]
            rc = self._bg(a_codes, a_scales, *ptrs, b_codes, b_scales, m, n, k, g, tm, tn, tk, out)
        self._chk(rc, "block_gemm")
        return out

    def block_products(self, a_codes, b_codes, g=128):
        assert not self.is_ref
        m, k = a_codes.shape
        n = b_codes.shape[1]
        out = np.zeros((cdiv(m, g), cdiv(n, g), cdiv(k, g), g, g), np.int32)
        self._chk(self._bp(np.ascontiguousarray(a_codes, np.int16),
                           np.ascontiguousarray(b_codes, np.int16), m, n, k, g, out),
                  "block_products")
        return out

    def gemm_oracle(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        out = np.zeros((m, n), np.float32)
        self._chk(self._oracle(a, b, m, n, k, out), "gemm_oracle")
        return out

    def compare(self, actual, reference):
        out = np.zeros(4, np.float64)
        self._cmp(np.ascontiguousarray(actual, np.float32).ravel(),
                  np.ascontiguousarray(reference, np.float32).ravel(), actual.size, out)
        return dict(rmse=out[0], max_abs_err=out[1], cosine_similarity=out[2],
                    underflow_fraction=out[3])

    # -- policy.hpp ----------------------------------------------------------
    def score_blocks_absmax(self, x, g=128):
        x = np.ascontiguousarray(x, np.float32)
        r, c = x.shape
        s = np.zeros((cdiv(r, g), cdiv(c, g)), np.float64)
        self._chk(self._score(x, r, c, g, s), "score_blocks")
        return s

    def mask_threshold(self, scores, theta):
        s = np.ascontiguousarray(scores, np.float64)
        m = np.zeros(s.shape, np.uint8)
        self._chk(self._mthr(s.ravel(), s.size, theta, m.reshape(-1)), "mask_threshold")
        return m

    def mask_topk(self, scores, rate):
        s = np.ascontiguousarray(scores, np.float64)
        m = np.zeros(s.shape, np.uint8)
        self._chk(self._mtopk(s.ravel(), s.size, rate, m.reshape(-1)), "mask_topk")
        return m

    def mask_rate(self, mask):
        m = np.ascontiguousarray(mask, np.uint8).ravel()
        return self._mrate(m, m.size)

    def controller_update(self, threshold, observed, r_min=0.1, r_max=0.3, alpha=1.3):
        out = dbl(0)
        if self.is_ref:
            lr = dbl(0)
            self._chk(self._ctl(threshold, 0.0, observed, r_min, r_max, alpha, C.byref(out),
                                C.byref(lr)), "controller_update")
        else:
            self._chk(self._ctl(threshold, observed, r_min, r_max, alpha, C.byref(out)),
                      "controller_update")
        return out.value


def compact_to_dense(rcomp, rsc, ridx, rows, cols, g):
    """Reference residuals[] + residual_index[] (quant.hpp:46-52) -> dense plane."""
    gr, gc = ridx.shape
    res_codes = np.zeros((rows, cols), np.int16)
    res_scales = np.zeros((gr, gc), np.float32)
    for bi in range(gr):
        for bj in range(gc):
            s = ridx[bi, bj]
            if s < 0:
                continue
            er, ec = min(g, rows - bi * g), min(g, cols - bj * g)
            blk = rcomp[s].reshape(-1)[: er * ec].reshape(er, ec)
            res_codes[bi * g: bi * g + er, bj * g: bj * g + ec] = blk
            res_scales[bi, bj] = rsc[s]
    return res_codes, res_scales


def dense_to_compact(res_codes, res_scales, mask, g):
    rows, cols = res_codes.shape
    gr, gc = mask.shape
    n = int(mask.sum())
    rcomp = np.zeros((max(n, 1), g, g), np.int16)
    rsc = np.zeros(max(n, 1), np.float32)
    ridx = -np.ones((gr, gc), np.int32)
    s = 0
    for bi in range(gr):
        for bj in range(gc):
            if not mask[bi, bj]:
                continue
            er, ec = min(g, rows - bi * g), min(g, cols - bj * g)
            rcomp[s].reshape(-1)[: er * ec] = res_codes[bi * g: bi * g + er,
                                                        bj * g: bj * g + ec].reshape(-1)
            rsc[s] = res_scales[bi, bj]
            ridx[bi, bj] = s
            s += 1
    return rcomp, rsc, ridx


_C = None
_REF = None


def C_oracle() -> Oracle:
    global _C
    if _C is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        _C = Oracle(ORACLE_SO, "orc_")
    return _C


def REF_oracle() -> Oracle | None:
    """The reference itself, or None when oracle/_ref was not built."""
    global _REF
    if _REF is None and os.path.exists(REF_SO):
        _REF = Oracle(REF_SO, "ref_")
    return _REF


class RefMlp:
    """The reference's own gate/up -> GluCombine -> down (QuantLinearLayer x 3,
    trainsim.hpp:38-118) with 128 x 128 blocks, through oracle/_ref."""

    def __init__(self, w_gate, w_up, w_down, threshold=1.0, g=128):
        r = REF_oracle()
        if r is None:
            raise FileNotFoundError("oracle/_ref not built")
        lib = r._l.lib
        self.lib = lib
        lib.ref_mlp_create.restype = C.c_void_p
        lib.ref_mlp_create.argtypes = [F32, F32, F32, i64, i64, i64, dbl]
        lib.ref_mlp_destroy.argtypes = [C.c_void_p]
        lib.ref_mlp_step.argtypes = [C.c_void_p, F32, F32, i64, i64, cint, F32, F32]
        lib.ref_mlp_grads.argtypes = [C.c_void_p, F32, F32, F32]
        lib.ref_mlp_controller.argtypes = [C.c_void_p, F64, F64]
        lib.ref_mlp_sgd.argtypes = [C.c_void_p, dbl]
        lib.ref_mlp_weights.argtypes = [C.c_void_p, F32, F32, F32]
        self.wg = np.ascontiguousarray(w_gate, np.float32)
        self.wu = np.ascontiguousarray(w_up, np.float32)
        self.wd = np.ascontiguousarray(w_down, np.float32)
        self.d_ff, self.d_model = self.wg.shape
        self.h = lib.ref_mlp_create(self.wg, self.wu, self.wd, self.d_model, self.d_ff, g, threshold)
        if not self.h:
            raise RuntimeError(r._err().decode())
        self._err = r._err

    def step(self, x, gy, step):
        x = np.ascontiguousarray(x, np.float32)
        gy = np.ascontiguousarray(gy, np.float32)
        y = np.zeros_like(x)
        gx = np.zeros_like(x)
        rc = self.lib.ref_mlp_step(self.h, x, gy, x.shape[0], self.d_model, step, y, gx)
        if rc:
            raise RuntimeError(self._err().decode())
        return y, gx

    def grads(self):
        gg = np.zeros((self.d_ff, self.d_model), np.float32)
        gu = np.zeros_like(gg)
        gd = np.zeros((self.d_model, self.d_ff), np.float32)
        self.lib.ref_mlp_grads(self.h, gg, gu, gd)
        return gg, gu, gd

    def apply_sgd(self, lr):
        if self.lib.ref_mlp_sgd(self.h, lr):
            raise RuntimeError(self._err().decode())

    def weights(self):
        wg = np.zeros((self.d_ff, self.d_model), np.float32)
        wu = np.zeros_like(wg)
        wd = np.zeros((self.d_model, self.d_ff), np.float32)
        if self.lib.ref_mlp_weights(self.h, wg, wu, wd):
            raise RuntimeError(self._err().decode())
        return wg, wu, wd

    def controller(self):
        rates = np.zeros(3)
        th = np.zeros(3)
        self.lib.ref_mlp_controller(self.h, rates, th)
        return rates, th

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_mlp_destroy(self.h)
            self.h = None


class RefLinear:
    """The reference's own QuantLinearLayer (trainsim.cpp:61-135), block 128,
    through oracle/_ref (test infrastructure)."""

    def __init__(self, w, threshold=1.0, layer_id=0, g=128, fallback_mode="threshold", fixed_rate=0.0):
        r = REF_oracle()
        if r is None:
            raise FileNotFoundError("oracle/_ref not built")
        lib = r._l.lib
        self.lib = lib
        lib.ref_linear_create.restype = C.c_void_p
        lib.ref_linear_create.argtypes = [F32, i64, i64, i64, dbl, cint, cint, dbl]
        lib.ref_linear_destroy.argtypes = [C.c_void_p]
        lib.ref_linear_forward.argtypes = [C.c_void_p, F32, i64, cint, F32]
        lib.ref_linear_backward.argtypes = [C.c_void_p, F32, i64, cint, F32]
        lib.ref_linear_grad.argtypes = [C.c_void_p, F32]
        lib.ref_linear_controller.argtypes = [C.c_void_p, F64, F64]
        lib.ref_linear_zero_grad.argtypes = [C.c_void_p]
        lib.ref_linear_sgd.argtypes = [C.c_void_p, dbl]
        lib.ref_linear_weight.argtypes = [C.c_void_p, F32]
        self.w = np.ascontiguousarray(w, np.float32)
        self.out_features, self.in_features = self.w.shape
        mode = {"threshold": 0, "fixed_rate": 1, "off": 2}[fallback_mode]
        self.h = lib.ref_linear_create(self.w, self.out_features, self.in_features, g, threshold,
                                       layer_id, mode, fixed_rate)
        if not self.h:
            raise RuntimeError(r._err().decode())
        self._err = r._err

    def _rc(self, rc):
        if rc:
            raise RuntimeError(self._err().decode())

    def forward(self, x, step):
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros((x.shape[0], self.out_features), np.float32)
        self._rc(self.lib.ref_linear_forward(self.h, x, x.shape[0], step, y))
        return y

    def backward(self, gy, step):
        gy = np.ascontiguousarray(gy, np.float32)
        gx = np.zeros((gy.shape[0], self.in_features), np.float32)
        self._rc(self.lib.ref_linear_backward(self.h, gy, gy.shape[0], step, gx))
        return gx

    def grad(self):
        g = np.zeros_like(self.w)
        self._rc(self.lib.ref_linear_grad(self.h, g))
        return g

    def controller_step(self):
        rate = np.zeros(1)
        th = np.zeros(1)
        self._rc(self.lib.ref_linear_controller(self.h, rate, th))
        return float(rate[0]), float(th[0])

    def zero_grad(self):
        self._rc(self.lib.ref_linear_zero_grad(self.h))

    def apply_sgd(self, lr):
        self._rc(self.lib.ref_linear_sgd(self.h, lr))

    def weight(self):
        w = np.zeros_like(self.w)
        self._rc(self.lib.ref_linear_weight(self.h, w))
        return w

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_linear_destroy(self.h)
            self.h = None


class RefGluBlock:
    """The reference's own pre-norm residual GLU block (GluBlock, trainsim.hpp:136-146,
    trainsim.cpp:294-308) through oracle/_ref (test infrastructure)."""

    def __init__(self, w_gate, w_up, w_down, threshold=1.0, g=128):
        r = REF_oracle()
        if r is None:
            raise FileNotFoundError("oracle/_ref not built")
        lib = r._l.lib
        self.lib = lib
        lib.ref_block_create.restype = C.c_void_p
        lib.ref_block_create.argtypes = [F32, F32, F32, i64, i64, i64, dbl]
        lib.ref_block_destroy.argtypes = [C.c_void_p]
        lib.ref_block_step.argtypes = [C.c_void_p, F32, F32, i64, cint, F32, F32]
        lib.ref_block_controller.argtypes = [C.c_void_p, F64]
        lib.ref_block_sgd.argtypes = [C.c_void_p, dbl]
        lib.ref_block_state.argtypes = [C.c_void_p] + [F32] * 8
        self.wg = np.ascontiguousarray(w_gate, np.float32)
        self.wu = np.ascontiguousarray(w_up, np.float32)
        self.wd = np.ascontiguousarray(w_down, np.float32)
        self.d_ff, self.d_model = self.wg.shape
        self.h = lib.ref_block_create(self.wg, self.wu, self.wd, self.d_model, self.d_ff, g, threshold)
        if not self.h:
            raise RuntimeError(r._err().decode())
        self._err = r._err

    def _rc(self, rc):
        if rc:
            raise RuntimeError(self._err().decode())

    def step(self, x, grad_out, step):
        x = np.ascontiguousarray(x, np.float32)
        grad_out = np.ascontiguousarray(grad_out, np.float32)
        y, gh = np.zeros_like(x), np.zeros_like(x)
        self._rc(self.lib.ref_block_step(self.h, x, grad_out, x.shape[0], step, y, gh))
        return y, gh

    def controller(self):
        th = np.zeros(3)
        self._rc(self.lib.ref_block_controller(self.h, th))
        return th

    def apply_sgd(self, lr):
        self._rc(self.lib.ref_block_sgd(self.h, lr))

    def state(self):
        """gain, grad_gain, (W_gate, W_up, W_down), (dW_gate, dW_up, dW_down)"""
        d, f = self.d_model, self.d_ff
        gain, gg = np.zeros(d, np.float32), np.zeros(d, np.float32)
        w = [np.zeros((f, d), np.float32), np.zeros((f, d), np.float32), np.zeros((d, f), np.float32)]
        g = [np.zeros_like(a) for a in w]
        self._rc(self.lib.ref_block_state(self.h, gain, gg, *w, *g))
        return gain, gg, tuple(w), tuple(g)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_block_destroy(self.h)
            self.h = None


class RefSilu:
    """The reference's own SiluLayer (trainsim.cpp:265-290) through oracle/_ref."""

    def __init__(self):
        r = REF_oracle()
        if r is None:
            raise FileNotFoundError("oracle/_ref not built")
        lib = r._l.lib
        self.lib = lib
        lib.ref_silu_create.restype = C.c_void_p
        lib.ref_silu_create.argtypes = []
        lib.ref_silu_destroy.argtypes = [C.c_void_p]
        lib.ref_silu_forward.argtypes = [C.c_void_p, F32, i64, i64, F32]
        lib.ref_silu_backward.argtypes = [C.c_void_p, F32, i64, i64, F32]
        self.h = lib.ref_silu_create()
        self._err = r._err

    def forward(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros_like(x)
        if self.lib.ref_silu_forward(self.h, x, x.shape[0], x.shape[1], y):
            raise RuntimeError(self._err().decode())
        return y

    def backward(self, gy):
        gy = np.ascontiguousarray(gy, np.float32)
        gx = np.zeros_like(gy)
        if self.lib.ref_silu_backward(self.h, gy, gy.shape[0], gy.shape[1], gx):
            raise RuntimeError(self._err().decode())
        return gx

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_silu_destroy(self.h)
            self.h = None


class RefRmsNorm:
    """The reference's own RmsNorm (trainsim.cpp:145-219) through oracle/_ref."""

    def __init__(self, dim):
        r = REF_oracle()
        if r is None:
            raise FileNotFoundError("oracle/_ref not built")
        lib = r._l.lib
        self.lib = lib
        lib.ref_rms_create.restype = C.c_void_p
        lib.ref_rms_create.argtypes = [i64]
        lib.ref_rms_destroy.argtypes = [C.c_void_p]
        lib.ref_rms_forward.argtypes = [C.c_void_p, F32, i64, F32]
        lib.ref_rms_backward.argtypes = [C.c_void_p, F32, i64, F32]
        lib.ref_rms_state.argtypes = [C.c_void_p, F32, F32]
        lib.ref_rms_sgd.argtypes = [C.c_void_p, dbl]
        self.dim = dim
        self.h = lib.ref_rms_create(dim)
        self._err = r._err

    def _rc(self, rc):
        if rc:
            raise RuntimeError(self._err().decode())

    def forward(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros_like(x)
        self._rc(self.lib.ref_rms_forward(self.h, x, x.shape[0], y))
        return y

    def backward(self, gy):
        gy = np.ascontiguousarray(gy, np.float32)
        gx = np.zeros_like(gy)
        self._rc(self.lib.ref_rms_backward(self.h, gy, gy.shape[0], gx))
        return gx

    def state(self):
        g = np.zeros(self.dim, np.float32)
        gg = np.zeros(self.dim, np.float32)
        self._rc(self.lib.ref_rms_state(self.h, g, gg))
        return g, gg

    def apply_sgd(self, lr):
        self._rc(self.lib.ref_rms_sgd(self.h, lr))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_rms_destroy(self.h)
            self.h = None
