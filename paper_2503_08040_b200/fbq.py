"""Reference-shaped operator API on device tensors (the fbq:: names).

Mirrors /root/reference/proj/include/fbq/{quant,gemm,policy}.hpp -- same
names, same argument meaning, same error behaviour (ValueError where the
reference throws std::invalid_argument) -- but operates on torch CUDA tensors
and calls the sm_100a kernels through the C ABI (include/fbq_b200.h).
PyTorch provides device memory and streams only; every computation here is one
of our kernels.

Differences that are representation-only (values are bit-identical):
* codes are int8 (the reference stores int16, quant.hpp:31), in planes whose
  row stride ``ldq`` is padded to a multiple of 16 (TMA rule);
* the fallback mask is a bitmap (uint32 words) and the residuals live in a
  dense "lo" plane next to the primary "hi" codes (quant.hpp:40-57 keeps a
  compact vector + index; ``FallbackTensor.residual_blocks()`` gives that view);
* ``transpose(QuantizedTensor)`` is a zero-copy view (quant.cpp:106-126
  copies): the GEMM reads the same bytes MN-major instead.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _capi as K

BLOCK = 128
LEVEL = 127


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def cdiv(a: int, b: int) -> int:
    return (a + b - 1) // b


def _ld16(n: int) -> int:
    return max(16, (n + 15) // 16 * 16)


def _dtype_code(x: torch.Tensor) -> int:
    if x.dtype == torch.float32:
        return K.FBQ_F32
    if x.dtype == torch.bfloat16:
        return K.FBQ_BF16
    raise ValueError(f"unsupported input dtype {x.dtype} (fp32 or bf16)")


def _check_input(x: torch.Tensor) -> torch.Tensor:
    if not x.is_cuda:
        raise ValueError("fbq B200 ops take CUDA tensors (no CPU fallback)")
    if x.dim() != 2:
        raise ValueError("expected a 2-D matrix")
    if x.stride(1) != 1:
        x = x.contiguous()
    return x


def _check_geometry(block, bits):
    # BitWidth / GroupGeometry validation (quant.cpp:10-12, matrix.cpp:55-57)
    if bits < 2 or bits > 16:
        raise ValueError("bit-width must be in [2, 16]")
    if block != BLOCK or bits != 8:
        raise NotImplementedError(
            "B200 hot path supports 128x128 blocks and 8-bit codes (FBQ_ERR_UNSUPPORTED)")


@dataclass
class QuantizedTensor:
    """quant.hpp:23-36.  ``codes`` int8 [stored_rows, ldq]; ``scales`` fp32 stored grid.

    ``transposed`` marks a zero-copy transpose view: logical (rows, cols) but
    the bytes are the (cols, rows) tensor's.
    """
    rows: int
    cols: int
    codes: torch.Tensor
    scales: torch.Tensor
    transposed: bool = False
    bits: int = 8
    block: int = BLOCK

    @property
    def ldq(self) -> int:
        return self.codes.stride(0)

    @property
    def stored_shape(self):
        return (self.cols, self.rows) if self.transposed else (self.rows, self.cols)

    def grid_rows(self) -> int:
        return cdiv(self.rows, self.block)

    def grid_cols(self) -> int:
        return cdiv(self.cols, self.block)

    def scale_at(self, bi: int, bj: int) -> float:
        s = self.scales[bj, bi] if self.transposed else self.scales[bi, bj]
        return float(s)

    def codes_int16(self) -> torch.Tensor:
        """Logical codes as the reference stores them (int16, rows x cols)."""
        r, c = self.stored_shape
        v = self.codes[:r, :c].to(torch.int16)
        return v.t().contiguous() if self.transposed else v

    def scales_logical(self) -> torch.Tensor:
        return self.scales.t().contiguous() if self.transposed else self.scales


@dataclass
class FallbackTensor:
    """quant.hpp:40-57: primary codes + an int8 residual for each masked block."""
    primary: QuantizedTensor
    mask_bits: torch.Tensor          # int32 words (bit b = block b, row-major grid)
    res_codes: torch.Tensor          # int8 dense lo plane (same layout as primary.codes)
    res_scales: torch.Tensor         # fp32 grid (0 where unmasked)
    masked_count: torch.Tensor | None = None  # int32[1] on device

    @property
    def mask(self) -> torch.Tensor:
        """uint8 per block, row-major grid (quant.hpp:42)."""
        return bits_to_mask(self.mask_bits, self.primary.grid_rows(), self.primary.grid_cols())

    def masked(self, bi: int, bj: int) -> bool:
        b = bi * self.primary.grid_cols() + bj
        return bool((int(self.mask_bits[b >> 5]) >> (b & 31)) & 1)

    def residual_blocks(self):
        """Compact view (residuals[], residual_index[]) in the reference's order."""
        gr, gc = self.primary.grid_rows(), self.primary.grid_cols()
        m = self.mask.cpu()
        res, idx = [], torch.full((gr, gc), -1, dtype=torch.int32)
        for bi in range(gr):
            for bj in range(gc):
                if not m[bi, bj]:
                    continue
                r0, c0 = bi * BLOCK, bj * BLOCK
                er, ec = min(BLOCK, self.primary.rows - r0), min(BLOCK, self.primary.cols - c0)
                idx[bi, bj] = len(res)
                res.append((self.res_codes[r0:r0 + er, c0:c0 + ec].to(torch.int16).cpu(),
                            float(self.res_scales[bi, bj])))
        return res, idx


def mask_to_bits(mask: torch.Tensor) -> torch.Tensor:
    m = mask.reshape(-1).to(torch.int64)
    n = m.numel()
    words = torch.zeros(cdiv(max(n, 1), 32) * 32, dtype=torch.int64, device=mask.device)
    words[:n] = m != 0
    w = words.view(-1, 32) << torch.arange(32, device=mask.device, dtype=torch.int64)
    w = w.sum(1)
    return torch.where(w >= 2 ** 31, w - 2 ** 32, w).to(torch.int32)


def bits_to_mask(bits: torch.Tensor, gr: int, gc: int) -> torch.Tensor:
    n = gr * gc
    b = bits.to(torch.int64) & 0xFFFFFFFF
    sh = torch.arange(32, device=bits.device, dtype=torch.int64)
    m = ((b.view(-1, 1) >> sh) & 1).reshape(-1)[:n]
    return m.to(torch.uint8).view(gr, gc)


def _alloc_codes(rows, cols, device):
    ldq = _ld16(cols)
    return torch.empty((max(rows, 0), ldq), dtype=torch.int8, device=device)


def _alloc_grid(rows, cols, device, dtype=torch.float32):
    return torch.empty((cdiv(rows, BLOCK), cdiv(cols, BLOCK)), dtype=dtype, device=device)


# ----------------------------------------------------------------- quant.hpp
def quantize_rtn(x: torch.Tensor, block: int = BLOCK, bits: int = 8) -> QuantizedTensor:
    """quant.cpp:36-53 -- K1 with no fallback."""
    _check_geometry(block, bits)
    x = _check_input(x)
    r, c = x.shape
    codes, scales = _alloc_codes(r, c, x.device), _alloc_grid(r, c, x.device)
    K.call("fbq_cuda_quantize_rtn", x.data_ptr(), _dtype_code(x), r, c, x.stride(0),
           codes.data_ptr(), codes.stride(0), scales.data_ptr(), _stream())
    return QuantizedTensor(r, c, codes, scales)


def quantize_stochastic(x: torch.Tensor, seed: int, row_offset: int = 0, block: int = BLOCK,
                        bits: int = 8) -> QuantizedTensor:
    """quant.cpp:55-84 -- K2.  ``seed`` is the DeterministicRng seed (rng.hpp:22-30)."""
    _check_geometry(block, bits)
    x = _check_input(x)
    r, c = x.shape
    codes, scales = _alloc_codes(r, c, x.device), _alloc_grid(r, c, x.device)
    K.call("fbq_cuda_quantize_stochastic", x.data_ptr(), _dtype_code(x), r, c, x.stride(0),
           seed & (2 ** 64 - 1), row_offset, codes.data_ptr(), codes.stride(0),
           scales.data_ptr(), _stream())
    return QuantizedTensor(r, c, codes, scales)


def fallback_quantize(x: torch.Tensor, mask: torch.Tensor | None = None, *,
                      theta: float | None = None, block: int = BLOCK, bits: int = 8,
                      sr_seed: int | None = None, sr_row_offset: int = 0):
    """quant.cpp:128-176.  ``mask`` (uint8 grid) as in the reference, or
    ``theta`` to fuse score_blocks(AbsMax)+mask_threshold (trainsim.cpp:80-84).
    With ``sr_seed`` the stochastic context codes (trainsim.cpp:100-102) are
    produced by the same pass and returned as a second value."""
    _check_geometry(block, bits)
    x = _check_input(x)
    r, c = x.shape
    gr, gc = cdiv(r, BLOCK), cdiv(c, BLOCK)
    dev = x.device
    if mask is not None:
        if tuple(mask.shape) not in ((gr, gc), (gr * gc,)):
            raise ValueError("fallback mask does not match the block grid")  # quant.cpp:132-134
        mode, bits_t, th = K.FBQ_MASK_GIVEN, mask_to_bits(mask.to(dev)), 1.0
    elif theta is not None:
        if not theta > 0.0:
            raise ValueError("threshold must be > 0")  # policy.cpp:74
        mode, th = K.FBQ_MASK_THRESHOLD, float(theta)
        bits_t = torch.empty(cdiv(max(gr * gc, 1), 32), dtype=torch.int32, device=dev)  # all bits written
    else:
        raise ValueError("fallback_quantize needs a mask or a threshold")
    codes, scales = _alloc_codes(r, c, dev), _alloc_grid(r, c, dev)
    res_codes, res_scales = _alloc_codes(r, c, dev), _alloc_grid(r, c, dev)
    count = torch.empty(1, dtype=torch.int32, device=dev)  # zeroed in-stream by the call
    sr = _alloc_codes(r, c, dev) if sr_seed is not None else None
    K.call("fbq_cuda_quantize_fallback", x.data_ptr(), _dtype_code(x), r, c, x.stride(0), mode,
           th, bits_t.data_ptr(), codes.data_ptr(), codes.stride(0), scales.data_ptr(),
           res_codes.data_ptr(), res_scales.data_ptr(), count.data_ptr(), None,
           sr.data_ptr() if sr is not None else None,
           (sr_seed or 0) & (2 ** 64 - 1), sr_row_offset, _stream())
    f = FallbackTensor(QuantizedTensor(r, c, codes, scales), bits_t, res_codes, res_scales, count)
    if sr is not None:
        return f, QuantizedTensor(r, c, sr, scales)
    return f


def dequantize(q: QuantizedTensor) -> torch.Tensor:
    """quant.cpp:86-104 (K4)."""
    r, c = q.stored_shape
    out = torch.empty((r, c), dtype=torch.float32, device=q.codes.device)
    K.call("fbq_cuda_dequantize", q.codes.data_ptr(), q.ldq, q.scales.data_ptr(), None, None,
           None, r, c, out.data_ptr(), max(c, 1), _stream())
    return out.t() if q.transposed else out


def dequantize_fallback(f: FallbackTensor) -> torch.Tensor:
    """quant.cpp:178-202 (K4)."""
    q = f.primary
    r, c = q.stored_shape
    out = torch.empty((r, c), dtype=torch.float32, device=q.codes.device)
    K.call("fbq_cuda_dequantize", q.codes.data_ptr(), q.ldq, q.scales.data_ptr(),
           f.mask_bits.data_ptr(), f.res_codes.data_ptr(), f.res_scales.data_ptr(), r, c,
           out.data_ptr(), max(c, 1), _stream())
    return out


def transpose(q: QuantizedTensor) -> QuantizedTensor:
    """quant.cpp:106-126, as a zero-copy view."""
    return replace(q, rows=q.cols, cols=q.rows, transposed=not q.transposed)


# ------------------------------------------------------------------ gemm.hpp
def _gemm(qa: QuantizedTensor, qb: QuantizedTensor, fb: FallbackTensor | None, out=None,
          out_dtype=torch.float32, accumulate=False, exact=True):
    if qa.cols != qb.rows:
        raise ValueError("block gemm: inner dimensions differ")  # gemm.cpp:80
    if qa.bits > 8 or qb.bits > 8:
        raise ValueError("block gemm: operand bit-widths must be <= 8")
    M, Kd, N = qa.rows, qa.cols, qb.cols
    a_major = K.FBQ_MN_MAJOR if qa.transposed else K.FBQ_K_MAJOR
    b_major = K.FBQ_K_MAJOR if qb.transposed else K.FBQ_MN_MAJOR
    dev = qa.codes.device
    if out is None:
        out = (torch.zeros if accumulate else torch.empty)((M, N), dtype=out_dtype, device=dev)
    if out.shape != (M, N) or out.stride(1) != 1:
        raise ValueError("output shape mismatch")
    od = K.FBQ_F32 if out.dtype == torch.float32 else K.FBQ_BF16
    if fb is not None:
        mb, rc, rs = fb.mask_bits.data_ptr(), fb.res_codes.data_ptr(), fb.res_scales.data_ptr()
    else:
        mb = rc = rs = None
    K.call("fbq_cuda_gemm", qa.codes.data_ptr(), qa.ldq, qa.scales.data_ptr(), a_major,
           qb.codes.data_ptr(), qb.ldq, qb.scales.data_ptr(), b_major, mb, rc, rs, M, N, Kd,
           out.data_ptr(), od, out.stride(0), int(accumulate),
           K.FBQ_EPI_EXACT if exact else K.FBQ_EPI_FMA, _stream())
    return out


def block_quant_gemm(qa: QuantizedTensor, qb: QuantizedTensor, **kw) -> torch.Tensor:
    """gemm.cpp:190-193: A (M x K) times B (K x N), int32 per block, fp32 across blocks."""
    return _gemm(qa, qb, None, **kw)


def fallback_gemm(fa: FallbackTensor, qb: QuantizedTensor, **kw) -> torch.Tensor:
    """gemm.cpp:195-198 / Algorithm 1."""
    if fa.primary.transposed:
        raise ValueError("fallback A operand must be K-major")
    return _gemm(fa.primary, qb, fa, **kw)


def tiled_block_gemm(qa: QuantizedTensor, qb: QuantizedTensor, tile=(128, 128, 128), **kw):
    """gemm.cpp:200-203.  Integer tile products are associative, so every valid
    tile gives the block GEMM bit-for-bit; the tensor-core path always computes
    the full 128-deep block with K=32 MMA sub-steps."""
    for t in tile:
        if t < 1 or BLOCK % t:
            raise ValueError("tile sides must divide the block sides")
    return block_quant_gemm(qa, qb, **kw)


def block_products(qa: QuantizedTensor, qb: QuantizedTensor, fb: FallbackTensor | None = None):
    """Raw int32 per-block products (gemm.cpp:140-145) from the tcgen05 path."""
    M, Kd, N = qa.rows, qa.cols, qb.cols
    MB, NB, KB = cdiv(M, BLOCK), cdiv(N, BLOCK), cdiv(Kd, BLOCK)
    n = MB * NB * KB * BLOCK * BLOCK
    out = torch.zeros(n * (2 if fb is not None else 1), dtype=torch.int32, device=qa.codes.device)
    a_major = K.FBQ_MN_MAJOR if qa.transposed else K.FBQ_K_MAJOR
    b_major = K.FBQ_K_MAJOR if qb.transposed else K.FBQ_MN_MAJOR
    K.call("fbq_cuda_gemm_block_products", qa.codes.data_ptr(), qa.ldq, a_major,
           qb.codes.data_ptr(), qb.ldq, b_major,
           fb.mask_bits.data_ptr() if fb is not None else None,
           fb.res_codes.data_ptr() if fb is not None else None, M, N, Kd, out.data_ptr(),
           _stream())
    prim = out[:n].view(MB, NB, KB, BLOCK, BLOCK)
    if fb is None:
        return prim
    return prim, out[n:].view(MB, NB, KB, BLOCK, BLOCK)


# ---------------------------------------------------------------- policy.hpp
def score_blocks(x: torch.Tensor, block: int = BLOCK) -> torch.Tensor:
    """policy.cpp:12-28 (AbsMax criterion) -> float64 grid."""
    _check_geometry(block, 8)
    x = _check_input(x)
    r, c = x.shape
    amax = _alloc_grid(r, c, x.device)
    K.call("fbq_cuda_block_absmax", x.data_ptr(), _dtype_code(x), r, c, x.stride(0),
           amax.data_ptr(), _stream())
    return amax.to(torch.float64)


def mask_threshold(scores: torch.Tensor, threshold: float) -> torch.Tensor:
    """policy.cpp:73-80 (strict >)."""
    if not threshold > 0.0:
        raise ValueError("threshold must be > 0")
    return (scores > threshold).to(torch.uint8)


def mask_topk(scores: torch.Tensor, rate: float) -> torch.Tensor:
    """policy.cpp:56-71: exactly ceil(rate*n) top scores, ties -> lower index."""
    if rate < 0.0 or rate > 1.0:
        raise ValueError("rate must be in [0, 1]")
    n = scores.numel()
    if not scores.is_cuda:
        # host-resident scores: the host policy, like the reference's own
        # mask_topk; stable sort on descending score keeps ascending index among ties
        flat = scores.reshape(-1).to(torch.float64)
        k = min(n, math.ceil(rate * n))
        order = torch.sort(-flat, stable=True).indices[:k]
        m = torch.zeros(n, dtype=torch.uint8)
        m[order] = 1
        return m.view(scores.shape)
    # device scores (score_blocks): fbq_cuda_mask_topk, no host round trip.
    # the AbsMax scores are fp32 values widened to double: exact in fp32
    flat = scores.reshape(-1).to(torch.float32).contiguous()
    bits = torch.empty(cdiv(max(n, 1), 32), dtype=torch.int32, device=scores.device)
    if n:
        K.call("fbq_cuda_mask_topk", flat.data_ptr(), n, float(rate), bits.data_ptr(), None,
               _stream())
    gr, gc = (scores.shape if scores.dim() == 2 else (1, n))
    return bits_to_mask(bits, gr, gc).view(scores.shape)


def theta_for_rate(scores, rate: float):
    """A THRESHOLD-mode theta that flags ceil(rate*n) blocks under policy.cpp:77's
    strict `score > theta` -- or, when that count splits a group of tied scores,
    the nearest count at a tie boundary.  Returns (theta, flagged_fraction).
    theta is a score value itself (strictly below the flagged ones), so the
    strict compare makes the count exact; with no block flagged it is the
    maximum score, with every block flagged it is below the minimum.  (Host
    helper for benchmarks and tests: the fallback rate a threshold realises.)"""
    s = np.sort(np.asarray(scores, dtype=np.float64).reshape(-1))[::-1]
    n = s.size
    if n == 0:
        return 1.0, 0.0
    k = min(n, math.ceil(rate * n))

    def cut_ok(c):  # top c are strictly above the rest
        return c == 0 or c == n or s[c - 1] > s[c]
    lo, hi = k, k
    while not cut_ok(lo):
        lo -= 1
    while not cut_ok(hi):
        hi += 1
    c = lo if (k - lo) <= (hi - k) else hi
    if c == 0:
        theta = float(s[0]) if s[0] > 0 else 1.0
    elif c == n:
        theta = float(s[-1]) * 0.5  # every positive score above it
    else:
        theta = float(s[c])
    return theta, c / n


def mask_rate(mask: torch.Tensor) -> float:
    """policy.cpp:82-87."""
    if mask.numel() == 0:
        return 0.0
    return float((mask != 0).sum()) / mask.numel()


@dataclass
class ControllerConfig:
    """policy.hpp:32-41 / policy.cpp:89-95."""
    r_min: float = 0.1
    r_max: float = 0.3
    alpha: float = 1.3

    def __post_init__(self):
        if not (0.0 <= self.r_min < self.r_max <= 1.0):
            raise ValueError("need 0 <= r_min < r_max <= 1")
        if not self.alpha > 1.0:
            raise ValueError("alpha must be > 1")


@dataclass
class FallbackThresholdState:
    threshold: float = 1.0
    last_rate: float = 0.0


def controller_update(state: FallbackThresholdState, observed_rate: float,
                      cfg: ControllerConfig = ControllerConfig()) -> FallbackThresholdState:
    """policy.cpp:97-109 (Algorithm 2 delay-threshold update)."""
    if observed_rate < 0.0 or observed_rate > 1.0:
        raise ValueError("observed rate must be in [0, 1]")
    th = state.threshold
    if observed_rate < cfg.r_min:
        th /= cfg.alpha
    elif observed_rate > cfg.r_max:
        th *= cfg.alpha
    return FallbackThresholdState(th, observed_rate)


def derive_seed(base: int, a: int, b: int = 0) -> int:
    """rng.hpp:56-58 (host-side integer math)."""
    return bits_at(bits_at(base, a), b)


def bits_at(seed: int, n: int) -> int:
    """rng.hpp:28-30."""
    M = 2 ** 64 - 1
    z = (seed + (n + 1) * 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def layer_seed(base: int, layer_id: int, tag: int, step: int) -> int:
    """trainsim.cpp:16-19 (tag 0 = X context, 1 = dY)."""
    return derive_seed(base, layer_id * 4 + tag, step)


# ------------------------------------------------------------------ RmsNorm
class SiluLayer:
    """SiluLayer (trainsim.hpp:118-131, trainsim.cpp:265-290) on the device: y =
    silu(x), the input kept as its 10-bit 1 x 128 context; backward gx = gy *
    silu'(dequantized context).  exact: the reference's double silu / silu'
    (bit-exact); otherwise the fp32 fast forms of the GLU training path."""

    def __init__(self, exact: bool = True, bits: int = 10):
        self.exact = bool(exact)
        self.bits = bits
        self._ctx = None

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        x = _check_input(x)
        r, c = x.shape
        y = torch.empty_like(x)
        ldc = _ld16(c)
        codes = torch.empty((r, ldc), dtype=torch.int16, device=x.device)
        scales = torch.empty((r, cdiv(c, BLOCK)), dtype=torch.float32, device=x.device)
        K.call("fbq_cuda_silu_forward", x.data_ptr(), _dtype_code(x), r, c, x.stride(0), y.data_ptr(),
               y.stride(0), codes.data_ptr(), ldc, scales.data_ptr(), self.bits, int(self.exact), _stream())
        self._ctx = (codes, scales, r, c)
        return y

    def backward(self, gy: torch.Tensor) -> torch.Tensor:
        if self._ctx is None:
            raise RuntimeError("silu: backward without context")  # trainsim.cpp:280-282
        codes, scales, r, c = self._ctx
        gy = _check_input(gy)
        if tuple(gy.shape) != (r, c):
            raise ValueError("gradient shape does not match the forward input")
        gx = torch.empty_like(gy)
        K.call("fbq_cuda_silu_backward", codes.data_ptr(), codes.stride(0), scales.data_ptr(), gy.data_ptr(),
               _dtype_code(gy), r, c, gy.stride(0), gx.data_ptr(), gx.stride(0), int(self.exact), _stream())
        return gx

    def context(self):
        """(int16 codes [rows, ld], fp32 scales [rows, ceil(cols/128)]) of the last forward."""
        return self._ctx[0], self._ctx[1]


class RmsNorm:
    """RmsNorm (trainsim.hpp:75-97, trainsim.cpp:145-211) on the device: gain
    starts at 1, the input is kept as its 10-bit 1 x 128 context, backward
    accumulates grad_gain; apply_sgd / zero_grad as in the reference."""

    def __init__(self, dim: int, device="cuda"):
        self.dim = dim
        self.gain = torch.ones(dim, dtype=torch.float32, device=device)
        self.grad_gain = torch.zeros(dim, dtype=torch.float32, device=device)
        self._ctx = None

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        x = _check_input(x)
        r, c = x.shape
        if c != self.dim:
            raise ValueError("width does not match the gain vector")  # trainsim.cpp:156-158
        y = torch.empty_like(x)
        ldc = _ld16(c)
        codes = torch.empty((r, ldc), dtype=torch.int16, device=x.device)
        scales = torch.empty((r, cdiv(c, BLOCK)), dtype=torch.float32, device=x.device)
        rms = torch.empty(r, dtype=torch.float32, device=x.device)
        K.call("fbq_cuda_rmsnorm_forward", x.data_ptr(), _dtype_code(x), r, c, x.stride(0),
               self.gain.data_ptr(), y.data_ptr(), y.stride(0), codes.data_ptr(), ldc,
               scales.data_ptr(), rms.data_ptr(), _stream())
        self._ctx = (codes, scales, r, c)
        return y

    def forward_quantized(self, x: torch.Tensor, *, mask: torch.Tensor | None = None,
                          theta: float | None = None, sr_seed: int | None = None,
                          sr_seed2: int | None = None, row_offset: int = 0):
        """forward() fused with the next linear's input quantizer: the same
        context as forward(), and for y = forward(x) exactly the outputs of
        fallback_quantize(y, mask | theta, sr_seed) (+ a second stochastic plane
        with sr_seed2), without materialising y.  Returns the FallbackTensor and
        the stochastic QuantizedTensors (as fallback_quantize)."""
        x = _check_input(x)
        r, c = x.shape
        if c != self.dim:
            raise ValueError("width does not match the gain vector")
        gr, gc = cdiv(r, BLOCK), cdiv(c, BLOCK)
        dev = x.device
        if mask is not None:
            mode, bits_t, th = K.FBQ_MASK_GIVEN, mask_to_bits(mask.to(dev)), 1.0
        elif theta is not None:
            if not theta > 0.0:
                raise ValueError("threshold must be > 0")
            mode, th = K.FBQ_MASK_THRESHOLD, float(theta)
            bits_t = torch.empty(cdiv(max(gr * gc, 1), 32), dtype=torch.int32, device=dev)
        else:
            raise ValueError("forward_quantized needs a mask or a threshold")
        ldc = _ld16(c)
        ctx = torch.empty((r, ldc), dtype=torch.int16, device=dev)
        ctx_s = torch.empty((r, gc), dtype=torch.float32, device=dev)
        rms = torch.empty(r, dtype=torch.float32, device=dev)
        codes, scales = _alloc_codes(r, c, dev), _alloc_grid(r, c, dev)
        res_codes, res_scales = _alloc_codes(r, c, dev), _alloc_grid(r, c, dev)
        count = torch.empty(1, dtype=torch.int32, device=dev)
        sr = _alloc_codes(r, c, dev) if sr_seed is not None else None
        sr2 = _alloc_codes(r, c, dev) if sr_seed2 is not None else None
        K.call("fbq_cuda_rmsnorm_quantize_input", x.data_ptr(), _dtype_code(x), r, c, x.stride(0),
               self.gain.data_ptr(), ctx.data_ptr(), ldc, ctx_s.data_ptr(), rms.data_ptr(), mode, th, None,
               bits_t.data_ptr(), codes.data_ptr(), codes.stride(0), scales.data_ptr(), res_codes.data_ptr(),
               res_scales.data_ptr(), count.data_ptr(), sr.data_ptr() if sr is not None else None,
               (sr_seed or 0) & (2 ** 64 - 1), sr2.data_ptr() if sr2 is not None else None,
               (sr_seed2 or 0) & (2 ** 64 - 1), row_offset, _stream())
        self._ctx = (ctx, ctx_s, r, c)
        f = FallbackTensor(QuantizedTensor(r, c, codes, scales), bits_t, res_codes, res_scales, count)
        extra = tuple(QuantizedTensor(r, c, t, scales) for t in (sr, sr2) if t is not None)
        return (f,) + extra if extra else f

    def context(self):
        """(int16 codes rows x ld, fp32 scales rows x ceil(cols/128)) of the last input."""
        return self._ctx[:2]

    def backward(self, gy: torch.Tensor) -> torch.Tensor:
        if self._ctx is None:
            raise RuntimeError("backward without context")  # trainsim.cpp:181-183
        codes, scales, r, c = self._ctx
        gy = _check_input(gy)
        gx = torch.empty_like(gy)
        row_ws = torch.empty(2 * r, dtype=torch.float64, device=gy.device)
        term = torch.empty((r, c), dtype=torch.float32, device=gy.device)
        K.call("fbq_cuda_rmsnorm_backward", codes.data_ptr(), codes.stride(0), scales.data_ptr(),
               gy.data_ptr(), _dtype_code(gy), r, c, gy.stride(0), self.gain.data_ptr(),
               gx.data_ptr(), gx.stride(0), self.grad_gain.data_ptr(), row_ws.data_ptr(),
               term.data_ptr(), _stream())
        return gx

    def zero_grad(self):
        self.grad_gain.zero_()

    def apply_sgd(self, lr: float):
        """gain[c] -= float(lr * double(grad_gain[c])) (trainsim.cpp:213-218)."""
        self.gain.sub_((lr * self.grad_gain.double()).float())
