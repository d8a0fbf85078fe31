"""SwiGLU MLP driver (include/fbq_b200_host.h) from Python.

``GluMlp`` mirrors the reference's gate/up -> GluCombine -> down composition
(QuantLinearLayer::forward/backward, trainsim.cpp:61-127; GluCombine,
trainsim.cpp:224-263).  The C++ driver owns its device workspaces; PyTorch
tensors are only used to hand it device pointers and streams.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _capi as K

lib = K.lib


class MlpConfig(C.Structure):
    _fields_ = [
        ("d_model", C.c_int64), ("d_ff", C.c_int64), ("max_tokens", C.c_int64),
        ("act_dtype", C.c_int), ("mid_dtype", C.c_int), ("epilogue", C.c_int),
        ("nonlinear_bits", C.c_int), ("layer_id_base", C.c_int), ("seed", C.c_uint64),
        ("threshold_init", C.c_double), ("r_min", C.c_double), ("r_max", C.c_double),
        ("alpha", C.c_double), ("ctx_format", C.c_int),
    ]


_F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_sigs = {
    "fbq_mlp_default_config": (None, [C.POINTER(MlpConfig)]),
    "fbq_mlp_create": (C.c_void_p, [C.POINTER(MlpConfig), _F32P, _F32P, _F32P]),
    "fbq_mlp_destroy": (None, [C.c_void_p]),
    "fbq_mlp_forward_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                         C.c_void_p, C.c_void_p]),
    "fbq_mlp_backward_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                          C.c_void_p, C.c_void_p]),
    "fbq_mlp_controller_step": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fbq_mlp_controller_step_blocks": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]),
    "fbq_mlp_count_ptr": (C.c_void_p, [C.c_void_p]),
    "fbq_mlp_zero_grad": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fbq_mlp_step_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int,
                                    C.c_void_p, C.c_void_p]),
    "fbq_mlp_step_host_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_int]),
    "fbq_mlp_host_sync": (C.c_int, [C.c_void_p]),
    "fbq_mlp_grad_ptr": (C.c_void_p, [C.c_void_p, C.c_int]),
    "fbq_mlp_wait_grad": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "fbq_mlp_get_grads": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "fbq_mlp_get_controller": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "fbq_host_last_error": (C.c_char_p, []),
    "fbq_mlp_set_thresholds": (C.c_int, [C.c_void_p, C.c_double, C.c_double]),
    "fbq_mlp_context_bytes": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "fbq_mlp_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "fbq_mlp_gemm_time": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "fbq_mlp_launch_count": (C.c_int64, [C.c_void_p]),
    "fbq_mlp_apply_sgd": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p]),
    "fbq_mlp_get_weights": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "fbq_mlp_set_sgd_lr": (C.c_int, [C.c_void_p, C.c_double]),
    "fbq_glublock_create": (C.c_void_p, [C.POINTER(MlpConfig), _F32P, _F32P, _F32P]),
    "fbq_glublock_destroy": (None, [C.c_void_p]),
    "fbq_glublock_mlp": (C.c_void_p, [C.c_void_p]),
    "fbq_glublock_forward_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                              C.c_void_p, C.c_void_p]),
    "fbq_glublock_backward_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                               C.c_void_p, C.c_void_p]),
    "fbq_glublock_zero_grad": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fbq_glublock_apply_sgd": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p]),
    "fbq_glublock_get_gain": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "fbq_glublock_gain_ptr": (C.c_void_p, [C.c_void_p, C.c_int]),
}
for _n, (_r, _a) in _sigs.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a


class LinearConfig(C.Structure):
    _fields_ = [("in_features", C.c_int64), ("out_features", C.c_int64), ("max_tokens", C.c_int64),
                ("act_dtype", C.c_int), ("epilogue", C.c_int), ("layer_id", C.c_int),
                ("seed", C.c_uint64), ("threshold_init", C.c_double), ("r_min", C.c_double),
                ("r_max", C.c_double), ("alpha", C.c_double), ("fallback_mode", C.c_int),
                ("fixed_rate", C.c_double)]


for _name, (_res, _args) in {
    "fbq_linear_default_config": (None, [C.c_void_p]),
    "fbq_linear_create": (C.c_void_p, [C.c_void_p, _F32P]),
    "fbq_linear_destroy": (None, [C.c_void_p]),
    "fbq_linear_forward_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                            C.c_void_p, C.c_void_p]),
    "fbq_linear_backward_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                             C.c_void_p, C.c_void_p]),
    "fbq_linear_controller_step": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fbq_linear_controller_step_blocks": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    "fbq_linear_count_ptr": (C.c_void_p, [C.c_void_p]),
    "fbq_linear_zero_grad": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fbq_linear_grad_ptr": (C.c_void_p, [C.c_void_p]),
    "fbq_linear_get_controller": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "fbq_linear_apply_sgd": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p]),
    "fbq_linear_get_weight": (C.c_int, [C.c_void_p, C.c_void_p]),
}.items():
    _f = getattr(lib, _name)
    _f.restype, _f.argtypes = _res, _args


def _check(st, what):
    if st != K.FBQ_OK:
        raise K.FbqError(st, f"{what} ({lib.fbq_host_last_error().decode()})")


class _DevArray:
    """__cuda_array_interface__ view of a driver-owned device buffer."""

    def __init__(self, ptr, shape, typestr="<f4"):
        if not ptr:
            raise K.FbqError(K.FBQ_ERR_CUDA, f"null device pointer ({lib.fbq_host_last_error().decode()})")
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False), "version": 3,
            "strides": None,
        }


def _blocks(tokens: int, cols: int) -> int:
    return -(-tokens // 128) * -(-cols // 128)


def _check_act(t: torch.Tensor, dtype, cols: int, what: str):
    if not t.is_cuda or t.dtype != dtype or t.dim() != 2 or t.shape[1] != cols:
        raise ValueError(f"{what}: expected a CUDA {dtype} tensor of shape (tokens, {cols}), got "
                         f"{t.device} {t.dtype} {tuple(t.shape)}")


def _check_out(out, tokens: int, cols: int, dtype, what: str):
    if out is not None and (not out.is_cuda or out.dtype != dtype or tuple(out.shape) != (tokens, cols)
                            or not out.is_contiguous()):
        raise ValueError(f"{what}: out must be a contiguous CUDA {dtype} tensor of shape "
                         f"({tokens}, {cols}), got {out.device} {out.dtype} {tuple(out.shape)}")


def _stream():
    return torch.cuda.current_stream().cuda_stream


class GluMlp:
    """Fallback-quantized SwiGLU MLP (d_model -> d_ff -> d_model) on B200."""

    def __init__(self, w_gate, w_up, w_down, max_tokens, *, act_dtype=torch.bfloat16,
                 mid_dtype=torch.bfloat16, exact=False, threshold_init=1.0, seed=0x5EED,
                 layer_id_base=0, nonlinear_bits=10, r_min=0.1, r_max=0.3, alpha=1.3,
                 ctx_packed=False):
        wg = np.ascontiguousarray(np.asarray(w_gate, np.float32))
        wu = np.ascontiguousarray(np.asarray(w_up, np.float32))
        wd = np.ascontiguousarray(np.asarray(w_down, np.float32))
        self.d_ff, self.d_model = wg.shape
        assert wu.shape == wg.shape and wd.shape == (self.d_model, self.d_ff)
        cfg = MlpConfig()
        lib.fbq_mlp_default_config(C.byref(cfg))
        cfg.d_model, cfg.d_ff, cfg.max_tokens = self.d_model, self.d_ff, max_tokens
        dt = {torch.float32: K.FBQ_F32, torch.bfloat16: K.FBQ_BF16}
        cfg.act_dtype, cfg.mid_dtype = dt[act_dtype], dt[mid_dtype]
        cfg.epilogue = K.FBQ_EPI_EXACT if exact else K.FBQ_EPI_FMA
        cfg.threshold_init, cfg.seed, cfg.layer_id_base = threshold_init, seed, layer_id_base
        cfg.nonlinear_bits, cfg.r_min, cfg.r_max, cfg.alpha = nonlinear_bits, r_min, r_max, alpha
        # GluCombine a / b contexts: int16 codes (the reference's storage) or
        # packed 10-bit planes (the paper's context memory)
        cfg.ctx_format = 1 if ctx_packed else 0
        self.cfg = cfg
        self.act_dtype = act_dtype
        self.max_tokens = max_tokens
        self._create(cfg, wg, wu, wd)

    def _create(self, cfg, wg, wu, wd):
        h = lib.fbq_mlp_create(C.byref(cfg), wg, wu, wd)
        if not h:
            raise K.FbqError(K.FBQ_ERR_ARG, f"fbq_mlp_create ({lib.fbq_host_last_error().decode()})")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # (module globals are gone at interpreter exit)
            lib.fbq_mlp_destroy(h)
            self._h = None

    # -- device API ----------------------------------------------------------
    def forward(self, x: torch.Tensor, step: int, row_offset: int = 0, out=None):
        _check_act(x, self.act_dtype, self.d_model, "GluMlp.forward x")
        _check_out(out, x.shape[0], self.d_model, self.act_dtype, "GluMlp.forward")
        x = x.contiguous()
        y = out if out is not None else torch.empty_like(x)
        _check(lib.fbq_mlp_forward_device(self._h, x.data_ptr(), x.shape[0], row_offset, step,
                                          y.data_ptr(), _stream()), "forward")
        return y

    def backward(self, gy: torch.Tensor, step: int, row_offset: int = 0, out=None):
        _check_act(gy, self.act_dtype, self.d_model, "GluMlp.backward dY")
        _check_out(out, gy.shape[0], self.d_model, self.act_dtype, "GluMlp.backward")
        gy = gy.contiguous()
        gx = out if out is not None else torch.empty_like(gy)
        _check(lib.fbq_mlp_backward_device(self._h, gy.data_ptr(), gy.shape[0], row_offset, step,
                                           gx.data_ptr(), _stream()), "backward")
        return gx

    def controller_step(self, global_tokens: int | None = None):
        """controller_step (trainsim.cpp:129-133).  Data parallel: after the
        masked counts (count_tensor) were summed over ranks, pass the global
        token count so the rate is that of the whole batch."""
        if global_tokens is None:
            _check(lib.fbq_mlp_controller_step(self._h, _stream()), "controller_step")
        else:
            _check(lib.fbq_mlp_controller_step_blocks(
                self._h, _blocks(global_tokens, self.d_model), _blocks(global_tokens, self.d_ff),
                _stream()), "controller_step")

    def count_tensor(self) -> torch.Tensor:
        """Device int32[2]: masked blocks of the last forward (gate/up, down)."""
        return torch.as_tensor(_DevArray(lib.fbq_mlp_count_ptr(self._h), (2,), "<i4"), device="cuda")

    def zero_grad(self):
        _check(lib.fbq_mlp_zero_grad(self._h, _stream()), "zero_grad")

    def wait_grad(self, which: int, stream) -> None:
        """Make `stream` wait until gradient `which` (0 gate, 1 up, 2 down) of the
        last enqueued backward is final (each right after its own GEMM)."""
        _check(lib.fbq_mlp_wait_grad(self._h, which, stream.cuda_stream), "wait_grad")

    def grad_tensors(self):
        """Device fp32 views (gate+up contiguous, down) for the DP all-reduce."""
        gu = torch.as_tensor(_DevArray(lib.fbq_mlp_grad_ptr(self._h, 0),
                                       (2 * self.d_ff, self.d_model)), device="cuda")
        gd = torch.as_tensor(_DevArray(lib.fbq_mlp_grad_ptr(self._h, 2),
                                       (self.d_model, self.d_ff)), device="cuda")
        return gu, gd

    # -- host API (reference value semantics) --------------------------------
    def step_host(self, x: np.ndarray, gy: np.ndarray, step: int, y=None, gx=None):
        """fwd+bwd over host fp32 buffers (pinned numpy/torch CPU tensors welcome)."""
        t = x.shape[0]
        y = np.empty_like(x) if y is None else y
        gx = np.empty_like(x) if gx is None else gx

        def ptr(a):
            return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data

        _check(lib.fbq_mlp_step_host(self._h, ptr(x), ptr(gy), t, step, ptr(y), ptr(gx)),
               "step_host")
        return y, gx

    STEP_ZERO_GRAD, STEP_CONTROLLER, STEP_SGD = 1, 2, 4

    def step_host_async(self, x, gy, step: int, y, gx, flags: int = 0):
        """Enqueue one pipelined host-buffer step (fbq_mlp_step_host_async); the
        buffers must stay alive and y/gx must not be read before host_sync()."""
        def ptr(a):
            return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data

        _check(lib.fbq_mlp_step_host_async(self._h, ptr(x), ptr(gy), x.shape[0], step, ptr(y),
                                           ptr(gx), flags), "step_host_async")

    def host_sync(self):
        _check(lib.fbq_mlp_host_sync(self._h), "host_sync")

    def grads_host(self):
        gg = np.empty((self.d_ff, self.d_model), np.float32)
        gu = np.empty_like(gg)
        gd = np.empty((self.d_model, self.d_ff), np.float32)
        _check(lib.fbq_mlp_get_grads(self._h, gg.ctypes.data, gu.ctypes.data, gd.ctypes.data),
               "get_grads")
        return gg, gu, gd

    def apply_sgd(self, lr: float):
        """QuantLinearLayer::apply_sgd on gate, up, down (trainsim.cpp:137-143), on the
        current stream after the backward; fused with the next forward's RTN(W)."""
        _check(lib.fbq_mlp_apply_sgd(self._h, lr, _stream()), "apply_sgd")

    def set_sgd_lr(self, lr: float):
        """Learning rate of STEP_SGD in step_host_async."""
        _check(lib.fbq_mlp_set_sgd_lr(self._h, lr), "set_sgd_lr")

    def weights_host(self):
        wg = np.empty((self.d_ff, self.d_model), np.float32)
        wu = np.empty_like(wg)
        wd = np.empty((self.d_model, self.d_ff), np.float32)
        _check(lib.fbq_mlp_get_weights(self._h, wg.ctypes.data, wu.ctypes.data, wd.ctypes.data),
               "get_weights")
        return wg, wu, wd

    def set_thresholds(self, theta_gate_up: float, theta_down: float):
        _check(lib.fbq_mlp_set_thresholds(self._h, theta_gate_up, theta_down), "set_thresholds")

    def context_bytes(self, tokens: int):
        """(bytes saved for the backward by this driver, bytes a BF16 MLP saves)
        at `tokens` tokens -- PAPER.md:527,535 (contexts at 62 % of BF16)."""
        ours, bf = C.c_int64(), C.c_int64()
        _check(lib.fbq_mlp_context_bytes(self._h, tokens, C.byref(ours), C.byref(bf)), "context_bytes")
        return ours.value, bf.value

    def set_profiling(self, on: bool):
        _check(lib.fbq_mlp_set_profiling(self._h, int(on)), "set_profiling")

    def gemm_time(self):
        """(summed GEMM milliseconds, number of GEMM launches) since the last call."""
        ms, n = C.c_double(), C.c_int64()
        _check(lib.fbq_mlp_gemm_time(self._h, C.byref(ms), C.byref(n)), "gemm_time")
        return ms.value, n.value

    def launch_count(self) -> int:
        return lib.fbq_mlp_launch_count(self._h)

    def controller_state(self):
        r = (C.c_double * 2)()
        t = (C.c_double * 2)()
        _check(lib.fbq_mlp_get_controller(self._h, r, t), "get_controller")
        return list(r), list(t)


class GluBlock(GluMlp):
    """The reference's pre-norm residual GLU block (GluBlock, trainsim.hpp:136-146,
    trainsim.cpp:294-308): out = h + down(silu(gate(norm(h))) * up(norm(h))), with
    the RmsNorm (gain 1 at start) fused into the gate/up input quantizer and the
    residual adds fused into the down GEMM / the norm backward
    (include/fbq_b200_host.h, fbq_glublock_*).  Every GluMlp method that reads or
    steers the linears (controller_step, grads_host, weights_host,
    controller_state, set_thresholds, wait_grad, ...) acts on the block's
    gate/up/down driver."""

    def _create(self, cfg, wg, wu, wd):
        b = lib.fbq_glublock_create(C.byref(cfg), wg, wu, wd)
        if not b:
            raise K.FbqError(K.FBQ_ERR_ARG, f"fbq_glublock_create ({lib.fbq_host_last_error().decode()})")
        self._b = b
        self._h = lib.fbq_glublock_mlp(b)  # owned by the block

    def __del__(self):
        b = getattr(self, "_b", None)
        if b and lib is not None:
            lib.fbq_glublock_destroy(b)
            self._b = self._h = None

    def forward(self, h: torch.Tensor, step: int, row_offset: int = 0, out=None):
        _check_act(h, self.act_dtype, self.d_model, "GluBlock.forward h")
        _check_out(out, h.shape[0], self.d_model, self.act_dtype, "GluBlock.forward")
        h = h.contiguous()
        y = out if out is not None else torch.empty_like(h)
        _check(lib.fbq_glublock_forward_device(self._b, h.data_ptr(), h.shape[0], row_offset, step,
                                               y.data_ptr(), _stream()), "GluBlock forward")
        return y

    def backward(self, grad_out: torch.Tensor, step: int, row_offset: int = 0, out=None):
        _check_act(grad_out, self.act_dtype, self.d_model, "GluBlock.backward grad_out")
        _check_out(out, grad_out.shape[0], self.d_model, self.act_dtype, "GluBlock.backward")
        grad_out = grad_out.contiguous()
        gh = out if out is not None else torch.empty_like(grad_out)
        _check(lib.fbq_glublock_backward_device(self._b, grad_out.data_ptr(), grad_out.shape[0], row_offset,
                                                step, gh.data_ptr(), _stream()), "GluBlock backward")
        return gh

    def zero_grad(self):
        _check(lib.fbq_glublock_zero_grad(self._b, _stream()), "GluBlock zero_grad")

    def apply_sgd(self, lr: float):
        _check(lib.fbq_glublock_apply_sgd(self._b, lr, _stream()), "GluBlock apply_sgd")

    def gain_host(self):
        """(gain, grad_gain) of the block's RmsNorm, host fp32 (synchronous)."""
        g = np.empty(self.d_model, np.float32)
        gg = np.empty(self.d_model, np.float32)
        _check(lib.fbq_glublock_get_gain(self._b, g.ctypes.data, gg.ctypes.data), "GluBlock get_gain")
        return g, gg

    def gain_tensors(self):
        """Device fp32 views (gain, grad_gain) of the block's RmsNorm (DP all-reduce)."""
        return tuple(torch.as_tensor(_DevArray(lib.fbq_glublock_gain_ptr(self._b, w), (self.d_model,)),
                                     device="cuda") for w in (0, 1))

    def step_host(self, *a, **k):  # the host-buffer step APIs belong to the bare MLP driver
        raise NotImplementedError("GluBlock: use the device API")

    step_host_async = step_host


class QuantLinear:
    """One fallback-quantized linear layer on B200 -- the reference's
    QuantLinearLayer (trainsim.hpp:38-73, trainsim.cpp:61-135): forward keeps the
    stochastic X context, backward returns dX and accumulates dW."""

    def __init__(self, weight, max_tokens, *, act_dtype=torch.bfloat16, exact=False,
                 threshold_init=1.0, seed=0x5EED, layer_id=0, r_min=0.1, r_max=0.3, alpha=1.3,
                 fallback_mode="threshold", fixed_rate=0.0):
        w = np.ascontiguousarray(np.asarray(weight, np.float32))
        self.out_features, self.in_features = w.shape
        cfg = LinearConfig()
        lib.fbq_linear_default_config(C.byref(cfg))
        cfg.in_features, cfg.out_features, cfg.max_tokens = self.in_features, self.out_features, max_tokens
        cfg.act_dtype = {torch.float32: K.FBQ_F32, torch.bfloat16: K.FBQ_BF16}[act_dtype]
        cfg.epilogue = K.FBQ_EPI_EXACT if exact else K.FBQ_EPI_FMA
        cfg.layer_id, cfg.seed, cfg.threshold_init = layer_id, seed, threshold_init
        cfg.r_min, cfg.r_max, cfg.alpha = r_min, r_max, alpha
        cfg.fallback_mode = {"threshold": 0, "fixed_rate": 1, "off": 2}[fallback_mode]
        cfg.fixed_rate = fixed_rate
        self.cfg, self.act_dtype, self.max_tokens = cfg, act_dtype, max_tokens
        h = lib.fbq_linear_create(C.byref(cfg), w)
        if not h:
            raise K.FbqError(K.FBQ_ERR_ARG, f"fbq_linear_create ({lib.fbq_host_last_error().decode()})")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib.fbq_linear_destroy(h)
            self._h = None

    def forward(self, x: torch.Tensor, step: int, row_offset: int = 0, out=None):
        _check_act(x, self.act_dtype, self.in_features, "QuantLinear.forward x")
        _check_out(out, x.shape[0], self.out_features, self.act_dtype, "QuantLinear.forward")
        if x.shape[0] > self.max_tokens:
            raise ValueError(f"QuantLinear.forward: {x.shape[0]} tokens > max_tokens {self.max_tokens}")
        x = x.contiguous()
        y = out if out is not None else torch.empty(x.shape[0], self.out_features, device=x.device,
                                                    dtype=self.act_dtype)
        _check(lib.fbq_linear_forward_device(self._h, x.data_ptr(), x.shape[0], row_offset, step,
                                             y.data_ptr(), _stream()), "linear forward")
        return y

    def backward(self, gy: torch.Tensor, step: int, row_offset: int = 0, out=None):
        _check_act(gy, self.act_dtype, self.out_features, "QuantLinear.backward dY")
        _check_out(out, gy.shape[0], self.in_features, self.act_dtype, "QuantLinear.backward")
        if gy.shape[0] > self.max_tokens:
            raise ValueError(f"QuantLinear.backward: {gy.shape[0]} tokens > max_tokens {self.max_tokens}")
        gy = gy.contiguous()
        gx = out if out is not None else torch.empty(gy.shape[0], self.in_features, device=gy.device,
                                                     dtype=self.act_dtype)
        _check(lib.fbq_linear_backward_device(self._h, gy.data_ptr(), gy.shape[0], row_offset, step,
                                              gx.data_ptr(), _stream()), "linear backward")
        return gx

    def controller_step(self, global_tokens: int | None = None):
        if global_tokens is None:
            _check(lib.fbq_linear_controller_step(self._h, _stream()), "linear controller_step")
        else:
            _check(lib.fbq_linear_controller_step_blocks(
                self._h, _blocks(global_tokens, self.in_features), _stream()), "linear controller_step")

    def count_tensor(self) -> torch.Tensor:
        """Device int32[1]: masked blocks of the last forward (Threshold mode)."""
        return torch.as_tensor(_DevArray(lib.fbq_linear_count_ptr(self._h), (1,), "<i4"), device="cuda")

    def zero_grad(self):
        _check(lib.fbq_linear_zero_grad(self._h, _stream()), "linear zero_grad")

    def grad(self) -> torch.Tensor:
        return torch.as_tensor(_DevArray(lib.fbq_linear_grad_ptr(self._h),
                                         (self.out_features, self.in_features)), device="cuda")

    def controller_state(self):
        r, t = C.c_double(), C.c_double()
        _check(lib.fbq_linear_get_controller(self._h, C.byref(r), C.byref(t)), "linear get_controller")
        return r.value, t.value

    def apply_sgd(self, lr: float):
        """QuantLinearLayer::apply_sgd (trainsim.cpp:137-143), fused with the next forward's RTN(W)."""
        _check(lib.fbq_linear_apply_sgd(self._h, lr, _stream()), "linear apply_sgd")

    def weight_host(self):
        w = np.empty((self.out_features, self.in_features), np.float32)
        _check(lib.fbq_linear_get_weight(self._h, w.ctypes.data), "linear get_weight")
        return w
