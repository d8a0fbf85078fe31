"""B200-native (sm_100a) Fallback-Quantization hot path.

Reference-shaped operator API: ``paper_2503_08040_b200.fbq`` (quantize_rtn,
quantize_stochastic, fallback_quantize, dequantize[_fallback], transpose,
block_quant_gemm, fallback_gemm, score_blocks, mask_threshold, mask_topk,
mask_rate, controller_update).  Linear / MLP drivers: ``.linear``.
C ABI: include/fbq_b200.h, implemented by lib/libfbq_b200.so.

Submodules load lib/libfbq_b200.so on first use and raise ImportError if it
is missing (build with ``python -m paper_2503_08040_b200.build``): there is no
CPU fallback.
"""
import importlib

__all__ = ["fbq", "linear"]


def __getattr__(name):
    if name in __all__:
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
