"""Generate golden vectors by running the UNMODIFIED reference (oracle/_ref).

    make -C oracle ref && python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Inputs are stored alongside the outputs so
the fixtures are self-contained (the GPU box has no /root/reference).
Residuals are stored in the reference's own compact form (residuals[] in
mask order + residual_index[], quant.hpp:46-52).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import REF_oracle, dense_to_compact  # noqa: E402
from tests.helpers import outlier_matrix  # noqa: E402


def main():
    R = REF_oracle()
    if R is None:
        raise SystemExit("oracle/_ref/libfbq_ref.so not built (make -C oracle ref)")
    g = {}
    # rng.hpp streams
    seeds = np.array([0, 1, 0x5EED, 2**63 + 12345], np.uint64)
    ns = np.array([0, 1, 2, 1000, 2**40 + 7], np.uint64)
    g["rng_seeds"], g["rng_ns"] = seeds, ns
    g["rng_bits"] = np.array([[R.bits_at(int(s), int(n)) for n in ns] for s in seeds], np.uint64)
    g["rng_uniform"] = np.array([[R.uniform_at(int(s), int(n)) for n in ns] for s in seeds])
    g["rng_normal"] = np.array([[R.normal_at(int(s), int(n)) for n in ns] for s in seeds],
                               np.float32)
    g["derive_seed"] = np.array([R.derive_seed(0x5EED, a, b) for a in range(6) for b in range(3)],
                                np.uint64)

    # quantize_rtn, ragged both ways (quant.cpp:36-53)
    x = outlier_matrix(200, 300, seed=101, channels=[5, 250], tokens=[17], occasional=4)
    g["rtn_x"] = x
    g["rtn_codes"], g["rtn_scales"] = R.quantize_rtn(x)

    # quantize_stochastic (quant.cpp:55-84), seed as layer_seed(0x5eed, 2, 1, 9)
    x = outlier_matrix(128, 384, seed=102, channels=[33])
    seed = R.layer_seed(0x5EED, 2, 1, 9)
    g["sr_x"], g["sr_seed"] = x, np.uint64(seed)
    g["sr_codes"], g["sr_scales"] = R.quantize_stochastic(x, seed)

    # score_blocks + mask_topk + fallback_quantize (policy.cpp, quant.cpp:128-176)
    x = outlier_matrix(256, 384, seed=103, channels=[7], tokens=[200], occasional=6)
    scores = R.score_blocks_absmax(x)
    mask = R.mask_topk(scores, 0.34)
    c, s, rc, rs = R.fallback_quantize(x, mask)
    rcomp, rsc, ridx = dense_to_compact(rc, rs, mask, 128)
    g.update(fb_x=x, fb_scores=scores, fb_mask=mask, fb_codes=c, fb_scales=s,
             fb_res_compact=rcomp, fb_res_scales=rsc, fb_res_index=ridx)
    g["fb_mask_thr"] = R.mask_threshold(scores, float(np.median(scores)))
    g["fb_theta"] = float(np.median(scores))
    g["fb_dequant"] = R.dequantize_fallback(c, s, mask, rc, rs)

    # block_quant_gemm / fallback_gemm / tiled (gemm.cpp:101-203): A = fb x, B K x N
    b = outlier_matrix(384, 200, seed=104, body=0.02)
    bc, bs = R.quantize_rtn(b)
    g["gemm_b"] = b
    g["gemm_block"] = R.block_gemm(c, s, bc, bs)
    g["gemm_fallback"] = R.block_gemm(c, s, bc, bs, mask=mask, res_codes=rc, res_scales=rs)
    g["gemm_tiled"] = R.block_gemm(c, s, bc, bs, tile=(32, 64, 16))
    g["gemm_oracle"] = R.gemm_oracle(R.dequantize_fallback(c, s, mask, rc, rs), R.dequantize(bc, bs))

    # controller (policy.cpp:97-109)
    g["ctl"] = np.array([R.controller_update(1.0, r) for r in (0.05, 0.35, 0.2, 0.1, 0.3)])

    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
