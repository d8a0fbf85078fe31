"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
host-side logic (bitmaps, policy mirror, seeds) matches the oracle."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w\s\*]+?\b(fbq_\w+)\s*\(", src, flags=re.M):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol():
    from paper_2503_08040_b200 import _capi
    syms = declared_symbols()
    assert len(syms) >= 12, syms
    lib = ctypes.CDLL(_capi.LIB_PATH)
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    from paper_2503_08040_b200 import _capi
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_and_argument_errors_without_gpu():
    """Validation happens before any CUDA call, so it works on a CPU box."""
    from paper_2503_08040_b200 import _capi as K
    lib = K.lib
    assert lib.fbq_block_side() == 128
    assert lib.fbq_status_string(K.FBQ_ERR_SHAPE) == b"shape/geometry mismatch"
    # bad dtype / negative shape / null output / misaligned ld
    assert lib.fbq_cuda_quantize_rtn(None, 7, 1, 1, 1, None, 16, None, None) == K.FBQ_ERR_ARG
    assert lib.fbq_cuda_quantize_rtn(None, 0, -1, 1, 1, None, 16, None, None) == K.FBQ_ERR_SHAPE
    assert lib.fbq_cuda_quantize_rtn(None, 0, 0, 0, 0, None, 16, None, None) == K.FBQ_OK
    assert lib.fbq_cuda_gemm(1024, 24, 1, 0, 2048, 32, 1, 0, None, None, None, 128, 128, 128,
                             4096, 0, 128, 0, 0, None) == K.FBQ_ERR_UNSUPPORTED
    assert lib.fbq_cuda_gemm(None, 16, None, 0, None, 16, None, 0, None, None, None, 0, 5, 5,
                             None, 0, 5, 0, 0, None) == K.FBQ_OK
    assert lib.fbq_cuda_gemm(None, 16, None, 3, None, 16, None, 0, None, None, None, 1, 1, 1,
                             None, 0, 1, 0, 0, None) == K.FBQ_ERR_ARG
    assert lib.fbq_cuda_quantize_fallback(1024, 0, 4, 4, 4, 1, 0.0, 2048, None, 16, None, None,
                                          None, None, None, None, 0, 0, None) == K.FBQ_ERR_ARG


def test_mask_bits_roundtrip():
    import torch
    from paper_2503_08040_b200 import fbq
    rng = np.random.default_rng(0)
    for gr, gc in [(1, 1), (3, 11), (64, 112), (7, 33)]:
        m = torch.from_numpy((rng.random((gr, gc)) < 0.3).astype(np.uint8))
        bits = fbq.mask_to_bits(m)
        assert bits.numel() == (gr * gc + 31) // 32
        assert torch.equal(fbq.bits_to_mask(bits, gr, gc), m)


def test_policy_mirror_matches_oracle(orc):
    import torch
    from paper_2503_08040_b200 import fbq
    rng = np.random.default_rng(1)
    for n in [1, 4, 100, 7168]:
        s = np.round(rng.random(n) * 10, 1)  # many ties
        for rate in [0.0, 0.05, 0.2, 0.5, 1.0]:
            got = fbq.mask_topk(torch.from_numpy(s), rate).numpy()
            assert np.array_equal(got, orc.mask_topk(s, rate))
        got = fbq.mask_threshold(torch.from_numpy(s), 5.0).numpy()
        assert np.array_equal(got, orc.mask_threshold(s, 5.0))
        assert fbq.mask_rate(torch.from_numpy(got)) == orc.mask_rate(got)
    st = fbq.FallbackThresholdState(1.0)
    for r in [0.05, 0.05, 0.5, 0.2, 0.31, 0.0]:
        st2 = fbq.controller_update(st, r)
        assert st2.threshold == orc.controller_update(st.threshold, r)
        st = st2
    with pytest.raises(ValueError):
        fbq.controller_update(st, 1.5)
    with pytest.raises(ValueError):
        fbq.mask_threshold(torch.zeros(3), 0.0)
    with pytest.raises(ValueError):
        fbq.ControllerConfig(0.3, 0.1, 1.3)


def test_seed_derivation_matches_oracle(orc):
    from paper_2503_08040_b200 import fbq
    for a in range(5):
        for b in range(4):
            assert fbq.derive_seed(0x5EED, a, b) == orc.derive_seed(0x5EED, a, b)
            assert fbq.bits_at(12345 + a, b) == orc.bits_at(12345 + a, b)


def test_ops_refuse_cpu_tensors():
    import torch
    from paper_2503_08040_b200 import fbq
    with pytest.raises(ValueError):
        fbq.quantize_rtn(torch.zeros(4, 4))
    with pytest.raises(NotImplementedError):
        fbq.quantize_rtn(torch.zeros(4, 4), block=32)


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without the sm_100a library the package refuses to import."""
    import subprocess
    import sys
    env = dict(os.environ, FBQ_B200_LIB_OVERRIDE=str(tmp_path / "absent" / "libfbq_b200.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_2503_08040_b200.fbq"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "no CPU fallback" in r.stderr
