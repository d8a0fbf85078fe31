"""GPU: the bit-exact fp32 rounding of K1/K2 (fbq_round.cuh) against the
reference's double formulas (kernels.cpp:24-40, quant.cpp:66-80), via the
element-wise probe kernel: an exhaustive binade of x, adversarial near-ties,
every scale binade incl. subnormal/tiny scales, and SR near-threshold cases."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def ref_rtn(x, a):
    t = np.rint(x.astype(np.float64) / a.astype(np.float64))  # numpy rint = ties-to-even
    return np.clip(t, -127, 127).astype(np.int8)


def ref_sr(x, a, bits):
    t = x.astype(np.float64) / a.astype(np.float64)
    f = np.floor(t)
    frac = t - f
    u = (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    f = np.where((frac > 0) & (u < frac), f + 1, f)
    return np.clip(f, -127, 127).astype(np.int8)


def probe(x, a, bits=None):
    import ctypes
    import torch
    from paper_2503_08040_b200 import _capi as K
    n = x.size
    xd = torch.from_numpy(x).cuda()
    ad = torch.from_numpy(a).cuda()
    bd = torch.from_numpy(bits.view(np.int64)).cuda() if bits is not None else None
    rtn = torch.empty(n, dtype=torch.int8, device="cuda")
    sr = torch.empty(n, dtype=torch.int8, device="cuda") if bits is not None else None
    K.check(K.lib.fbq_cuda_round_probe(xd.data_ptr(), ad.data_ptr(),
                                       bd.data_ptr() if bd is not None else None, rtn.data_ptr(),
                                       sr.data_ptr() if sr is not None else None, n,
                                       torch.cuda.current_stream().cuda_stream), "probe")
    torch.cuda.synchronize()
    return rtn.cpu().numpy(), (sr.cpu().numpy() if sr is not None else None)


def test_rtn_exhaustive_binade():
    """Every float in [1, 2) (2^23 values) against several scales."""
    x = (np.arange(1 << 23, dtype=np.uint32) | np.uint32(0x3F800000)).view(np.float32)
    for amax in (2.0, 1.9999999, 1.7320508, 1.0000001):
        a = np.full_like(x, np.float32(amax) / np.float32(127.0))
        got, _ = probe(x, a)
        assert np.array_equal(got, ref_rtn(x, a)), amax
        got, _ = probe(-x, a)
        assert np.array_equal(got, ref_rtn(-x, a)), amax


def test_rtn_near_ties_all_scale_binades():
    rng = np.random.default_rng(0)
    n = 1 << 22
    e = rng.integers(-149, 100, n)
    a = (rng.uniform(1, 2, n) * 2.0 ** e).astype(np.float32)
    a = np.where(a == 0, np.float32(1e-45), a).astype(np.float32)
    k = rng.integers(-127, 128, n)
    # values within a few ulp of (k +- 1/2) * a, exact ties and random values
    base = ((k + 0.5 * rng.choice([-1, 1], n)) * a.astype(np.float64)).astype(np.float32)
    jitter = rng.integers(-3, 4, n).astype(np.int32)
    x = (base.view(np.int32) + jitter).view(np.float32)
    x = np.where(np.abs(x) > 127 * a, base, x).astype(np.float32)
    x[::7] = (k[::7] * a[::7].astype(np.float64)).astype(np.float32)
    ok = np.isfinite(x)
    x, a = x[ok], a[ok]
    got, _ = probe(x, a)
    assert np.array_equal(got, ref_rtn(x, a))


def test_stochastic_rounding_adversarial():
    rng = np.random.default_rng(1)
    n = 1 << 22
    e = rng.integers(-140, 60, n)
    a = (rng.uniform(1, 2, n) * 2.0 ** e).astype(np.float32)
    x = (rng.uniform(-127, 127, n) * a.astype(np.float64)).astype(np.float32)
    bits = rng.integers(0, 2 ** 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    # force u ~ frac for a quarter of the cases (exercises the exact fallback)
    t = x.astype(np.float64) / a.astype(np.float64)
    frac = t - np.floor(t)
    near = (np.clip(frac, 0, 1 - 2 ** -53) * 2.0 ** 53).astype(np.uint64)
    sel = rng.random(n) < 0.25
    delta = rng.integers(-2 ** 20, 2 ** 20, n).astype(np.int64)
    forced = ((near.astype(np.int64) + delta).clip(0, 2 ** 53 - 1).astype(np.uint64)) << np.uint64(11)
    bits = np.where(sel, forced, bits).astype(np.uint64)
    rtn, sr = probe(x, a, bits)
    assert np.array_equal(sr, ref_sr(x, a, bits))
    assert np.array_equal(rtn, ref_rtn(x, a))
