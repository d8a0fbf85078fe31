"""GPU: the bit-exact fp32 rounding of K1/K2/GLU (fbq_round.cuh) against the
reference's double formulas (kernels.cpp:24-40, quant.cpp:66-80), via the
element-wise probe kernel: an exhaustive binade of x, adversarial near-ties,
every scale binade incl. subnormal/tiny scales, and SR near-threshold cases --
for the scalar functions (path 0) and for the vector fast paths with their
exact fallback that the kernels run (path 1: 8-bit RTN / SR, path 2: the
10-bit context RTN)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def ref_rtn(x, a, level=127):
    t = np.rint(x.astype(np.float64) / a.astype(np.float64))  # numpy rint = ties-to-even
    return np.clip(t, -level, level).astype(np.int16 if level > 127 else np.int8)


def mix64(z):
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def ref_sr(x, a, bits):
    t = x.astype(np.float64) / a.astype(np.float64)
    f = np.floor(t)
    frac = t - f
    u = (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    f = np.where((frac > 0) & (u < frac), f + 1, f)
    return np.clip(f, -127, 127).astype(np.int8)


def probe(x, a, bits=None, path=0, rtn=True):
    import torch
    from paper_2503_08040_b200 import _capi as K
    n = x.size
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ad = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    bd = torch.from_numpy(bits.view(np.int64)).cuda() if bits is not None else None
    o_r = torch.empty(n, dtype=torch.int16 if path in (2, 4) else torch.int8, device="cuda") if rtn else None
    o_s = torch.empty(n, dtype=torch.int8, device="cuda") if bits is not None else None
    K.check(K.lib.fbq_cuda_round_probe(xd.data_ptr(), ad.data_ptr(),
                                       bd.data_ptr() if bd is not None else None,
                                       o_r.data_ptr() if o_r is not None else None,
                                       o_s.data_ptr() if o_s is not None else None, n, path,
                                       torch.cuda.current_stream().cuda_stream), "probe")
    torch.cuda.synchronize()
    return (o_r.cpu().numpy() if o_r is not None else None), (o_s.cpu().numpy() if o_s is not None else None)


def near_tie_inputs(rng, n, level, emin=-149, emax=100):
    e = rng.integers(emin, emax, n)
    a = (rng.uniform(1, 2, n) * 2.0 ** e).astype(np.float32)
    a = np.where(a == 0, np.float32(1e-45), a).astype(np.float32)
    k = rng.integers(-level, level + 1, n)
    base = ((k + 0.5 * rng.choice([-1, 1], n)) * a.astype(np.float64)).astype(np.float32)
    jitter = rng.integers(-3, 4, n).astype(np.int32)
    x = (base.view(np.int32) + jitter).view(np.float32)
    x[::7] = (k[::7] * a[::7].astype(np.float64)).astype(np.float32)
    ok = np.isfinite(x) & np.isfinite(base)
    return x[ok], a[ok]


@pytest.mark.parametrize("path", [0, 1])
def test_rtn_exhaustive_binade(path):
    """Every float in [1, 2) (2^23 values) against several scales."""
    x = (np.arange(1 << 23, dtype=np.uint32) | np.uint32(0x3F800000)).view(np.float32)
    for amax in (2.0, 1.9999999, 1.7320508, 1.0000001):
        xs = x if path == 0 else x[x <= np.float32(amax)]  # path 1: the kernels' domain |x| <= amax
        a = np.full_like(xs, np.float32(amax) / np.float32(127.0))
        for sgn in (1, -1):
            got, _ = probe(sgn * xs, a, path=path)
            assert np.array_equal(got, ref_rtn(sgn * xs, a)), (amax, sgn, path)


@pytest.mark.parametrize("path", [0, 1])
def test_rtn_near_ties_all_scale_binades(path):
    rng = np.random.default_rng(0)
    x, a = near_tie_inputs(rng, 1 << 22, 127)
    if path == 1:  # the kernels' domain: |x| <= amax = 127 a (up to a's rounding)
        keep = np.abs(x.astype(np.float64)) <= 127 * a.astype(np.float64)
        x, a = x[keep], a[keep]
    got, _ = probe(x, a, path=path)
    assert np.array_equal(got, ref_rtn(x, a))


def test_rtn_packed_vector_path_near_ties():
    """Path 3: the 8-wide packed fast path (FMUL2/FADD2/FFMA2, 3-input |d|
    max) with its exact fallback, on vectors sharing one scale: near-ties,
    exact ties, repeated values and tiny scales."""
    rng = np.random.default_rng(5)
    n = 1 << 21
    g = n // 8
    e = rng.integers(-140, 60, g)
    a = np.repeat((rng.uniform(1, 2, g) * 2.0 ** e).astype(np.float32), 8)
    k = rng.integers(-127, 128, n)
    half = 0.5 * rng.choice([-1, 1, 0], n)
    base = ((k + half) * a.astype(np.float64)).astype(np.float32)
    jit = rng.integers(-3, 4, n).astype(np.int32)
    x = (base.view(np.int32) + jit).view(np.float32)
    x[::5] = np.repeat(x[::40], 8)[: x[::5].size]  # repeated values across vectors
    amax = 127 * a.astype(np.float64)
    x = np.where(np.abs(x.astype(np.float64)) <= amax, x, (np.sign(x) * amax).astype(np.float32))
    x = np.where(np.isfinite(x), x, 0).astype(np.float32)
    got, _ = probe(x, a, path=3)
    assert np.array_equal(got, ref_rtn(x, a))


def test_rtn10_packed_vector_path_near_ties():
    """Path 4: group_rtn's packed level-511 path (10-bit contexts) -- the fast
    path's window(511) boundary test and the packed exact fix (parity-denormal
    tie rule) on vectors sharing one scale: near-ties, exact ties, repeated values."""
    rng = np.random.default_rng(15)
    n = 1 << 21
    g = n // 8
    e = rng.integers(-140, 60, g)
    a = np.repeat((rng.uniform(1, 2, g) * 2.0 ** e).astype(np.float32), 8)
    k = rng.integers(-511, 512, n)
    half = 0.5 * rng.choice([-1, 1, 0], n)
    base = ((k + half) * a.astype(np.float64)).astype(np.float32)
    jit = rng.integers(-3, 4, n).astype(np.int32)
    x = (base.view(np.int32) + jit).view(np.float32)
    x[::5] = np.repeat(x[::40], 8)[: x[::5].size]
    amax = 511 * a.astype(np.float64)
    x = np.where(np.abs(x.astype(np.float64)) <= amax, x, (np.sign(x) * amax).astype(np.float32))
    x = np.where(np.isfinite(x), x, 0).astype(np.float32)
    got, _ = probe(x, a, path=4)
    assert np.array_equal(got, ref_rtn(x, a, 511))


def test_rtn10_context_path():
    rng = np.random.default_rng(3)
    x, a = near_tie_inputs(rng, 1 << 22, 511)
    keep = np.abs(x.astype(np.float64)) <= 511 * a.astype(np.float64)
    x, a = x[keep], a[keep]
    got, _ = probe(x, a, path=2)
    assert np.array_equal(got, ref_rtn(x, a, 511))


def sr_cases(rng, n, counters):
    e = rng.integers(-140, 60, n)
    a = (rng.uniform(1, 2, n) * 2.0 ** e).astype(np.float32)
    x = (rng.uniform(-127, 127, n) * a.astype(np.float64)).astype(np.float32)
    x[::11] = (np.rint(x[::11].astype(np.float64) / a[::11]) * a[::11]).astype(np.float32)  # frac == 0
    x[::13] = (127 * a[::13].astype(np.float64)).astype(np.float32)                          # the amax element
    keep = np.abs(x.astype(np.float64)) <= 127 * a.astype(np.float64)
    x, a = x[keep], a[keep]
    m = x.size
    if not counters:
        bits = rng.integers(0, 2 ** 63, m, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, m, dtype=np.uint64)
        t = x.astype(np.float64) / a.astype(np.float64)
        frac = t - np.floor(t)
        near = (np.clip(frac, 0, 1 - 2 ** -53) * 2.0 ** 53).astype(np.uint64)
        sel = rng.random(m) < 0.25
        delta = rng.integers(-2 ** 20, 2 ** 20, m).astype(np.int64)
        forced = ((near.astype(np.int64) + delta).clip(0, 2 ** 53 - 1).astype(np.uint64)) << np.uint64(11)
        return x, a, np.where(sel, forced, bits).astype(np.uint64)
    z = rng.integers(0, 2 ** 63, m, dtype=np.uint64) * np.uint64(2)
    return x, a, z


def test_stochastic_rounding_adversarial_scalar():
    rng = np.random.default_rng(1)
    x, a, bits = sr_cases(rng, 1 << 22, counters=False)
    rtn, sr = probe(x, a, bits, path=0)
    assert np.array_equal(sr, ref_sr(x, a, bits))
    assert np.array_equal(rtn, ref_rtn(x, a))


def test_stochastic_rounding_vector_path():
    """The kernels' SR path takes the splitmix64 counter and decides with the
    top 23 mixed bits; the reference uses all 53 -- compare on the mixed bits."""
    rng = np.random.default_rng(2)
    x, a, z = sr_cases(rng, 1 << 22, counters=True)
    # force near-threshold cases: search counters whose u lands within 2^-20 of frac
    rtn, sr = probe(x, a, z, path=1)
    bits = mix64(z)
    assert np.array_equal(sr, ref_sr(x, a, bits))
    assert np.array_equal(rtn, ref_rtn(x, a))
    # near-threshold: choose x so that frac == u(bits) up to a few ulp
    u = (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    k = np.floor(x.astype(np.float64) / a)
    x2 = ((k + u) * a.astype(np.float64)).astype(np.float32)
    keep = np.abs(x2.astype(np.float64)) <= 127 * a.astype(np.float64)
    x2, a2, z2, b2 = x2[keep], a[keep], z[keep], bits[keep]
    _, sr2 = probe(x2, a2, z2, path=1, rtn=False)
    assert np.array_equal(sr2, ref_sr(x2, a2, b2))
