"""The PHILOX draw stream (include/hd.h hd_philox_normals).

* hd_philox_normals equals a numpy restatement of Philox4x32-10 (Salmon et al.,
  SC'11) + Box-Muller on 53-bit uniforms, to rounding of the transcendentals;
* the stream is deterministic, keyed by the probe index, bounded by
  sqrt(-2 ln 2^-53) and has Gaussian moments and tail frequency;
* a draws="philox" operator consumes exactly that stream: it is bitwise equal
  to an injected-draw operator fed with hd_philox_normals(seed, probe index).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    m32 = np.uint64(0xFFFFFFFF)
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & m32 for c in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0), np.uint64(k1)
    for _ in range(10):
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & m32
        hi1, lo1 = p1 >> np.uint64(32), p1 & m32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + np.uint64(W0)) & m32
        k1 = (k1 + np.uint64(W1)) & m32
    return c0, c1, c2, c3


def philox_normals_np(seed, stream, probe, n):
    q = np.arange((n + 1) // 2, dtype=np.uint64)
    w = philox4x32_10(q & np.uint64(0xFFFFFFFF), q >> np.uint64(32), np.full_like(q, probe),
                      np.full_like(q, stream), seed & 0xFFFFFFFF, seed >> 32)
    a = (w[0] << np.uint64(32)) | w[1]
    b = (w[2] << np.uint64(32)) | w[3]
    u1 = ((a >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (b >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    out = np.empty(2 * len(q))
    out[0::2] = r * np.cos(2 * np.pi * u2)
    out[1::2] = r * np.sin(2 * np.pi * u2)
    return out[:n], u1, u2


@pytest.mark.parametrize("seed,stream,probe,n", [(1, 0, 0, 100_001), (0xDEADBEEFCAFEF00D, 3, 77, 4096),
                                                 (7, 1, 2**31 - 1, 999)])
def test_philox_stream_matches_restatement(lm, seed, stream, probe, n):
    got = lm.philox_normals(seed, probe, n, stream=stream).cpu().numpy()
    want, _, _ = philox_normals_np(seed, stream, probe, n)
    assert got.shape == (n,)
    # numpy's sin(2*pi*u) carries the rounding of 2*pi*u (<= 4.4e-16 absolute
    # at u ~ 1, times r <= 8.6); the device reduces u exactly first
    assert np.max(np.abs(got - want)) < 1e-13
    assert abs(got.mean()) < 5 / np.sqrt(n) and abs(got.std() - 1) < 5 / np.sqrt(n)


def test_philox_stream_tails_and_determinism(lm):
    n = 1 << 21
    a = lm.philox_normals(11, 5, n).cpu().numpy()
    b = lm.philox_normals(11, 5, n).cpu().numpy()
    assert np.array_equal(a, b)
    c = lm.philox_normals(11, 6, n).cpu().numpy()
    assert not np.array_equal(a, c)
    assert np.all(np.isfinite(a)) and np.max(np.abs(a)) < 8.58  # sqrt(-2 ln 2^-53)
    want, _, _ = philox_normals_np(11, 0, 5, n)
    assert np.max(np.abs(a - want)) < 1e-13
    # 5-sigma tail frequency within its binomial band
    p = 5.733e-7
    assert abs(np.sum(np.abs(a) > 5) - p * n) < 6 * np.sqrt(p * n) + 1


@pytest.mark.parametrize("ens", ["haar", "ginibre"])
def test_operator_consumes_the_philox_stream(lm, ens):
    import torch
    seed, T = 99, 14
    if ens == "haar":
        n = 20_001
        a = lm.HaarOperator(n, seed=seed, capacity=T)
        b = lm.HaarOperator(n, seed=seed, draws="injected", capacity=T)
        lens = [n] * T
        sides = ["right"] * (T // 2) + ["left"] * (T - T // 2)
    else:
        m, n = 9_000, 12_345
        a = lm.GinibreOperator(m, n, 0.3, seed, capacity=T)
        b = lm.GinibreOperator(m, n, 0.3, seed, draws="injected", capacity=T)
        sides = ["right", "left"] * (T // 2)
        lens = [m if s == "right" else n for s in sides]
    draws = [lm.philox_normals(seed, k, L).cpu().numpy() for k, L in enumerate(lens)]
    b.push_draws(np.concatenate(draws))
    rng = np.random.default_rng(3)
    for s in sides:
        x = rng.standard_normal(n if s == "right" else (m if ens == "ginibre" else n))
        ya, yb = np.asarray(a.probe(x, s)), np.asarray(b.probe(x, s))
        assert np.array_equal(ya, yb)
    torch.cuda.synchronize()
