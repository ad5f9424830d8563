"""fp32 storage/streaming (dtype "f32": panels and vectors in fp32, each
lane's chunk-local partial sums in fp32, every cross-lane reduction and the
k x k algebra in fp64) against the fp64 oracle with the north star's fp32
tolerance, 1e-4 relative per iterate."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL32 = 1e-4


def rel(a, b):
    return np.linalg.norm(np.asarray(a, dtype=np.float64) - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n", [257, 5000, 70001])
def test_f32_haar_probe_sequence(orc, lm, n):
    seed, T = 3 + n, 20
    sides = ["right" if t % 4 else "left" for t in range(T)]
    ref = orc.Operator("haar", n=n, seed=seed)
    op = lm.HaarOperator(n, seed=seed, dtype="f32", draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    aux = orc.RandomSource(seed + 1)
    for t, s in enumerate(sides):
        x = aux.normal_vector(n).astype(np.float32)
        got, want = op.probe(x, s), ref.probe(x.astype(np.float64), s)
        assert got.dtype == np.float32
        assert rel(got, want) < TOL32, (t, s, rel(got, want))


def test_f32_haar_tanh_mix_run_and_goe(orc, lm):
    n, T, seed = 20000, 30, 8
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    x1 = x1.astype(np.float32).astype(np.float64)  # the fp32 operator starts from the rounded x_1
    want = orc.Operator("haar", n=n, seed=seed).run("tanh_mix", "right", T, x1, keep=True)
    op = lm.HaarOperator(n, seed=seed, dtype="f32", draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1.astype(np.float32), T, update="tanh_mix", sides="right", keep_trajectory=True)
    assert max(rel(got[t], want[t]) for t in range(T + 1)) < TOL32
    n = 3000
    ref = orc.Operator("goe", n=n, sigma=n ** -0.5, seed=seed)
    op = lm.GOEOperator(n, seed, sigma=n ** -0.5, dtype="f32", draws="injected", capacity=10)
    op.push_draws(orc.draws_for(seed, [n] * 20))
    aux = orc.RandomSource(9)
    for _ in range(10):
        x = aux.normal_vector(n).astype(np.float32)
        assert rel(op.probe(x), ref.probe(x.astype(np.float64), "right")) < TOL32


def test_f32_rectangular_ginibre_and_shards(orc, lm):
    m, n, seed, T = 2100, 1500, 4, 16
    sides = ["right" if t % 2 == 0 else "left" for t in range(T)]
    draws = orc.draws_for(seed, [m if s == "right" else n for s in sides])
    aux = orc.RandomSource(5)
    seq = [(aux.normal_vector(n if s == "right" else m).astype(np.float32), s) for s in sides]
    ref = orc.Operator("ginibre", m=m, n=n, sigma=0.6, seed=seed)
    want = [ref.probe(x.astype(np.float64), s) for x, s in seq]
    op = lm.GinibreOperator(m, n, 0.6, seed, dtype="f32", draws="injected", capacity=T)
    op.push_draws(draws)
    for t, (x, s) in enumerate(seq):
        assert rel(op.probe(x, s), want[t]) < TOL32, t
    # the same operator as two row shards (virtual shards, in-process exchange)
    ex, outs, errs = lm.Exchange.local(2), [None, None], []

    def worker(r):
        try:
            sh = lm.GinibreOperator(m, n, 0.6, seed, dtype="f32", draws="injected", capacity=T, shard=(r, 2),
                                    exchange=ex)
            sh.push_draws(draws)
            res = []
            for x, s in seq:
                lo, hi = sh.shard_range("cols" if s == "right" else "rows")
                res.append(sh.probe(np.ascontiguousarray(x[lo:hi]), s))
            outs[r] = res
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs
    for t in range(T):
        assert rel(np.concatenate([outs[0][t], outs[1][t]]), want[t]) < TOL32, t


def test_f32_config2_scale_against_f64(lm):
    """Config 2 in fp32 (n = 1e6, T = 100, tanh mix): the fp32 operator (fp32
    panels, chunk-local fp32 partial sums, fp64 reductions and algebra) tracks
    the fp64 operator on the same Philox matrix within the fp32 tolerance over
    the whole trajectory (the fp32 draws are the fp64 draws rounded)."""
    import torch
    n, T, seed = 1_000_000, 100, 12
    x1 = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    x1 /= x1.norm()
    x1 = x1.float().double()
    a = lm.HaarOperator(n, seed=seed, capacity=T)
    b = lm.HaarOperator(n, seed=seed, dtype="f32", capacity=T)
    ya = a.run(x1, T, update="tanh_mix", sides="right", keep_trajectory=True)
    yb = b.run(x1.float(), T, update="tanh_mix", sides="right", keep_trajectory=True)
    errs = [float((yb[t].double() - ya[t]).norm() / ya[t].norm()) for t in range(T + 1)]
    assert max(errs) < TOL32, max(errs)
