"""Read-before-write guard: with HD_POISON=1 every device allocation of the
library starts as 0xFF bytes (NaN doubles, -1 ints). Every probe sequence and
run below must still match the oracle — any buffer consumed before it is
written turns the result into NaN or garbage."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def poison(monkeypatch):
    monkeypatch.setenv("HD_POISON", "1")


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


@pytest.mark.parametrize("ens,m,n,cap", [("ginibre", 3000, 5001, 4), ("ginibre", 700, 600, 64),
                                         ("haar", 0, 4099, 4), ("goe", 0, 2050, 3)])
def test_poisoned_probe_sequences(orc, lm, ens, m, n, cap):
    T, seed = 24, 17
    rng = np.random.default_rng(seed)
    if ens == "ginibre":
        sides = ["right" if rng.random() < 0.5 else "left" for _ in range(T)]
        ref = orc.Operator(ens, m=m, n=n, sigma=0.5, seed=seed)
        op = lm.GinibreOperator(m, n, 0.5, seed, draws="injected", capacity=cap)
        op.push_draws(orc.draws_for(seed, [m if s == "right" else n for s in sides]))
    elif ens == "haar":
        sides = ["right" if rng.random() < 0.5 else "left" for _ in range(T)]
        ref = orc.Operator(ens, n=n, seed=seed)
        op = lm.HaarOperator(n, seed=seed, draws="injected", capacity=cap)
        op.push_draws(orc.draws_for(seed, [n] * T))
    else:
        sides = ["right"] * T
        ref = orc.Operator(ens, n=n, sigma=0.5, seed=seed)
        op = lm.GOEOperator(n, seed, sigma=0.5, draws="injected", capacity=cap)
        op.push_draws(orc.draws_for(seed, [n] * (2 * T)))
    aux = orc.RandomSource(seed + 1)
    for t, s in enumerate(sides):
        x = aux.normal_vector((n if s == "right" else m) if ens == "ginibre" else n)
        got, want = op.probe(x, s), ref.probe(x, s)
        assert np.all(np.isfinite(got)), (t, s)
        assert rel(got, want) < 1e-10, (t, s, rel(got, want))


@pytest.mark.parametrize("ens", ["haar", "ginibre", "goe"])
def test_poisoned_runs(orc, lm, ens):
    n, T, seed = 3001, 20, 23
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    if ens == "haar":
        ref = orc.Operator(ens, n=n, seed=seed)
        want = ref.run("tanh_mix", "right", T, x1, keep=True)
        op = lm.HaarOperator(n, seed=seed, draws="injected", capacity=T)
        op.push_draws(orc.draws_for(seed, [n] * T))
        got = op.run(x1, T, update="tanh_mix", sides="right", keep_trajectory=True)
    elif ens == "ginibre":
        ref = orc.Operator(ens, m=n, n=n, sigma=n ** -0.5, seed=seed)
        want = ref.run("normalize", "alternate", T, x1, keep=True)
        op = lm.GinibreOperator(n, n, n ** -0.5, seed, draws="injected", capacity=T)
        op.push_draws(orc.draws_for(seed, [n] * T))
        got = op.run(x1, T, update="normalize", sides="alternate", keep_trajectory=True)
    else:
        ref = orc.Operator(ens, n=n, sigma=n ** -0.5, seed=seed)
        want = ref.run("normalize", "right", T, x1, keep=True)
        op = lm.GOEOperator(n, seed, sigma=n ** -0.5, draws="injected", capacity=T)
        op.push_draws(orc.draws_for(seed, [n] * (2 * T)))
        got = op.run(x1, T, update="normalize", sides="right", keep_trajectory=True)
    for t in range(T + 1):
        assert rel(got[t], want[t]) < 1e-9, (t, rel(got[t], want[t]))


@pytest.mark.parametrize("ens", ["ginibre", "goe", "haar"])
def test_poisoned_philox_deterministic(lm, ens):
    # two operators with the same seed, one grown from capacity 2, must agree bitwise
    import torch
    n, T = 20001, 16
    x1 = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    outs = []
    for cap in (T, 2):
        if ens == "ginibre":
            op = lm.GinibreOperator(n, n, n ** -0.5, 9, capacity=cap)
        elif ens == "goe":
            op = lm.GOEOperator(n, 9, sigma=n ** -0.5, capacity=cap)
        else:
            op = lm.HaarOperator(n, seed=9, capacity=cap)
        x, tr = x1.clone(), []
        for t in range(T):
            y = op.probe(x, "left" if (ens == "ginibre" and t % 2) else "right")
            tr.append(y.clone())
            x = y / y.norm()
        outs.append(torch.stack(tr))
    assert torch.isfinite(outs[0]).all()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("ens,m,n,cap", [("haar", 0, 2311, 3), ("ginibre", 1500, 2100, 2), ("ginibre", 900, 640, 40)])
def test_poisoned_complex_probe_sequences(orc, lm, ens, m, n, cap):
    # the fused complex sequences (csrc/hd_complex_fused.cuh, hd_complex_gin.cuh): partial
    # buffers, Gram matrices, speculative dots and panel growth under poisoned allocations
    T, seed = 30, 23
    rng = np.random.default_rng(seed)
    sides = ["right" if rng.random() < 0.6 else "left" for _ in range(T)]
    if ens == "haar":
        ref = orc.COperator("haar", n=n, seed=seed)
        op = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=cap)
        lens = [n] * T
    else:
        ref = orc.COperator("ginibre", m=m, n=n, sigma=0.8, seed=seed)
        op = lm.GinibreOperator(m, n, 0.8, seed, dtype="c128", draws="injected", capacity=cap)
        lens = [m if s == "right" else n for s in sides]
    op.push_draws(orc.complex_draws_for(seed, lens).view(np.complex128))
    aux = orc.RandomSource(seed + 1)
    for t, s in enumerate(sides):
        x = aux.normal_complex_vector(n if (s == "right" or ens == "haar") else m)
        got = op.probe(x, s)
        assert np.all(np.isfinite(got.view(np.float64))), t
        assert rel(got, ref.probe(x, s)) < 1e-10, (t, s)
