"""HD_DRAWS_REFERENCE: the device operator draws the reference's own
RandomSource(seed, stream) stream (xoshiro256++ + ziggurat), so an operator
built from the same arguments as the reference's (module.cpp:68-110:
GinibreOperator(m, n, sigma, seed) / HaarOperator(n, seed) with
RandomSource(seed)) is the same matrix: no draws are injected here, the
oracle operator is simply constructed with the same seed."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


@pytest.mark.parametrize("ens,m,n", [("haar", 0, 3001), ("haar", 0, 1), ("ginibre", 700, 901), ("ginibre", 1, 5),
                                     ("goe", 0, 513)])
def test_reference_mode_probe_sequence(orc, lm, ens, m, n):
    seed = 1234 + n
    T = min(n if ens != "ginibre" else min(m, n), 24)
    rng = np.random.default_rng(seed)
    sides = ["right" if (ens == "goe" or rng.random() < 0.5) else "left" for _ in range(T)]
    if ens == "haar":
        ref, op = orc.Operator("haar", n=n, seed=seed), lm.HaarOperator(n, seed=seed, draws="reference", capacity=4)
    elif ens == "ginibre":
        ref = orc.Operator("ginibre", m=m, n=n, sigma=0.7, seed=seed)
        op = lm.GinibreOperator(m, n, 0.7, seed, draws="reference", capacity=4)
    else:
        ref = orc.Operator("goe", n=n, sigma=1.0, seed=seed)
        op = lm.GOEOperator(n, seed, draws="reference", capacity=4)
    aux = orc.RandomSource(seed, 1)
    for t, s in enumerate(sides):
        x = aux.normal_vector(n if (s == "right" or ens != "ginibre") else m)
        got, want = op.probe(x, s), ref.probe(x, s)
        assert rel(got, want) < 1e-10, (t, s, rel(got, want))
    assert op.remaining_probes == ref.remaining_probes


def test_reference_mode_runs_match_reference_runs(orc, lm):
    # config 2 dynamics (tanh mix) and config 1 dynamics (normalize, alternating)
    n, T, seed = 5000, 25, 77
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    want = orc.Operator("haar", n=n, seed=seed).run("tanh_mix", "right", T, x1, keep=True)
    got = lm.HaarOperator(n, seed=seed, draws="reference").run(x1, T, update="tanh_mix", sides="right",
                                                               keep_trajectory=True)
    assert max(rel(got[t], want[t]) for t in range(T + 1)) < 1e-9
    n, T = 4096, 50
    x1 = orc.RandomSource(1, 1).normal_vector(n)
    want = orc.Operator("ginibre", m=n, n=n, sigma=n ** -0.5, seed=1).run("normalize", "alternate", T, x1, keep=True)
    got = lm.GinibreOperator(n, n, n ** -0.5, 1, draws="reference").run(x1, T, update="normalize",
                                                                        keep_trajectory=True)
    assert max(rel(got[t], want[t]) for t in range(T + 1)) < 1e-9


def test_reference_mode_reset_reseed_and_failed_probe(orc, lm):
    n = 300
    op = lm.HaarOperator(n, seed=5, draws="reference")
    x = orc.RandomSource(6).normal_vector(n)
    y1 = op.probe(x, "right")
    bad = x.copy()
    bad[3] = np.nan
    with pytest.raises(ValueError):
        op.probe(bad, "right")  # rejected before any draw is consumed (operators.hpp:44-48)
    y2 = op.probe(x, "left")
    ref = orc.Operator("haar", n=n, seed=5)
    assert rel(y1, ref.probe(x, "right")) < 1e-12
    assert rel(y2, ref.probe(x, "left")) < 1e-12
    op.reset()
    assert rel(op.probe(x, "right"), y1) < 1e-15
    op.reseed(99)
    assert rel(op.probe(x, "right"), orc.Operator("haar", n=n, seed=99).probe(x, "right")) < 1e-12


def test_reference_mode_device_inputs_and_exhaustion(orc, lm):
    import torch

    n = 64
    op = lm.HaarOperator(n, seed=3, draws="reference")
    ref = orc.Operator("haar", n=n, seed=3)
    aux = orc.RandomSource(4)
    for t in range(n):
        x = aux.normal_vector(n)
        got = op.probe(torch.from_numpy(x).cuda(), "right" if t % 2 else "left").cpu().numpy()
        assert rel(got, ref.probe(x, "right" if t % 2 else "left")) < 1e-10
    with pytest.raises(lm.BudgetExhausted):
        op.probe(np.ones(n), "right")
