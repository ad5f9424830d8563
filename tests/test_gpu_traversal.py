"""Stream order and L2 residency hints of the streaming kernels.

The fold pass streams its panel last-to-first (so it starts on the chunks the
k_dots pass just read, still in L2) and k_dots marks the end of its stream
evict-last. Neither may change results beyond the rounding of a reordered sum:
the L2 hints are bitwise-neutral, the reversed fold equals the forward one to
1e-12 and both match the oracle. HD_FOLD_FORWARD / HD_L2_KEEP_MB are read when
an operator is created."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


def _haar_run(orc, lm, n, T, seed):
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    op = lm.HaarOperator(n, seed=seed, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    return op.run(x1, T, update="tanh_mix", sides="right"), x1


def _ginibre_probes(orc, lm, m, n, T, seed):
    rng = np.random.default_rng(seed)
    sides = ["right" if rng.random() < 0.5 else "left" for _ in range(T)]
    op = lm.GinibreOperator(m, n, 0.5, seed, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [m if s == "right" else n for s in sides]))
    aux = orc.RandomSource(seed + 1)
    ys = []
    for s in sides:
        x = aux.normal_vector(n if s == "right" else m)
        ys.append(np.asarray(op.probe(x, s)))
    return np.concatenate(ys)


@pytest.mark.parametrize("n", [70001, 300000])
def test_haar_fold_order_and_l2_hints(orc, lm, monkeypatch, n):
    T, seed = 40, 23
    monkeypatch.setenv("HD_L2_KEEP_MB", "0")
    no_hint, x1 = _haar_run(orc, lm, n, T, seed)
    monkeypatch.setenv("HD_L2_KEEP_MB", "4")  # forces the evict-last path at this size
    hint, _ = _haar_run(orc, lm, n, T, seed)
    assert np.array_equal(hint, no_hint)
    monkeypatch.setenv("HD_FOLD_FORWARD", "1")
    fwd, _ = _haar_run(orc, lm, n, T, seed)
    assert rel(hint, fwd) < 1e-12
    want = orc.Operator("haar", n=n, seed=seed).run("tanh_mix", "right", T, x1, keep=False)[0]
    assert rel(hint, want) < 1e-9
    assert rel(fwd, want) < 1e-9


def test_ginibre_fold_order(orc, lm, monkeypatch):
    m, n, T, seed = 40000, 25003, 30, 29
    rev = _ginibre_probes(orc, lm, m, n, T, seed)
    monkeypatch.setenv("HD_FOLD_FORWARD", "1")
    fwd = _ginibre_probes(orc, lm, m, n, T, seed)
    assert rel(rev, fwd) < 1e-12
