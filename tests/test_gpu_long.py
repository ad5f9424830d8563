"""Long chains and large n: parity with the oracle far past the usual test
depths (hundreds of reflectors per chain, including the spiked-GOE power
method of config 5), and bitwise determinism at large n across panel
capacities (growth paths) — the regime where a stream-ordering race once
showed up (tests/test_gpu_streams.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


def test_spiked_goe_300_steps(orc, lm):
    n, T, seed = 3000, 300, 31
    u = orc.RandomSource(seed, 1).normal_vector(n)
    u /= np.linalg.norm(u)
    x1 = orc.RandomSource(seed, 2).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    xr, ovr = orc.Operator("goe", n=n, sigma=n ** -0.5, seed=seed).spiked_power(u, x1, T)
    for cap in (T, 16):
        op = lm.GOEOperator(n, seed, sigma=n ** -0.5, draws="injected", capacity=cap)
        op.push_draws(orc.draws_for(seed, [n] * (2 * T)))
        x, ov = lm.spiked_power(op, u, x1, T)
        assert rel(x, xr) < 1e-9
        assert np.max(np.abs(ov - ovr)) < 1e-9


def test_haar_600_and_ginibre_600_probes(orc, lm):
    n, T = 2000, 600
    ref = orc.Operator("haar", n=n, seed=7)
    op = lm.HaarOperator(n, seed=7, draws="reference", capacity=T)
    aux = orc.RandomSource(8)
    for t in range(T):
        x = aux.normal_vector(n)
        s = "right" if t % 3 else "left"
        assert rel(op.probe(x, s), ref.probe(x, s)) < 1e-9, t
    m, n, T = 1500, 1200, 600
    ref = orc.Operator("ginibre", m=m, n=n, sigma=1.0, seed=9)
    op = lm.GinibreOperator(m, n, 1.0, 9, draws="reference", capacity=64)  # grows 64 -> 128 -> ...
    aux = orc.RandomSource(10)
    for t in range(T):
        s = "right" if t % 2 == 0 else "left"
        x = aux.normal_vector(n if s == "right" else m)
        assert rel(op.probe(x, s), ref.probe(x, s)) < 1e-9, t


@pytest.mark.parametrize("ens", ["haar", "goe", "ginibre"])
def test_large_n_bitwise_determinism_across_capacities(lm, ens):
    import torch

    N, steps = 4_000_000, 24
    g = torch.Generator("cuda").manual_seed(5)
    x1 = torch.randn(N, device="cuda", generator=g, dtype=torch.float64)
    x1 /= x1.norm()
    trajs = []
    for cap in (steps, 8):
        if ens == "haar":
            op = lm.HaarOperator(N, seed=5, capacity=cap)
        elif ens == "goe":
            op = lm.GOEOperator(N, 5, sigma=N ** -0.5, capacity=cap)
        else:
            op = lm.GinibreOperator(N, N, N ** -0.5, 5, capacity=cap)
        x, tr = x1.clone(), []
        for t in range(steps):
            y = op.probe(x, "left" if (ens == "ginibre" and t % 2) else "right")
            tr.append(y[::997].clone())  # a strided sample keeps the memory small
            x = y / y.norm()
        trajs.append(torch.stack(tr))
        del op
        torch.cuda.empty_cache()
    assert torch.equal(trajs[0], trajs[1])
