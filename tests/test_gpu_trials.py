"""Batched independent trials (BASELINE config 3 orchestration): concurrent
device operators on their own streams, reseeded per trial (seed + b), replay
one captured run graph each. Every trial must equal the same trial run alone
(bitwise: the kernels are deterministic and trials share no state)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ensemble,sides,update", [("ginibre", "alternate", "normalize"),
                                                   ("haar", "right", "tanh_mix")])
def test_trials_equal_single_runs(lm, ensemble, sides, update):
    torch = pytest.importorskip("torch")
    B, n, T, seed = 7, 3000, 20, 40
    x1 = torch.randn((B, n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    out = lm.run_trials(ensemble, B, n, T, seed=seed, update=update, sides=sides, concurrency=3, x1=x1)
    for b in (0, 3, 6):
        op = (lm.GinibreOperator(n, n, n ** -0.5, seed + b, capacity=T) if ensemble == "ginibre"
              else lm.HaarOperator(n, seed + b, capacity=T))
        ref = op.run(x1[b].clone(), T, update=update, sides=sides)
        assert torch.equal(out[b], ref), b
    assert not torch.equal(out[0], out[1])


def test_trials_fp32_and_reseed_replay(lm):
    torch = pytest.importorskip("torch")
    B, n, T = 5, 2000, 16
    a = lm.run_trials("ginibre", B, n, T, seed=3, dtype="f32", concurrency=2)
    b = lm.run_trials("ginibre", B, n, T, seed=3, dtype="f32", concurrency=4)
    assert a.dtype == torch.float32
    assert torch.equal(a, b)  # concurrency does not change any result
    norms = a.double().norm(dim=1)
    assert torch.allclose(norms, torch.ones_like(norms), atol=1e-5)
