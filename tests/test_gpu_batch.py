"""Batched independent trials (hd_batch_run / lazymat.batch_run, BASELINE
config 3): B operators run the same dynamics in lockstep, every kernel launch
issued once for all of them (gridDim.y = B) from one recorded, graph-captured
launch sequence. Each trial must equal the same operator run on its own: up
to the rounding of the re-associated GEMV-T partial sums (a batched launch
gives each trial 148/B SMs' worth of CTAs, so the warp -> tile split, and with
it the summation order, differs), and bitwise across repeated batched calls."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    import torch
    return float((a.double() - b.double()).norm() / b.double().norm())


def _single(lm, make, seed, x1, T, update, sides):
    op = make(seed)
    return op.run(x1, T, update=update, sides=sides)


@pytest.mark.parametrize("ens,n,T,update,sides,dtype,tol", [
    ("ginibre", 3000, 20, "normalize", "alternate", "f64", 1e-11),
    ("ginibre", 1100, 12, "identity", "right", "f64", 1e-11),
    ("haar", 20001, 15, "tanh_mix", "right", "f64", 1e-11),
    ("goe", 2050, 8, "normalize", "right", "f64", 1e-11),
    ("ginibre", 4000, 16, "normalize", "alternate", "f32", 2e-5),
])
def test_batched_trials_match_single_runs(lm, ens, n, T, update, sides, dtype, tol):
    import torch
    tdt = torch.float64 if dtype == "f64" else torch.float32
    make = {
        "ginibre": lambda s: lm.GinibreOperator(n, n, n ** -0.5, s, dtype=dtype, capacity=T),
        "haar": lambda s: lm.HaarOperator(n, s, dtype=dtype, capacity=T),
        "goe": lambda s: lm.GOEOperator(n, s, sigma=n ** -0.5, dtype=dtype, capacity=T),
    }[ens]
    B = 3
    g = torch.Generator("cuda").manual_seed(5)
    x1 = torch.randn((B, n), dtype=tdt, device="cuda", generator=g)
    x1 /= x1.norm(dim=1, keepdim=True)
    ops = [make(100 + b) for b in range(B)]
    out = torch.empty((B, n), dtype=tdt, device="cuda")
    for seeds in ([11, 12, 13], [21, 22, 23]):  # the second call replays the captured graph
        lm.batch_run(ops, x1, out, seeds, T, update, sides)
        torch.cuda.synchronize()
        for b in range(B):
            want = _single(lm, make, seeds[b], x1[b], T, update, sides)
            assert rel(out[b], torch.as_tensor(want, device="cuda")) < tol, (ens, seeds[b])
    again = torch.empty_like(out)
    lm.batch_run(ops, x1, again, [21, 22, 23], T, update, sides)
    torch.cuda.synchronize()
    assert torch.equal(out, again)


def test_run_trials_batched_matches_unbatched(lm):
    import torch
    n, T, trials = 5000, 16, 10
    ref = lm.run_trials("ginibre", trials, n, T, seed=3, concurrency=4)
    got = lm.run_trials("ginibre", trials, n, T, seed=3, concurrency=2, batch=4)  # 2 full chunks + tail of 2
    torch.cuda.synchronize()
    for b in range(trials):
        assert rel(got[b], ref[b]) < 1e-11


def test_batch_run_validation(lm):
    import torch
    n, T = 1000, 4
    a = lm.GinibreOperator(n, n, 0.1, 1, capacity=T)
    b = lm.GinibreOperator(n + 1, n + 1, 0.1, 2, capacity=T)
    x = torch.randn((2, n), dtype=torch.float64, device="cuda")
    o = torch.empty_like(x)
    with pytest.raises(Exception, match="share ensemble"):
        lm.batch_run([a, b], x, o, [1, 2], T)
    c = lm.GinibreOperator(n, n, 0.1, 3, capacity=T, draws="injected")
    with pytest.raises(Exception, match="Philox"):
        lm.batch_run([a, c], x, o, [1, 2], T)
    with pytest.raises(Exception, match="twice"):
        lm.batch_run([a, a], x, o, [1, 2], T)
