"""Two-pass Haar runs (csrc/hd_fused.cuh) through the C-ABI.

A Haar run with an elementwise update on a fresh operator streams each panel
once per probe (k_haar2p + k_small_2p). These tests pin it to the CPU oracle
(injected reference draws, every iterate), to the three-pass sequence
(HD_FUSED=0, same Philox matrix), and cover the precision fallback, the
continuation with ordinary probes, sides, dtypes, odd sizes and errors.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL64 = 1e-9
TOL32 = 1e-4


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def haar(lm, n, fused=True, **kw):
    old = os.environ.get("HD_FUSED")
    os.environ["HD_FUSED"] = "1" if fused else "0"
    try:
        return lm.HaarOperator(n, **kw)
    finally:
        if old is None:
            os.environ.pop("HD_FUSED")
        else:
            os.environ["HD_FUSED"] = old


def per_probe_launches(op, T):
    # a run's fixed launches (resets, the first probe's k_dots, the closing
    # stage) left out
    return (op.launch_count() - 5) / T


@pytest.mark.parametrize("n,T,update,sides", [(20000, 30, "tanh_mix", "right"), (4097, 40, "identity", "right"),
                                               (1001, 25, "tanh_mix", "left"), (257, 64, "identity", "left")])
def test_fused_run_matches_oracle_every_iterate(orc, lm, n, T, update, sides):
    seed = 11 + n
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    ref = orc.Operator("haar", n=n, seed=seed)
    want = ref.run(update, sides, T, x1, keep=True)
    op = haar(lm, n, seed=seed, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1, T, update=update, sides=sides, keep_trajectory=True)
    # the two-pass sequence ran (no fallback): stage + pass + trajectory copy per probe
    assert per_probe_launches(op, T) < 3.5
    for t in range(T + 1):
        assert rel(got[t], want[t]) < TOL64, (t, rel(got[t], want[t]))


def test_fused_run_reference_draws(orc, lm):
    n, T, seed = 3000, 20, 23
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    want = orc.Operator("haar", n=n, seed=seed).run("tanh_mix", "right", T, x1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="reference")
    got = op.run(x1, T, update="tanh_mix", sides="right")
    assert per_probe_launches(op, T) < 2.5
    assert rel(got, want) < TOL64


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
@pytest.mark.parametrize("n,T,update", [(65536, 100, "tanh_mix"), (3001, 50, "identity")])
def test_fused_equals_three_pass_philox(lm, dtype, tol, n, T, update):
    torch = pytest.importorskip("torch")
    tdt = torch.float64 if dtype == "f64" else torch.float32
    g = torch.Generator().manual_seed(n)
    x1 = torch.randn(n, generator=g, dtype=torch.float64)
    x1 = (x1 / x1.norm()).to(tdt).cuda()
    a = haar(lm, n, True, seed=5, dtype=dtype)
    b = haar(lm, n, False, seed=5, dtype=dtype)
    ya = a.run(x1, T, update=update, sides="right")
    yb = b.run(x1, T, update=update, sides="right")
    assert per_probe_launches(a, T) < 2.5 and per_probe_launches(b, T) > 4.5
    assert rel(ya.cpu(), yb.cpu()) < tol
    # the same run again (graph replay from the fresh state) is bitwise identical
    a.reset()
    yc = a.run(x1, T, update=update, sides="right", use_graph=True)
    a.reset()
    yd = a.run(x1, T, update=update, sides="right", use_graph=True)
    assert torch.equal(yc, yd)
    assert rel(yc.cpu(), ya.cpu()) < tol


def test_fused_fallback_reruns_three_pass(lm, monkeypatch):
    # an unsatisfiable guard forces the precision fallback at probe 1: the run
    # is redone from the fresh state through the three-pass sequence
    n, T = 5000, 20
    x1 = np.random.default_rng(1).standard_normal(n)
    b = haar(lm, n, False, seed=9)
    yb = b.run(x1, T, update="tanh_mix", sides="right")
    monkeypatch.setenv("HD_FUSED_GUARD", "2.0")
    a = haar(lm, n, True, seed=9)
    ya = a.run(x1, T, update="tanh_mix", sides="right")
    assert np.array_equal(ya, yb)
    assert a.launch_count() > b.launch_count()
    assert a.chain_sizes() == b.chain_sizes() and a.remaining_probes == b.remaining_probes


def test_fused_run_to_budget_falls_back_when_degenerate(orc, lm):
    # T = n: the last folds leave tails of a few rows; wherever the early norm
    # would lose precision the run falls back, and either way it matches
    n, seed = 96, 41
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    ref = orc.Operator("haar", n=n, seed=seed)
    want = ref.run("identity", "right", n, x1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="injected", capacity=8)
    op.push_draws(orc.draws_for(seed, [n] * n))
    got = op.run(x1, n, update="identity", sides="right")
    assert rel(got, want) < TOL64
    assert op.remaining_probes == 0


def test_fused_run_then_probes_continue(orc, lm):
    # state after a two-pass run (chains, T, Gram, D, speculative dots) serves
    # ordinary three-pass probes exactly like the reference operator
    n, T, seed = 2000, 15, 77
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    ref = orc.Operator("haar", n=n, seed=seed)
    want = ref.run("tanh_mix", "right", T, x1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="injected", capacity=T + 10)
    op.push_draws(orc.draws_for(seed, [n] * (T + 6)))
    got = op.run(x1, T, update="tanh_mix", sides="right")
    assert per_probe_launches(op, T) < 2.5
    assert rel(got, want) < TOL64
    aux = orc.RandomSource(seed + 2)
    for t, side in enumerate(["right", "right", "left", "right", "left", "left"]):
        x = aux.normal_vector(n)
        assert rel(op.probe(x, side), ref.probe(x, side)) < 1e-10, (t, side)
    assert op.chain_sizes() == ref.chain_sizes()


@pytest.mark.parametrize("rule", ["negative_at_zero", "zero_when_negative"])
def test_fused_sign_rules(orc, lm, rule):
    n, T, seed = 600, 12, 19
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    ref = orc.Operator("haar", n=n, seed=seed, sign_rule=rule)
    want = ref.run("identity", "right", T, x1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="injected", sign_rule=rule)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1, T, update="identity", sides="right")
    assert rel(got, want) < TOL64


def test_fused_rejects_nonfinite_x1_and_keeps_state(lm):
    n = 1000
    op = haar(lm, n, seed=3)
    x1 = np.ones(n)
    x1[7] = np.nan
    with pytest.raises(ValueError, match="non-finite input"):
        op.run(x1, 5, update="tanh_mix", sides="right")
    assert op.remaining_probes == n and op.chain_sizes() == (0, 0)
    y = op.run(np.ones(n), 5, update="tanh_mix", sides="right")
    assert np.all(np.isfinite(y))


def test_fused_async_run(lm):
    torch = pytest.importorskip("torch")
    n, T = 30000, 40
    x1 = torch.randn(n, dtype=torch.float64, device="cuda")
    a = haar(lm, n, True, seed=2)
    b = haar(lm, n, False, seed=2)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    a.run_async(x1, T, out, update="tanh_mix", sides="right")
    a.wait()
    yb = b.run(x1, T, update="tanh_mix", sides="right")
    assert rel(out.cpu(), yb.cpu()) < 1e-12


@pytest.mark.parametrize("cluster", ["1", "0"])
def test_fused_stage_variants_match(orc, lm, monkeypatch, cluster):
    # the stage on a 2-CTA cluster (default) and on one CTA (HD_2P_CLUSTER=0)
    # both match the oracle; the one-CTA variant stays covered
    monkeypatch.setenv("HD_2P_CLUSTER", cluster)
    n, T, seed = 12000, 40, 29
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    want = orc.Operator("haar", n=n, seed=seed).run("tanh_mix", "right", T, x1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1, T, update="tanh_mix", sides="right")
    assert per_probe_launches(op, T) < 2.5
    assert rel(got, want) < TOL64


@pytest.mark.parametrize("n,T,update", [(1, 1, "tanh_mix"), (2, 2, "identity"), (3, 3, "tanh_mix"), (255, 40, "tanh_mix"),
                                        (513, 60, "identity")])
def test_fused_tiny_and_ragged_shapes(orc, lm, n, T, update):
    seed = 101 + n
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    want = orc.Operator("haar", n=n, seed=seed).run(update, "right", T, x1, keep=True)
    op = haar(lm, n, seed=seed, draws="injected", capacity=4)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1, T, update=update, sides="right", keep_trajectory=True)
    for t in range(T + 1):
        assert rel(got[t], want[t]) < TOL64, (t, rel(got[t], want[t]))
    assert op.remaining_probes == n - T


@pytest.mark.parametrize("T", [300, 480])
def test_fused_long_run_crosses_tiles(orc, lm, T):
    # off beyond the first 256-row tile: the pivot tile moves, the stage's head
    # rows span several tiles, and the k x k state outgrows shared memory
    n, seed = 6000, 7
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    want = orc.Operator("haar", n=n, seed=seed).run("tanh_mix", "right", T, x1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="injected", capacity=16)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1, T, update="tanh_mix", sides="right")
    assert per_probe_launches(op, T) < 2.5
    assert rel(got, want) < TOL64


def test_fused_fp32_matches_oracle(orc, lm):
    n, T, seed = 8192, 50, 13
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    want = orc.Operator("haar", n=n, seed=seed).run("tanh_mix", "right", T, x1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="injected", dtype="f32", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1.astype(np.float32), T, update="tanh_mix", sides="right")
    assert per_probe_launches(op, T) < 2.5
    assert rel(got, want) < TOL32


def test_fused_graph_replays_across_reseeds(lm):
    torch = pytest.importorskip("torch")
    n, T = 50000, 30
    x1 = torch.randn(n, dtype=torch.float64, device="cuda")
    a = haar(lm, n, True, seed=1)
    outs = []
    for sd in (11, 12, 11):
        a.reseed(sd)
        outs.append(a.run(x1, T, update="tanh_mix", sides="right", use_graph=True).cpu())
    assert torch.equal(outs[0], outs[2]) and not torch.equal(outs[0], outs[1])
    b = haar(lm, n, False, seed=12)
    yb = b.run(x1, T, update="tanh_mix", sides="right").cpu()
    assert rel(outs[1], yb) < 1e-12


@pytest.mark.parametrize("T,sides", [(1, "right"), (2, "left"), (17, "right"), (40, "left")])
def test_fused_normalize_matches_oracle(orc, lm, T, sides):
    # normalize dynamics (bench.cpp:25-28): y_t and ||y_t||^2 from the pass, the
    # scaling by the next stage (x_{T+1} checked; trajectories take the
    # three-pass sequence for this map)
    n, seed = 5003, 57 + T
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    want = orc.Operator("haar", n=n, seed=seed).run("normalize", sides, T, x1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1, T, update="normalize", sides=sides)
    # two-pass: resets (at creation and at the run) + k_dots + 2 per probe + the
    # closing stage + k_small_norm + the final scaled copy
    assert op.launch_count() <= 2 * T + 10
    assert rel(got, want) < TOL64
    assert abs(np.linalg.norm(got) - 1.0) < 1e-12


def test_fused_normalize_equals_three_pass_philox(lm):
    torch = pytest.importorskip("torch")
    n, T = 65536, 100
    x1 = torch.randn(n, dtype=torch.float64, device="cuda")
    a = haar(lm, n, True, seed=8)
    b = haar(lm, n, False, seed=8)
    ya = a.run(x1, T, update="normalize", sides="right")
    yb = b.run(x1, T, update="normalize", sides="right")
    assert per_probe_launches(a, T) < 2.5 and per_probe_launches(b, T) > 4.5
    assert rel(ya.cpu(), yb.cpu()) < 1e-12


def test_fused_runs_match_dense_haar_in_law(lm):
    # production path (device Philox, two-pass runs) against a dense
    # simulation with Haar matrices (batched QR with sign correction): the law
    # of x_{T+1} under x_{t+1} = tanh(2 Q x_t) + 0.1 x_{t-1} from x_1 = e_1 (KS)
    torch = pytest.importorskip("torch")
    stats = pytest.importorskip("scipy.stats")
    n, T, trials = 6, 5, 3000
    x1 = np.zeros(n)
    x1[0] = 1.0
    op = haar(lm, n, True, seed=1, capacity=T)
    lazy = np.empty((trials, n))
    for b in range(trials):
        op.reseed(1000 + b)
        lazy[b] = op.run(x1, T, update="tanh_mix", sides="right")
    assert op.launch_count() < trials * (2 * T + 12)  # two-pass runs (no fallback storm)
    g = torch.Generator().manual_seed(5)
    G = torch.randn(trials, n, n, generator=g, dtype=torch.float64)
    Q, R = torch.linalg.qr(G)
    Q = Q * torch.sign(torch.diagonal(R, dim1=1, dim2=2))[:, None, :]
    x = torch.zeros(trials, n, dtype=torch.float64)
    x[:, 0] = 1.0
    xp = torch.zeros_like(x)
    for _ in range(T):
        y = torch.einsum("bij,bj->bi", Q, x)
        x, xp = torch.tanh(2.0 * y) + 0.1 * xp, x
    dense = x.numpy()
    alpha = 1e-3 / 3
    for name, a, d in [("coord0", lazy[:, 0], dense[:, 0]), ("coord_last", lazy[:, -1], dense[:, -1]),
                       ("sqnorm", (lazy ** 2).sum(1), (dense ** 2).sum(1))]:
        p = stats.ks_2samp(a, d).pvalue
        assert p > alpha, (name, p)


def test_fused_run_then_second_run_continues(orc, lm):
    # a second run on the same operator (no longer fresh) takes the three-pass
    # sequence from the two-pass run's end state; both match the oracle
    n, T1, T2, seed = 3000, 12, 9, 45
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    ref = orc.Operator("haar", n=n, seed=seed)
    w1 = ref.run("tanh_mix", "right", T1, x1, keep=False)[0]
    w2 = ref.run("normalize", "right", T2, w1, keep=False)[0]
    op = haar(lm, n, seed=seed, draws="injected", capacity=4)
    op.push_draws(orc.draws_for(seed, [n] * (T1 + T2)))
    g1 = op.run(x1, T1, update="tanh_mix", sides="right")
    assert rel(g1, w1) < TOL64
    before = op.launch_count()
    g2 = op.run(g1, T2, update="normalize", sides="right")
    assert op.launch_count() - before > 4 * T2  # three-pass sequence
    assert rel(g2, w2) < TOL64
    assert op.chain_sizes() == ref.chain_sizes()
