"""Row-sharded operators (north star: n beyond one GPU's HBM; SURVEY.md §8 e1;
DESIGN.md §7) as virtual shards on one GPU: k handles of one operator, each
driven from its own host thread, exchanging through the in-process exchange
(the NCCL exchange has the same contract across ranks). Each shard gets only
its rows of x and returns its rows of y; the stitched result must match the
unsharded oracle. Allocations are poisoned, so a head row the exchange
failed to deliver shows up as NaN."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def poison(monkeypatch):
    monkeypatch.setenv("HD_POISON", "1")


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


def make(lm, ens, m, n, seed, sigma, **kw):
    if ens == "haar":
        return lm.HaarOperator(n, seed=seed, **kw)
    if ens == "goe":
        return lm.GOEOperator(n, seed, sigma=sigma, **kw)
    return lm.GinibreOperator(m, n, sigma, seed, **kw)


def run_shards(lm, S, ens, m, n, seed, sigma, seq, draws=None, capacity=24, mode="injected", torch_io=False):
    """Drive S shard handles (one thread each) through the probe sequence
    seq = [(x_global, side)]; returns the stitched outputs."""
    ex = lm.Exchange.local(S)
    outs, errs = [None] * S, []

    def worker(r):
        try:
            op = make(lm, ens, m, n, seed, sigma, draws=mode, capacity=capacity, shard=(r, S), exchange=ex)
            if draws is not None:
                op.push_draws(draws)
            res = []
            for x, side in seq:
                lo, hi = op.shard_range("cols" if (side == "right" or ens == "goe") else "rows")
                xs = x[lo:hi]
                if torch_io:
                    import torch

                    xs = torch.from_numpy(np.ascontiguousarray(xs)).cuda()
                y = op.probe(xs, side)
                res.append(y.cpu().numpy() if torch_io else y)
            outs[r] = res
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(S)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0][1]
    return [np.concatenate([outs[r][t] for r in range(S)]) for t in range(len(seq))]


@pytest.mark.parametrize("ens,m,n,S", [("haar", 0, 3001, 2), ("haar", 0, 3001, 3), ("ginibre", 2100, 1500, 2),
                                       ("ginibre", 1300, 2900, 3), ("goe", 0, 1800, 2), ("haar", 0, 1800, 4)])
def test_sharded_probe_sequences_match_oracle(orc, lm, ens, m, n, S):
    seed, T = 40 + S, 20
    sigma = 0.8
    rng = np.random.default_rng(seed)
    sides = ["right" if (ens == "goe" or rng.random() < 0.5) else "left" for _ in range(T)]
    if ens == "ginibre":
        ref = orc.Operator("ginibre", m=m, n=n, sigma=sigma, seed=seed)
        draws = orc.draws_for(seed, [m if s == "right" else n for s in sides])
    elif ens == "haar":
        ref = orc.Operator("haar", n=n, seed=seed)
        draws = orc.draws_for(seed, [n] * T)
    else:
        ref = orc.Operator("goe", n=n, sigma=sigma, seed=seed)
        draws = orc.draws_for(seed, [n] * (2 * T))
    aux = orc.RandomSource(seed + 1)
    seq = [(aux.normal_vector(n if (s == "right" or ens != "ginibre") else m), s) for s in sides]
    got = run_shards(lm, S, ens, m, n, seed, sigma, seq, draws=draws)
    for t, (x, s) in enumerate(seq):
        want = ref.probe(x, s)
        assert np.all(np.isfinite(got[t])), t
        assert rel(got[t], want) < 1e-10, (t, s, rel(got[t], want))


@pytest.mark.parametrize("ens", ["haar", "ginibre", "goe"])
def test_sharded_philox_matches_unsharded(lm, orc, ens):
    # Philox draws are keyed by the global row: a sharded operator is the same
    # matrix as the unsharded one (sums differ only in reduction order)
    n, m, seed, T = 2600, 2600, 9, 16
    aux = orc.RandomSource(3)
    seq = [(aux.normal_vector(n), "right" if (t % 2 == 0 or ens != "ginibre") else "left") for t in range(T)]
    full = make(lm, ens, m, n, seed, n ** -0.5, capacity=T)
    want = [full.probe(x, s) for x, s in seq]
    got = run_shards(lm, 2, ens, m, n, seed, n ** -0.5, seq, mode="philox", capacity=T, torch_io=True)
    for t in range(T):
        assert rel(got[t], want[t]) < 1e-12, (t, rel(got[t], want[t]))
    again = run_shards(lm, 2, ens, m, n, seed, n ** -0.5, seq, mode="philox", capacity=T)
    assert all(np.array_equal(a, b) for a, b in zip(got, again))  # deterministic


def test_sharded_capacity_and_validation(lm):
    ex = lm.Exchange.local(2)
    with pytest.raises(ValueError, match="needs capacity"):
        lm.HaarOperator(2000, seed=1, shard=(0, 2), exchange=ex)
    with pytest.raises(ValueError, match="exchange size"):
        lm.HaarOperator(2000, seed=1, capacity=4, shard=(0, 3), exchange=ex)
    with pytest.raises(ValueError, match="shard 0 cannot hold"):
        lm.HaarOperator(600, seed=1, capacity=600, shard=(0, 2), exchange=ex)
    with pytest.raises(ValueError, match="too many shards"):
        lm.HaarOperator(1100, seed=1, capacity=4, shard=(0, 4), exchange=lm.Exchange.local(4))
    n, cap = 1500, 3
    seq = [(np.ones(n) / n, "right")] * (cap + 1)
    with pytest.raises(lm.ResourceCapExceeded, match="capacity"):
        run_shards(lm, 2, "haar", 0, n, 5, 1.0, seq, mode="philox", capacity=cap)
    op = lm.HaarOperator(n, seed=1, capacity=2, shard=(1, 2), exchange=ex)
    lo, hi = op.shard_range()
    assert (lo, hi) == lm.shard_plan(n, 2, 1, 256) and hi == n
    with pytest.raises(ValueError, match="input dimension"):
        op.probe(np.ones(n), "right")  # a shard takes its own rows only
    with pytest.raises(ValueError, match="sharded"):
        op.run(np.ones(hi - lo), 1)


@pytest.mark.parametrize("kind", ["nccl", "local"])
def test_one_shard_group_runs_the_exchange_path(orc, lm, kind):
    # a 1-rank NCCL communicator (or 1-shard local group) drives the full
    # sharded protocol — pack, allreduce, unpack after every streaming kernel
    # — on the single GPU; results equal the oracle (NCCL needs one GPU per
    # rank, so this is how the NCCL exchange is exercised on one device)
    ex = lm.Exchange.nccl(lm.Exchange.nccl_id(), 1, 0, 0) if kind == "nccl" else lm.Exchange.local(1)
    for ens, m, n in [("haar", 0, 2000), ("ginibre", 1500, 1100), ("goe", 0, 900)]:
        seed, T = 71, 12
        sides = ["right" if (ens != "ginibre" or t % 3) else "left" for t in range(T)]
        if ens == "ginibre":
            ref = orc.Operator(ens, m=m, n=n, sigma=0.9, seed=seed)
            op = lm.GinibreOperator(m, n, 0.9, seed, draws="injected", capacity=T, shard=(0, 1), exchange=ex)
            op.push_draws(orc.draws_for(seed, [m if s == "right" else n for s in sides]))
        elif ens == "haar":
            ref = orc.Operator(ens, n=n, seed=seed)
            op = lm.HaarOperator(n, seed=seed, draws="injected", capacity=T, shard=(0, 1), exchange=ex)
            op.push_draws(orc.draws_for(seed, [n] * T))
        else:
            ref = orc.Operator(ens, n=n, sigma=0.9, seed=seed)
            op = lm.GOEOperator(n, seed, sigma=0.9, draws="injected", capacity=T, shard=(0, 1), exchange=ex)
            op.push_draws(orc.draws_for(seed, [n] * (2 * T)))
        op.set_profiling(True)
        aux = orc.RandomSource(seed + 2)
        for s in sides:
            x = aux.normal_vector(m if (ens == "ginibre" and s == "left") else n)
            assert rel(op.probe(x, s), ref.probe(x, s)) < 1e-10
        # one exchange per streaming kernel whose results a single-CTA stage
        # needs (+ the final status exchange of Ginibre / GOE probes)
        per_probe = {"haar": 3, "ginibre": 4, "goe": 7}[ens]
        assert op.kernel_stats()["allreduce"]["launches"] == per_probe * T


@pytest.mark.parametrize("ens,kw", [("haar", {"skip_reflector": True}), ("ginibre", {"skip_reflector": True}),
                                    ("haar", {"sign_rule": "negative_at_zero"}), ("goe", {})])
def test_sharded_faults_and_reference_draws(orc, lm, ens, kw):
    # fault flags change which columns exist (skip_reflector drops the first
    # fold) and reference draws make every shard generate the reference's
    # stream: the stitched shards must still equal the oracle operator built
    # from the same seed, with no injected draws at all
    n, m, seed, T = 2600, 2100, 61, 14
    if ens == "ginibre":
        ref = orc.Operator("ginibre", m=m, n=n, sigma=0.9, seed=seed, **kw)
    elif ens == "haar":
        ref = orc.Operator("haar", n=n, seed=seed, **kw)
    else:
        ref = orc.Operator("goe", n=n, sigma=0.9, seed=seed)
    aux = orc.RandomSource(62)
    seq = [(aux.normal_vector(n if (t % 3 or ens != "ginibre") else m),
            "right" if (t % 3 or ens == "goe") else "left") for t in range(T)]
    want = [ref.probe(x, s) for x, s in seq]
    ex, outs, errs = lm.Exchange.local(2), [None, None], []

    def worker(r):
        try:
            op = make(lm, ens, m, n, seed, 0.9, draws="reference", capacity=T, shard=(r, 2), exchange=ex, **kw)
            res = []
            for x, s in seq:
                lo, hi = op.shard_range("cols" if (s == "right" or ens == "goe") else "rows")
                res.append(op.probe(np.ascontiguousarray(x[lo:hi]), s))
            outs[r] = res
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs
    for t in range(T):
        assert rel(np.concatenate([outs[0][t], outs[1][t]]), want[t]) < 1e-10, t


@pytest.mark.parametrize("two_pass", ["auto", "0"])
@pytest.mark.parametrize("S", [2, 3])
def test_sharded_spiked_power_run_matches_oracle(orc, lm, S, two_pass, monkeypatch):
    # config 5's workload row-sharded (virtual shards, one host thread each):
    # the GOE probes exchange their partial dots, the spike's <u, g> and ||g||^2
    # travel through the same exchange, every shard derives the same scalars;
    # fp64 runs take the two-pass kernels (one exchange per pass),
    # HD_GIN2P=0 the three-pass probes
    if two_pass == "0":
        monkeypatch.setenv("HD_GIN2P", "0")
    n, T, seed = 2400, 14, 71
    u = orc.RandomSource(seed, 1).normal_vector(n)
    u /= np.linalg.norm(u)
    x1 = orc.RandomSource(seed, 2).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    xr, ovr = orc.Operator("goe", n=n, sigma=n ** -0.5, seed=seed).spiked_power(u, x1, T)
    draws = orc.draws_for(seed, [n] * (2 * T))
    ex = lm.Exchange.local(S)
    outs, errs, kinds = [None] * S, [], [None] * S

    def worker(r):
        try:
            op = lm.GOEOperator(n, seed, sigma=n ** -0.5, draws="injected", capacity=T, shard=(r, S), exchange=ex)
            op.push_draws(draws)
            op.set_profiling(True)
            lo, hi = op.shard_range("cols")
            outs[r] = lm.spiked_power(op, u[lo:hi], x1[lo:hi], T)
            kinds[r] = set(op.kernel_stats())
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(S)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0][1]
    x = np.concatenate([outs[r][0] for r in range(S)])
    assert rel(x, xr) < 1e-9
    for r in range(S):
        assert np.max(np.abs(outs[r][1] - ovr)) < 1e-9
        assert ("gin2p" in kinds[r]) == (two_pass == "auto")
