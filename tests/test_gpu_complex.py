"""Complex-field device operators (dtype "c128") against
the complex oracle (oracle/hd_oracle_complex.cpp), which restates the
reference's Scalar = complex<double> instantiation and is pinned by the
reference's complex tests (tests/test_oracle_complex.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("n", [1, 7, 300, 2049])
def test_complex_haar_sequence(orc, lm, n):
    seed, T = 50 + n, min(n, 20)
    rng = np.random.default_rng(seed)
    sides = ["right" if rng.random() < 0.6 else "left" for _ in range(T)]
    ref = orc.COperator("haar", n=n, seed=seed)
    op = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=4)
    op.push_draws(orc.complex_draws_for(seed, [n] * T).view(np.complex128))
    aux = orc.RandomSource(seed + 1)
    for t, s in enumerate(sides):
        x = aux.normal_complex_vector(n)
        got, want = op.probe(x, s), ref.probe(x, s)
        assert got.dtype == np.complex128
        assert rel(got, want) < 1e-10, (t, s, rel(got, want))
        assert abs(np.linalg.norm(got) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)  # unitary
    assert op.remaining_probes == ref.remaining_probes


@pytest.mark.parametrize("m,n", [(1, 1), (1, 3), (3, 1), (13, 10), (10, 13), (300, 257), (1000, 2100)])
def test_complex_ginibre_sequence(orc, lm, m, n):
    seed, T = 7 + m, min(m, n, 18)
    rng = np.random.default_rng(seed)
    sides = ["right" if rng.random() < 0.5 else "left" for _ in range(T)]
    ref = orc.COperator("ginibre", m=m, n=n, sigma=0.7, seed=seed)
    op = lm.GinibreOperator(m, n, 0.7, seed, dtype="c128", draws="injected", capacity=3)
    op.push_draws(orc.complex_draws_for(seed, [m if s == "right" else n for s in sides]).view(np.complex128))
    aux = orc.RandomSource(seed + 2)
    for t, s in enumerate(sides):
        x = aux.normal_complex_vector(n if s == "right" else m)
        got, want = op.probe(x, s), ref.probe(x, s)
        assert rel(got, want) < 1e-10, (t, s, rel(got, want))
    assert op.probe_counts() == (sides.count("right"), sides.count("left"))


def test_complex_goe_from_the_inner_ginibre(orc, lm):
    # GOEOperator over complex: (A x + A^H x) / sqrt(2) (ensembles.hpp:117-127)
    n, seed, T = 200, 3, 10
    inner = orc.COperator("ginibre", m=n, n=n, sigma=1.0, seed=seed)
    op = lm.GOEOperator(n, seed, dtype="c128", draws="injected", capacity=T)
    op.push_draws(orc.complex_draws_for(seed, [n] * (2 * T)).view(np.complex128))
    aux = orc.RandomSource(4)
    for _ in range(T):
        x = aux.normal_complex_vector(n)
        want = (inner.probe(x, "right") + inner.probe(x, "left")) * 0.7071067811865475244
        assert rel(op.probe(x, "right"), want) < 1e-10


def test_complex_reference_draws_need_no_injection(orc, lm):
    for ens, m, n in [("haar", 0, 500), ("ginibre", 400, 300)]:
        seed = 88
        if ens == "haar":
            ref, op = orc.COperator("haar", n=n, seed=seed), lm.HaarOperator(n, seed=seed, dtype="c128",
                                                                            draws="reference")
        else:
            ref = orc.COperator("ginibre", m=m, n=n, sigma=1.0, seed=seed)
            op = lm.GinibreOperator(m, n, 1.0, seed, dtype="c128", draws="reference")
        aux = orc.RandomSource(9)
        for t in range(12):
            s = "right" if t % 3 else "left"
            x = aux.normal_complex_vector(n if (s == "right" or ens == "haar") else m)
            assert rel(op.probe(x, s), ref.probe(x, s)) < 1e-10


def test_complex_reference_properties_philox(lm, orc):
    # test_haar.cpp:113-131 and test_ginibre.cpp:117-132 on the production draws
    q = lm.HaarOperator(12, seed=92, dtype="c128").reconstruct()
    assert np.max(np.abs(q.conj().T @ q - np.eye(12))) <= 1e-12
    op = lm.HaarOperator(9, seed=93, dtype="c128")
    aux = orc.RandomSource(94)
    x, w = aux.normal_complex_vector(9), aux.normal_complex_vector(9)
    qx = op.probe(x, "right")
    assert abs(np.linalg.norm(qx) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    assert abs(np.vdot(w, qx) - np.vdot(op.probe(w, "left"), x)) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(w)
    op = lm.GinibreOperator(13, 10, 1.0, 21, dtype="c128")
    x, w = aux.normal_complex_vector(10), aux.normal_complex_vector(13)
    lhs, rhs = np.vdot(w, op.probe(x, "right")), np.vdot(op.probe(w, "left"), x)
    assert abs(lhs - rhs) <= 1e-10 * (abs(lhs) + 1.0)
    op2 = lm.GinibreOperator(13, 10, 1.0, 23, dtype="c128")
    z1, z2 = op2.probe(x, "right"), op2.probe(x, "right")
    assert np.linalg.norm(z1 - z2) <= 1e-12 * np.linalg.norm(z1)


def test_complex_torch_io_and_errors(lm, orc):
    import torch

    n = 64
    op = lm.HaarOperator(n, seed=5, dtype="c128", capacity=8)
    ref = lm.HaarOperator(n, seed=5, dtype="c128", capacity=8)
    x = orc.RandomSource(6).normal_complex_vector(n)
    y = op.probe(torch.from_numpy(x).cuda(), "right")
    assert y.dtype == torch.complex128 and y.is_cuda
    assert np.linalg.norm(y.cpu().numpy() - ref.probe(x, "right")) <= 1e-12 * np.linalg.norm(x)
    bad = x.copy()
    bad[3] = complex(np.nan, 0)
    with pytest.raises(ValueError, match="non-finite"):
        op.probe(bad, "right")
    with pytest.raises(ValueError, match="non-finite"):
        op.probe(torch.from_numpy(bad).cuda(), "right")
    with pytest.raises(ValueError, match="dimension mismatch"):
        op.probe(np.ones(n + 1, complex), "right")
    with pytest.raises(ValueError, match="complex operators"):
        op.run(x, 2)
    small = lm.HaarOperator(3, seed=1, dtype="c128")
    for _ in range(3):
        small.probe(np.ones(3, complex), "right")
    with pytest.raises(lm.BudgetExhausted):
        small.probe(np.ones(3, complex), "right")
    small.reset()
    assert small.remaining_probes == 3


def test_complex_user_dynamics(orc, lm):
    # run_dynamics over a complex operator (dynamics.hpp is generic in Scalar):
    # normalised alternating power iteration on a complex Ginibre matrix,
    # against the complex oracle driven the same way
    import torch

    m, n, T, seed = 600, 500, 12, 17
    ref = orc.COperator("ginibre", m=m, n=n, sigma=m ** -0.5, seed=seed)
    x = orc.RandomSource(seed, 1).normal_complex_vector(n)
    want = [x]
    for t in range(1, T + 1):
        y = ref.probe(want[-1], "right" if t % 2 else "left")
        want.append(y / np.linalg.norm(y))
    op = lm.GinibreOperator(m, n, m ** -0.5, seed, dtype="c128", draws="reference")
    spec = lm.DynamicsSpec(T, 0, [torch.from_numpy(x).cuda()], lambda t: "right" if t % 2 else "left",
                           lambda t, y, h: y / torch.linalg.vector_norm(y))
    traj = lm.run_dynamics(op, spec)
    for t in range(T + 1):
        assert rel(traj[t].cpu().numpy(), want[t]) < 1e-9, t


# ---- fused Haar probe (csrc/hd_complex_fused.cuh): four panel passes, the fold
# member's Gram column from the k x k Gram matrix and the t x k head corner
@pytest.mark.parametrize("n,T,cap", [(5000, 120, 4), (1300, 200, 64)])
def test_complex_haar_long_chain_vs_oracle(orc, lm, n, T, cap):
    # long chains, capacity doubling on the way (W, T, G and D grow), mixed sides
    seed = 11 + n
    rng = np.random.default_rng(seed)
    ref = orc.COperator("haar", n=n, seed=seed)
    op = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=cap)
    op.push_draws(orc.complex_draws_for(seed, [n] * T).view(np.complex128))
    aux = orc.RandomSource(seed + 1)
    x = aux.normal_complex_vector(n)
    x /= np.linalg.norm(x)
    worst = 0.0
    for t in range(T):
        s = "right" if rng.random() < 0.7 else "left"
        got, want = op.probe(x, s), ref.probe(x, s)
        worst = max(worst, rel(got, want))
        # the iterate plus a fresh component: Q^H (Q x) alone would fold onto an exactly
        # zero tail (a reflector built from rounding noise, in the reference too)
        x = want / np.linalg.norm(want) + 0.5 * aux.normal_complex_vector(n) / np.sqrt(n)
    assert worst < 1e-10, worst


@pytest.mark.parametrize("skip", [False, True])
def test_complex_haar_fused_matches_generic_sequence(orc, lm, monkeypatch, skip):
    n, T, seed = 3001, 40, 23
    draws = orc.complex_draws_for(seed, [n] * T).view(np.complex128)
    ref = orc.COperator("haar", n=n, seed=seed, skip_reflector=skip)
    ops = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("HD_CX_FUSED", flag)  # read at hd_create
        ops[flag] = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=T, skip_reflector=skip)
        ops[flag].push_draws(draws)
    aux = orc.RandomSource(seed + 1)
    x = aux.normal_complex_vector(n)
    for t in range(T):
        s = "left" if t % 5 == 3 else "right"
        a, b, want = ops["1"].probe(x, s), ops["0"].probe(x, s), ref.probe(x, s)
        assert rel(a, b) < 1e-11, (t, rel(a, b))
        assert rel(a, want) < 1e-10, (t, rel(a, want))
        x = want / np.linalg.norm(want) + 0.5 * aux.normal_complex_vector(n) / np.sqrt(n)
    assert ops["1"].launch_count() < ops["0"].launch_count() / 2


def test_complex_haar_fused_reset_and_budget_edge(orc, lm):
    # every probe of the budget (the last tail has one row), then a reset run
    n, seed = 37, 5
    op = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=2)
    for rep in range(2):
        ref = orc.COperator("haar", n=n, seed=seed)
        op.push_draws(orc.complex_draws_for(seed, [n] * n).view(np.complex128))
        aux = orc.RandomSource(seed + rep)
        for t in range(n):
            x = aux.normal_complex_vector(n)
            s = "right" if t % 2 else "left"
            assert rel(op.probe(x, s), ref.probe(x, s)) < 1e-10, (rep, t)
        with pytest.raises(lm.BudgetExhausted):
            op.probe(x, "right")
        op.reset()


def test_complex_haar_flagged_device_input_leaves_the_operator_untouched(orc, lm):
    # device inputs are validated by a device flag the state-changing kernels test; a
    # rejected probe must not advance the operator (operators.hpp:44-48)
    import torch

    n, seed, T = 700, 31, 9
    draws = orc.complex_draws_for(seed, [n] * T).view(np.complex128)
    ref = orc.COperator("haar", n=n, seed=seed)
    op = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=4)
    op.push_draws(draws)
    aux = orc.RandomSource(seed + 1)
    for t in range(T):
        x = aux.normal_complex_vector(n)
        if t in (0, 4, 5):
            bad = x.copy()
            bad[(7 * t) % n] = complex(0.0, np.inf)
            before = op.remaining_probes
            with pytest.raises(ValueError, match="non-finite"):
                op.probe(torch.from_numpy(bad).cuda(), "right")
            assert op.remaining_probes == before
        s = "left" if t % 3 == 1 else "right"
        got = op.probe(torch.from_numpy(x).cuda(), s).cpu().numpy()
        assert rel(got, ref.probe(x, s)) < 1e-10, t


def test_complex_haar_two_rows_per_thread_variant(orc, lm, monkeypatch):
    monkeypatch.setenv("HD_CX_NROWS", "2")
    n, seed, T = 2500, 41, 24
    ref = orc.COperator("haar", n=n, seed=seed)
    op = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=T)
    op.push_draws(orc.complex_draws_for(seed, [n] * T).view(np.complex128))
    aux = orc.RandomSource(seed + 1)
    for t in range(T):
        x = aux.normal_complex_vector(n)
        s = "left" if t % 4 == 2 else "right"
        assert rel(op.probe(x, s), ref.probe(x, s)) < 1e-10, t


# ---- fused Ginibre / GOE probes (csrc/hd_complex_gin.cuh)
@pytest.mark.parametrize("m,n,T,cap", [(2600, 1900, 90, 3), (1500, 3100, 120, 200)])
def test_complex_ginibre_long_run_vs_oracle(orc, lm, m, n, T, cap):
    seed = 3 + m
    rng = np.random.default_rng(seed)
    sides = ["right" if rng.random() < 0.55 else "left" for _ in range(T)]
    ref = orc.COperator("ginibre", m=m, n=n, sigma=0.9 / np.sqrt(m), seed=seed)
    op = lm.GinibreOperator(m, n, 0.9 / np.sqrt(m), seed, dtype="c128", draws="injected", capacity=cap)
    op.push_draws(orc.complex_draws_for(seed, [m if s == "right" else n for s in sides]).view(np.complex128))
    aux = orc.RandomSource(seed + 2)
    worst = 0.0
    for t, s in enumerate(sides):
        x = aux.normal_complex_vector(n if s == "right" else m)
        worst = max(worst, rel(op.probe(x, s), ref.probe(x, s)))
    assert worst < 1e-10, worst
    assert op.probe_counts() == (sides.count("right"), sides.count("left"))


@pytest.mark.parametrize("skip", [False, True])
def test_complex_ginibre_fused_matches_generic_sequence(orc, lm, monkeypatch, skip):
    m, n, T, seed = 1100, 900, 30, 19
    sides = ["left" if t % 3 == 1 else "right" for t in range(T)]
    draws = orc.complex_draws_for(seed, [m if s == "right" else n for s in sides]).view(np.complex128)
    ref = orc.COperator("ginibre", m=m, n=n, sigma=1.0, seed=seed, skip_reflector=skip)
    ops = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("HD_CX_FUSED", flag)  # read at hd_create
        ops[flag] = lm.GinibreOperator(m, n, 1.0, seed, dtype="c128", draws="injected", capacity=8,
                                       skip_reflector=skip)
        ops[flag].push_draws(draws)
    aux = orc.RandomSource(seed + 1)
    for t, s in enumerate(sides):
        x = aux.normal_complex_vector(n if s == "right" else m)
        a, b, want = ops["1"].probe(x, s), ops["0"].probe(x, s), ref.probe(x, s)
        assert rel(a, b) < 1e-11, (t, rel(a, b))
        assert rel(a, want) < 1e-10, (t, rel(a, want))
    assert ops["1"].launch_count() < ops["0"].launch_count() / 3


def test_complex_goe_device_inputs_and_flagged_probe(orc, lm):
    import torch

    n, seed, T = 500, 13, 14
    inner = orc.COperator("ginibre", m=n, n=n, sigma=1.0, seed=seed)
    op = lm.GOEOperator(n, seed, dtype="c128", draws="injected", capacity=4)
    op.push_draws(orc.complex_draws_for(seed, [n] * (2 * T)).view(np.complex128))
    aux = orc.RandomSource(4)
    for t in range(T):
        x = aux.normal_complex_vector(n)
        if t in (0, 6):
            bad = x.copy()
            bad[t] = complex(np.nan, 1.0)
            with pytest.raises(ValueError, match="non-finite"):
                op.probe(torch.from_numpy(bad).cuda(), "right")
        want = (inner.probe(x, "right") + inner.probe(x, "left")) * 0.7071067811865475244
        got = op.probe(torch.from_numpy(x).cuda(), "right").cpu().numpy()
        assert rel(got, want) < 1e-10, t


def test_complex_fused_large_n_properties(lm, monkeypatch):
    # size-independent properties at a size the oracle does not reach (n = 2^20 + 77 rows:
    # ragged last row block; device Philox draws; device tensors in and out)
    import torch

    n, T = (1 << 20) + 77, 10
    gen = torch.Generator(device="cuda").manual_seed(5)
    rnd = lambda k: torch.complex(torch.randn(k, dtype=torch.float64, device="cuda", generator=gen),  # noqa: E731
                                  torch.randn(k, dtype=torch.float64, device="cuda", generator=gen))
    haar = lm.HaarOperator(n, seed=9, dtype="c128", capacity=2 * T + 2)
    monkeypatch.setenv("HD_CX_FUSED", "0")
    generic = lm.HaarOperator(n, seed=9, dtype="c128", capacity=2 * T + 2)
    monkeypatch.delenv("HD_CX_FUSED")
    for t in range(T):
        x, w = rnd(n), rnd(n)
        s = "left" if t % 3 == 2 else "right"
        opp = "left" if s == "right" else "right"
        y = haar.probe(x, s)
        assert abs(float(y.norm() / x.norm()) - 1.0) < 1e-12  # unitary
        assert float((y - generic.probe(x, s)).norm() / y.norm()) < 1e-12
        z = haar.probe(w, opp)  # the same lazily sampled Q from the other side
        assert float((z - generic.probe(w, opp)).norm() / z.norm()) < 1e-12
        lhs, rhs = torch.vdot(w, y), torch.vdot(z, x)
        assert abs(complex(lhs - rhs)) < 1e-10 * float(x.norm() * w.norm())
    m2, n2 = 700_001, 400_003
    gin = lm.GinibreOperator(m2, n2, m2 ** -0.5, 3, dtype="c128", capacity=2 * T)
    monkeypatch.setenv("HD_CX_FUSED", "0")
    gin0 = lm.GinibreOperator(m2, n2, m2 ** -0.5, 3, dtype="c128", capacity=2 * T)
    monkeypatch.delenv("HD_CX_FUSED")
    for t in range(T):
        x, w = rnd(n2), rnd(m2)
        y = gin.probe(x, "right")
        assert float((y - gin0.probe(x, "right")).norm() / y.norm()) < 1e-12
        z = gin.probe(w, "left")
        assert float((z - gin0.probe(w, "left")).norm() / z.norm()) < 1e-12
        lhs, rhs = torch.vdot(w, y), torch.vdot(z, x)  # the same lazily sampled matrix from both sides
        assert abs(complex(lhs - rhs)) < 1e-10 * (abs(complex(lhs)) + float(x.norm() * w.norm()) * m2 ** -0.5)
    # a repeated probe answers from the same matrix (last: its fold tail is rounding noise, so the
    # reflector it appends is implementation-specific, in the reference too)
    y2 = gin.probe(x, "right")
    assert float((y2 - y).norm() / y.norm()) < 1e-11


def test_complex_haar_speculative_draw_dots(orc, lm, monkeypatch):
    # the last pass of a fused Haar probe takes the next draw's dots (three panel passes per
    # probe when the side repeats): with the draws queued ahead, one at a time (no
    # speculation possible), and with HD_CX_SPEC=0 — all against the oracle
    n, T, seed = 2600, 36, 77
    draws = orc.complex_draws_for(seed, [n] * T).view(np.complex128).reshape(T, n)
    sides = ["left" if t % 7 in (3, 4) else "right" for t in range(T)]
    ref = orc.COperator("haar", n=n, seed=seed)
    ahead = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=6)
    ahead.push_draws(draws.reshape(-1))
    single = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=6)
    monkeypatch.setenv("HD_CX_SPEC", "0")
    off = lm.HaarOperator(n, seed=seed, dtype="c128", draws="injected", capacity=6)
    off.push_draws(draws.reshape(-1))
    aux = orc.RandomSource(seed + 1)
    for t, s in enumerate(sides):
        x = aux.normal_complex_vector(n)
        single.push_draws(draws[t])
        want = ref.probe(x, s)
        for name, op in (("ahead", ahead), ("single", single), ("off", off)):
            assert rel(op.probe(x, s), want) < 1e-10, (name, t)
    # the speculative pass replaces the draw's GEMV-T job: fewer algorithmic bytes
    ahead.set_profiling(True)
    off.set_profiling(True)
    ahead.reset(), off.reset()
    for op in (ahead, off):
        op.push_draws(draws.reshape(-1))
        for t in range(T):
            op.probe(aux.normal_complex_vector(n), "right")
    b = lambda op: sum(v["alg_bytes"] for v in op.kernel_stats().values())  # noqa: E731
    assert b(ahead) < 0.85 * b(off)


@pytest.mark.parametrize("ens", ["haar", "ginibre", "goe"])
def test_complex_philox_rejected_probe_does_not_shift_the_stream(lm, ens):
    # production draws: a rejected device input must leave counters, the early-drawn next
    # draw and its speculative dots as they were — the twin that never saw it stays identical
    import torch

    n, T = 3000, 12
    mk = {"haar": lambda: lm.HaarOperator(n, seed=5, dtype="c128", capacity=4),
          "ginibre": lambda: lm.GinibreOperator(n + 100, n, 0.03, 5, dtype="c128", capacity=4),
          "goe": lambda: lm.GOEOperator(n, 5, dtype="c128", capacity=4)}[ens]
    a, b = mk(), mk()
    gen = torch.Generator(device="cuda").manual_seed(1)
    for t in range(T):
        side = "left" if (ens != "goe" and t % 4 == 1) else "right"
        k = n + 100 if (ens == "ginibre" and side == "left") else n
        x = torch.complex(torch.randn(k, dtype=torch.float64, device="cuda", generator=gen),
                          torch.randn(k, dtype=torch.float64, device="cuda", generator=gen))
        if t in (0, 5, 6):
            bad = x.clone()
            bad[t * 3] = complex(float("inf"), 0.0)
            with pytest.raises(ValueError, match="non-finite"):
                a.probe(bad, side)
        ya, yb = a.probe(x, side), b.probe(x, side)
        assert float((ya - yb).norm() / yb.norm()) < 1e-14, (ens, t)
    assert a.remaining_probes == b.remaining_probes
