"""Parity of the B200 path (through the C-ABI) against the CPU oracle.

The oracle restates the reference (oracle/hd_oracle.cpp) and both sides
consume identical Gaussian draws: the device operator runs in injected-draw
mode fed with RandomSource(seed).normals(len) per probe — the exact sequence
the reference operator draws (ginibre.hpp:67,86; haar.hpp:48).

Tolerances (north_star): every iterate within 1e-9 relative (fp64), 1e-4
(fp32). Individual probes of well-conditioned inputs are checked at 1e-10.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL64 = 1e-9
TOL32 = 1e-4


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a, dtype=np.float64) - b) / (nb if nb > 0 else 1.0)


def draw_lengths_ginibre(m, n, sides):
    return [m if s == "right" else n for s in sides]


# ------------------------------------------------------------------- Haar
def test_haar_first_probe_closed_form(orc, lm):
    # test_haar.cpp:35-45: first probe = (||x|| / ||g||) g
    n = 10
    op = lm.HaarOperator(n, seed=71, draws="injected")
    g = orc.RandomSource(71).normal_vector(n)
    op.push_draws(g)
    x = orc.RandomSource(72).normal_vector(n)
    y = op.probe(x, "right")
    expect = (np.linalg.norm(x) / np.linalg.norm(g)) * g
    assert np.linalg.norm(y - expect) <= 1e-12 * np.linalg.norm(x)


@pytest.mark.parametrize("n", [1, 2, 10, 257, 4096, 70001])
def test_haar_probe_sequence(orc, lm, n):
    seed = 81 + n
    T = min(n, 24)
    sides = ["left" if t % 3 == 0 else "right" for t in range(T)]
    ref = orc.Operator("haar", n=n, seed=seed)
    op = lm.HaarOperator(n, seed=seed, draws="injected", capacity=8)
    op.push_draws(orc.draws_for(seed, [n] * T))
    aux = orc.RandomSource(seed + 1)
    for t, s in enumerate(sides):
        x = aux.normal_vector(n)
        want = ref.probe(x, s)
        got = op.probe(x, s)
        assert rel(got, want) < 1e-10, (t, s, rel(got, want))
        # every probe preserves norms (test_haar.cpp:47-56)
        assert abs(np.linalg.norm(got) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    assert op.remaining_probes == ref.remaining_probes
    assert op.chain_sizes() == ref.chain_sizes()


def test_haar_run_tanh_mix(orc, lm):
    # BASELINE config 2 dynamics at reduced n: x_{t+1} = tanh(2 Q x_t) + 0.1 x_{t-1}
    n, T, seed = 20000, 30, 5
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    ref = orc.Operator("haar", n=n, seed=seed)
    want = ref.run("tanh_mix", "right", T, x1, keep=True)
    op = lm.HaarOperator(n, seed=seed, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1, T, update="tanh_mix", sides="right", keep_trajectory=True)
    for t in range(T + 1):
        assert rel(got[t], want[t]) < TOL64, (t, rel(got[t], want[t]))


def test_haar_reconstruct_orthogonal(lm):
    op = lm.HaarOperator(16, seed=91)
    q = op.reconstruct()
    assert np.max(np.abs(q.T @ q - np.eye(16))) <= 1e-12
    assert op.remaining_probes == 0
    with pytest.raises(ValueError):
        op.reconstruct()


def test_haar_reconstruct_column0_reference_draw(orc, lm):
    # test_haar.cpp:98-111: column 0 is g/||g|| of the seed's first draw
    n = 16
    op = lm.HaarOperator(n, seed=91, draws="injected")
    op.push_draws(orc.draws_for(91, [n] * n))
    q = op.reconstruct()
    g = orc.RandomSource(91).normal_vector(n)
    assert np.linalg.norm(q[:, 0] - g / np.linalg.norm(g)) <= 1e-12
    ref = orc.Operator("haar", n=n, seed=91)
    qr = np.stack([ref.probe(np.eye(n)[j], "right") for j in range(n)], axis=1)
    assert np.max(np.abs(q - qr)) < 1e-12


# ---------------------------------------------------------------- Ginibre
def test_ginibre_first_probes_closed_form(orc, lm):
    # test_ginibre.cpp:56-77
    m, n, sigma = 12, 7, 0.75
    op = lm.GinibreOperator(m, n, sigma=sigma, seed=99, draws="injected")
    op.push_draws(orc.RandomSource(99).normal_vector(m))
    x = np.array([1, -2, 0.5, 3, 0, 1, -1.0])
    y = op.probe(x, "right")
    g = orc.RandomSource(99).normal_vector(m)
    assert np.linalg.norm(y - sigma * np.linalg.norm(x) * g) <= 1e-12 * np.linalg.norm(y)

    m, n = 9, 6
    op = lm.GinibreOperator(m, n, sigma=1.0, seed=100, draws="injected")
    op.push_draws(orc.RandomSource(100).normal_vector(n))
    w = np.ones(m)
    y = op.probe(w, "left")
    g = orc.RandomSource(100).normal_vector(n)
    assert y.shape == (n,)
    assert np.linalg.norm(y - np.linalg.norm(w) * g) <= 1e-12 * np.linalg.norm(y)


@pytest.mark.parametrize("m,n", [(1, 1), (12, 7), (20, 16), (6, 9), (300, 257), (4096, 4096), (3000, 50001)])
def test_ginibre_probe_sequence(orc, lm, m, n):
    seed = 5 + m + n
    T = min(m, n, 20)
    rng = np.random.default_rng(seed)
    sides = [("right" if rng.random() < 0.55 else "left") for _ in range(T)]
    ref = orc.Operator("ginibre", m=m, n=n, sigma=1.3, seed=seed)
    op = lm.GinibreOperator(m, n, sigma=1.3, seed=seed, draws="injected", capacity=4)
    op.push_draws(orc.draws_for(seed, draw_lengths_ginibre(m, n, sides)))
    aux = orc.RandomSource(seed + 7)
    for t, s in enumerate(sides):
        x = aux.normal_vector(n if s == "right" else m)
        want = ref.probe(x, s)
        got = op.probe(x, s)
        assert rel(got, want) < 1e-10, (t, s, rel(got, want))
    assert op.probe_counts() == ref.counts()
    assert op.chain_sizes() == ref.chain_sizes()
    assert op.remaining_probes == ref.remaining_probes


def test_ginibre_repeat_and_adjoint(orc, lm):
    # test_ginibre.cpp:79-115 on the device path (philox draws)
    op = lm.GinibreOperator(20, 16, 1.0, seed=5)
    aux = orc.RandomSource(6)
    x = aux.normal_vector(16)
    y1 = op.probe(x, "right")
    y2 = op.probe(x, "right")
    assert np.linalg.norm(y1 - y2) <= 1e-12 * np.linalg.norm(y1)
    w = aux.normal_vector(20)
    op.probe(w, "left")
    y3 = op.probe(x, "right")
    assert np.linalg.norm(y1 - y3) <= 1e-11 * np.linalg.norm(y1)

    op = lm.GinibreOperator(15, 11, 0.9, seed=12)
    aux = orc.RandomSource(13)
    x, w = aux.normal_vector(11), aux.normal_vector(15)
    ax, atw = op.probe(x, "right"), op.probe(w, "left")
    assert abs(w @ ax - atw @ x) <= 1e-10 * (abs(w @ ax) + 1.0)

    op = lm.GinibreOperator(24, 18, 1.3, seed=8)
    aux = orc.RandomSource(9)
    x1, x2 = aux.normal_vector(18), aux.normal_vector(18)
    y1, y2 = op.probe(x1, "right"), op.probe(x2, "right")
    y3 = op.probe(2.0 * x1 - 0.5 * x2, "right")
    assert np.linalg.norm(y3 - (2.0 * y1 - 0.5 * y2)) <= 1e-10 * (np.linalg.norm(y1) + np.linalg.norm(y2))


def test_ginibre_sigma_scales_exactly(orc, lm):
    # test_ginibre.cpp:134-144 — sigma applied last, bitwise
    a = lm.GinibreOperator(10, 10, 1.0, seed=31)
    b = lm.GinibreOperator(10, 10, 2.5, seed=31)
    aux = orc.RandomSource(32)
    for _ in range(3):
        x = aux.normal_vector(10)
        ya, yb = a.probe(x, "right"), b.probe(x, "right")
        assert np.array_equal(yb, 2.5 * ya)


def test_zero_vector_probes_to_zero(lm):
    op = lm.GinibreOperator(6, 6, 1.0, seed=41)
    assert np.linalg.norm(op.probe(np.zeros(6), "right")) == 0.0
    assert op.remaining_probes == 5
    h = lm.HaarOperator(5, seed=89)
    assert np.linalg.norm(h.probe(np.zeros(5), "right")) == 0.0
    assert h.remaining_probes == 4


def test_ginibre_run_config1(orc, lm):
    # BASELINE config 1: m = n = 4096, sigma = 1/sqrt(n), T = 50, alternating,
    # x_{t+1} = y / ||y||, x_1 ~ N(0, I) from the data stream; every iterate.
    n, T, seed = 4096, 50, 1
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    ref = orc.Operator("ginibre", m=n, n=n, sigma=1 / np.sqrt(n), seed=seed)
    want = ref.run("normalize", "alternate", T, x1, keep=True)
    op = lm.GinibreOperator(n, n, sigma=1 / np.sqrt(n), seed=seed, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1, T, update="normalize", sides="alternate", keep_trajectory=True)
    errs = [rel(got[t], want[t]) for t in range(T + 1)]
    assert max(errs) < TOL64, max(errs)


# -------------------------------------------------------------------- GOE
def test_goe_probe_and_run(orc, lm):
    n, seed = 600, 321
    ref = orc.Operator("goe", n=n, sigma=1 / np.sqrt(n), seed=seed)
    op = lm.GOEOperator(n, seed=seed, sigma=1 / np.sqrt(n), draws="injected", capacity=10)
    T = 10
    op.push_draws(orc.draws_for(seed, [n] * (2 * T)))
    aux = orc.RandomSource(322)
    for t in range(4):
        x = aux.normal_vector(n)
        assert rel(op.probe(x, "right"), ref.probe(x, "right")) < 1e-10
    x = aux.normal_vector(n)
    want = ref.run("normalize", "alternate", T - 4, x, keep=False)[0]
    got = op.run(x, T - 4, update="normalize")
    assert rel(got, want) < TOL64


def test_goe_adjoint_symmetry(orc, lm):
    n = 8
    op = lm.GOEOperator(n, seed=321)
    aux = orc.RandomSource(322)
    x, w = aux.normal_vector(n), aux.normal_vector(n)
    ax = op.probe(x, "right")
    aw = op.probe(w, "left")
    assert abs(w @ ax - aw @ x) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(w)


# ------------------------------------------------------------------- fp32
def test_fp32_parity(orc, lm):
    n, T, seed = 3000, 20, 11
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    ref = orc.Operator("ginibre", m=n, n=n, sigma=1 / np.sqrt(n), seed=seed)
    want = ref.run("normalize", "alternate", T, x1, keep=False)[0]
    op = lm.GinibreOperator(n, n, sigma=1 / np.sqrt(n), seed=seed, draws="injected", dtype="f32", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    got = op.run(x1.astype(np.float32), T, update="normalize")
    assert got.dtype == np.float32
    assert rel(got, want) < TOL32


# -------------------------------------------------------------- semantics
def test_errors_leave_state_untouched(orc, lm):
    n, seed = 50, 3
    ref = orc.Operator("ginibre", m=n, n=n, seed=seed)
    op = lm.GinibreOperator(n, n, seed=seed, draws="injected")
    op.push_draws(orc.draws_for(seed, [n] * 3))
    with pytest.raises(ValueError, match="probe: input dimension mismatch"):
        op.probe(np.ones(n + 1), "right")
    bad = np.ones(n)
    bad[3] = np.nan
    with pytest.raises(ValueError, match="probe: non-finite input"):
        op.probe(bad, "right")
    with pytest.raises(ValueError, match="side must be"):
        op.probe(np.ones(n), "up")
    x = orc.RandomSource(4).normal_vector(n)
    assert rel(op.probe(x, "right"), ref.probe(x, "right")) < 1e-12
    assert op.remaining_probes == n - 1


def test_device_nonfinite_input_rejected(lm):
    torch = pytest.importorskip("torch")
    op = lm.HaarOperator(300, seed=1)
    x = torch.ones(300, dtype=torch.float64, device="cuda")
    x[7] = float("inf")
    with pytest.raises(ValueError, match="non-finite"):
        op.probe(x, "right")
    assert op.remaining_probes == 300
    y = op.probe(torch.ones(300, dtype=torch.float64, device="cuda"), "right")
    assert y.is_cuda and abs(float(y.norm()) - np.sqrt(300)) < 1e-9


def test_budget_exhausted(lm):
    op = lm.GinibreOperator(6, 4, sigma=0.5, seed=7)  # test_smoke.py:29-52
    assert (op.rows, op.cols, op.remaining_probes) == (6, 4, 4)
    x = np.ones(4)
    y1 = op.probe(x)
    y2 = op.probe(x, side="right")
    assert np.allclose(y1, y2, atol=1e-12)
    again = lm.GinibreOperator(6, 4, sigma=0.5, seed=7)
    assert np.array_equal(again.probe(x), y1)
    w = np.zeros(6)
    w[0] = 1.0
    assert op.probe(w, side="left").shape == (4,)
    assert op.remaining_probes == 1
    op.probe(x)
    with pytest.raises(lm.BudgetExhausted):
        op.probe(x)
    h = lm.HaarOperator(3, seed=2)
    for t in range(3):
        h.probe(np.ones(3), "left" if t % 2 else "right")
    with pytest.raises(lm.BudgetExhausted, match="HaarOperator: probe budget n spent"):
        h.probe(np.ones(3))


def test_run_validation_messages(lm):
    op = lm.GinibreOperator(8, 8, 1.0, seed=971)
    with pytest.raises(ValueError, match="iteration count exceeds the operator's probe budget"):
        op.run(np.ones(8), 9)
    op.run(np.ones(8), 8)
    assert op.remaining_probes == 0


def test_nonfinite_iterate_aborts_with_step(lm):
    # dynamics.hpp:64-67; identity update on a huge input overflows
    op = lm.GinibreOperator(8, 8, 1e200, seed=3)
    with pytest.raises(RuntimeError, match=r"non-finite iterate at step \d"):
        op.run(np.full(8, 1e200), 5, update="identity")
    # state is that after the failing step: remaining reflects served probes
    assert 0 < 8 - op.remaining_probes <= 5


def test_skip_reflector_fault(orc, lm):
    # test_ginibre.cpp:182-192 + parity of the faulted operator
    n, seed = 8, 61
    ref = orc.Operator("ginibre", m=n, n=n, seed=seed, skip_reflector=True)
    op = lm.GinibreOperator(n, n, seed=seed, draws="injected", skip_reflector=True)
    op.push_draws(orc.draws_for(seed, [n] * 4))
    x = orc.RandomSource(62).normal_vector(n)
    for t in range(4):
        s = "right" if t != 2 else "left"
        assert rel(op.probe(x, s), ref.probe(x, s)) < 1e-10
        assert op.chain_sizes() == ref.chain_sizes()
    href = orc.Operator("haar", n=20, seed=5, skip_reflector=True)
    h = lm.HaarOperator(20, seed=5, draws="injected", skip_reflector=True)
    h.push_draws(orc.draws_for(5, [20] * 6))
    aux = orc.RandomSource(6)
    for t in range(6):
        x = aux.normal_vector(20)
        s = "left" if t % 2 else "right"
        assert rel(h.probe(x, s), href.probe(x, s)) < 1e-10
    assert h.chain_sizes() == href.chain_sizes()


@pytest.mark.parametrize("rule", ["negative_at_zero", "zero_when_negative"])
def test_sign_rules(orc, lm, rule):
    n, seed = 40, 17
    ref = orc.Operator("haar", n=n, seed=seed, sign_rule=rule)
    op = lm.HaarOperator(n, seed=seed, draws="injected", sign_rule=rule)
    op.push_draws(orc.draws_for(seed, [n] * 8))
    aux = orc.RandomSource(18)
    for t in range(8):
        x = aux.normal_vector(n)
        want = ref.probe(x, "right")
        got = op.probe(x, "right")
        assert np.linalg.norm(got - want) <= 1e-10 * max(np.linalg.norm(want), 1.0), t


# ------------------------------------------------- philox production mode
def test_philox_deterministic_and_distributed(lm):
    a = lm.HaarOperator(5000, seed=9)
    b = lm.HaarOperator(5000, seed=9)
    x = np.random.default_rng(0).standard_normal(5000)
    ya, yb = a.probe(x), b.probe(x)
    assert np.array_equal(ya, yb)
    c = lm.HaarOperator(5000, seed=10)
    assert not np.array_equal(c.probe(x), ya)
    # first Ginibre probe entries carry variance sigma^2 (test_ginibre.cpp:162-180)
    m, sigma = 200000, 0.5
    op = lm.GinibreOperator(m, 4, sigma, seed=1000)
    y = op.probe(np.array([1.0, 0, 0, 0]), "right")
    assert abs(y.mean()) < 4 * sigma / np.sqrt(m)
    assert abs(y.var() - sigma ** 2) < 0.02 * sigma ** 2
    from scipy import stats

    assert stats.kstest(y / sigma, "norm").pvalue > 1e-3


def test_large_haar_isometry(lm):
    torch = pytest.importorskip("torch")
    n = 1_000_000
    op = lm.HaarOperator(n, seed=3, capacity=16)
    gen = torch.Generator(device="cuda").manual_seed(0)
    xs = []
    for t in range(16):
        x = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
        y = op.probe(x, "right" if t % 4 else "left")
        assert abs(float(y.norm()) - float(x.norm())) <= 1e-12 * float(x.norm())
        xs.append((x, y))
    # inner products between same-side probes are preserved
    (x1, y1), (x2, y2) = xs[1], xs[2]
    assert abs(float(y1 @ y2) - float(x1 @ x2)) <= 1e-10 * float(x1.norm() * x2.norm())


# ------------------------------------- BASELINE configs 4 and 5 dynamics
def test_amp_sparse_regression_parity(orc, lm):
    # config 4 shape at reduced n: m = 2n, entries N(0, 1/m), beta ~ Bernoulli(0.1) N(0,1), w ~ N(0, 0.01)
    n, T, seed = 1500, 12, 21
    m = 2 * n
    rng = np.random.default_rng(0)
    beta = (rng.random(n) < 0.1) * rng.standard_normal(n)
    w = 0.1 * rng.standard_normal(m)
    ref = orc.Operator("ginibre", m=m, n=n, sigma=m ** -0.5, seed=seed)
    xr, mser = ref.amp(beta, w, T)
    import torch

    for dev in (False, True):  # host arrays in/out, then CUDA tensors in/out (device-resident run)
        op = lm.GinibreOperator(m, n, m ** -0.5, seed, draws="injected", capacity=2 * T + 1)
        op.push_draws(orc.draws_for(seed, [m] + [n, m] * T))
        if dev:
            x, mse = lm.amp_sparse_regression(op, torch.tensor(beta, device="cuda"), torch.tensor(w, device="cuda"), T)
            x, mse = x.cpu().numpy(), mse.cpu().numpy()
        else:
            x, mse = lm.amp_sparse_regression(op, beta, w, T)
        assert rel(x, xr) < TOL64
        assert np.max(np.abs(mse - mser) / mser) < 1e-9
        assert mse[-1] < 0.5 * mse[0]  # AMP converges


def test_spiked_goe_power_parity(orc, lm):
    # config 5 shape at reduced n: GOE inner sigma = 1/sqrt(n), theta = 2
    n, T, seed = 900, 20, 31
    u = orc.RandomSource(seed, 1).normal_vector(n)
    u /= np.linalg.norm(u)
    x1 = orc.RandomSource(seed, 2).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    ref = orc.Operator("goe", n=n, sigma=n ** -0.5, seed=seed)
    xr, ovr = ref.spiked_power(u, x1, T)
    op = lm.GOEOperator(n, seed, sigma=n ** -0.5, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * (2 * T)))
    x, ov = lm.spiked_power(op, u, x1, T)
    assert rel(x, xr) < TOL64
    assert np.max(np.abs(ov - ovr)) < 1e-9
    assert abs(ovr[-1]) > 0.5  # theta = 2 > 1: the spike is detected


def test_run_rejects_nonfinite_host_x1_on_device(orc, lm):
    # the finiteness of x_1 (check_probe_input) is checked by the first device
    # pass: same message, operator state untouched, a valid run afterwards
    n, T, seed = 2000, 6, 12
    op = lm.HaarOperator(n, seed=seed, draws="injected", capacity=T)
    op.push_draws(orc.draws_for(seed, [n] * T))
    bad = np.ones(n)
    bad[11] = np.inf
    for graph in (False, True):
        with pytest.raises(ValueError, match="probe: non-finite input"):
            op.run(bad, T, update="normalize", sides="right", use_graph=graph)
        assert op.remaining_probes == n
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    want = orc.Operator("haar", n=n, seed=seed).run("normalize", "right", T, x1, keep=False)[0]
    out = np.empty(n)
    got = op.run(x1, T, update="normalize", sides="right", out=out)
    assert got is out and rel(out, want) < 1e-9
