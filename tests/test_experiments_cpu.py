"""CPU side of the application drivers: the statistics helpers (stats.cpp),
the product's spike-and-slab sampler, config validation, and the oracle
restatement of experiments.cpp / eigensolve.hpp checked against the
reference's own expectations (test_experiments.cpp, test_stats.cpp,
tests/python/test_smoke.py)."""
import math

import numpy as np
import pytest

from oracle import experiments as ex


def test_ks_survival_reference_values():
    # test_stats.cpp:28-37
    for f in (ex.ks_survival,):
        assert f(0.0) == 1.0 and f(-2.0) == 1.0
        assert abs(f(1.0) - 0.2699996716773545) <= 1e-12
        assert 0.0 <= f(5.0) < 1e-20
        assert f(0.5) > f(1.0) > f(2.0)


def test_two_sample_ks_product_matches_oracle(lm):
    assert lm.two_sample_ks([1.0, 2, 3, 4], [1.0, 2, 3, 4]) == {"statistic": 0.0, "p_value": 1.0}
    assert lm.two_sample_ks([0.0, 0, 0, 1], [0.0, 0, 1, 1])["statistic"] == 0.25  # ties (test_stats.cpp:58-63)
    assert lm.two_sample_ks([], [1.0, 2.0]) == {"statistic": 0.0, "p_value": 1.0}
    rng = np.random.default_rng(1)
    a = rng.standard_normal(500)
    assert lm.two_sample_ks(list(a), list(a + 5.0))["p_value"] < 1e-10  # test_smoke.py:88-95
    for k in range(20):
        x = rng.standard_normal(50 + k)
        y = np.round(rng.standard_normal(40 + 3 * k) + 0.1 * k, 1)  # with ties
        assert lm.two_sample_ks(x, y) == ex.two_sample_ks(list(x), list(y))


def test_moment_helpers(lm):
    from paper_2101_07464_b200.lazymat import experiments as pe

    x = [1.0, 2.0, 3.0, 4.0]
    assert pe.mean_of(x) == 2.5 == ex.mean_of(x)
    assert pe.stderr_of_mean(x) == ex.stderr_of_mean(x) == math.sqrt((5.0 / 3.0) / 4.0)
    assert pe.stderr_of_mean([3.0]) == 0.0 and pe.mean_of([]) == 0.0


def test_bernoulli_gaussian_product_matches_oracle(orc, lm):
    for seed, (n, rho, ss) in [(701, (100, 1.0, 2.0)), (5, (1000, 0.0, 2.0)), (9, (5000, 0.3, 1.5))]:
        got = lm.RandomSource(seed, 1).bernoulli_gaussian(n, rho, ss)
        want = ex.sample_bernoulli_gaussian(n, rho, ss, orc.RandomSource(seed, 1))
        assert np.array_equal(got, want)
    assert np.linalg.norm(lm.RandomSource(701).bernoulli_gaussian(100, 1.0, 2.0)) == 0.0
    mixed = lm.RandomSource(3).bernoulli_gaussian(100000, 0.3, 2.0)
    assert 29275 <= int((mixed == 0).sum()) <= 30725  # test_experiments.cpp:48-51
    for args, msg in [((0, 0.5, 1.0), "n must be positive"), ((4, -0.1, 1.0), "rho in"),
                      ((4, 1.1, 1.0), "rho in"), ((4, 0.5, 0.0), "sigma_s must be positive")]:
        with pytest.raises(ValueError, match=msg):
            lm.RandomSource(1).bernoulli_gaussian(*args)


@pytest.mark.parametrize("kw,msg", [({"n": 1}, "n must be at least 2"), ({"m_ratio": 0.001}, "empty design"),
                                    ({"iterations": 0}, "at least one iteration"), ({"lambda": 0.0}, "lambda, tau"),
                                    ({"tau": -1.0}, "lambda, tau"), ({"rho": 0.0}, "rho must lie"),
                                    ({"rho": 1.0}, "rho must lie"), ({"sigma_s": 0.0}, "sigma_s, sigma_w"),
                                    ({"sigma_w": 0.0}, "sigma_s, sigma_w"), ({"trials": 0}, "trials must be"),
                                    ({"backend": "gpu"}, "backend must be")])
def test_ista_validation_messages(lm, kw, msg):
    # experiments.cpp:45-56 via test_experiments.cpp:68-106
    with pytest.raises(ValueError, match=msg):
        lm.ista_curves(**kw)


@pytest.mark.parametrize("kw,msg", [({"n": 1}, "n must be at least 2"), ({"alpha": 1.0}, "alpha must exceed 1"),
                                    ({"tol": 0.0}, "tol must be positive"),
                                    ({"max_matvecs": 0}, "positive matvec budget"),
                                    ({"trials": 0}, "trials must be positive")])
def test_spectral_validation_messages(lm, kw, msg):
    with pytest.raises(ValueError, match=msg):
        lm.spectral_summary(**kw)


# ---------------------------------------------- the oracle restatement itself
def test_oracle_soft_threshold_and_design_height():
    x = np.array([3.0, -3, 0.5, -0.5, 0])
    assert np.array_equal(ex.soft_threshold(x, 1.0), np.array([2.0, -2, 0, 0, 0]))
    assert np.array_equal(ex.soft_threshold(x, 0.0), x)
    assert int(math.floor(256 * 0.5)) == 128 and int(math.floor(7 * 0.5)) == 3


def test_oracle_ista_behaviour():
    # test_experiments.cpp:108-185
    a, xa = ex.ista_trial(n=48, iterations=10, trial=3)
    b, xb = ex.ista_trial(n=48, iterations=10, trial=3)
    assert np.array_equal(a, b) and np.array_equal(xa, xb)
    assert not np.array_equal(a, ex.ista_trial(n=48, iterations=10, trial=4)[0])
    assert not np.array_equal(a, ex.ista_trial(n=48, iterations=10, trial=3, backend="direct")[0])
    for backend in ("hd", "direct"):
        mse, x = ex.ista_trial(n=64, iterations=15, backend=backend)
        assert mse.size == 15 and x.size == 64 and np.all(mse >= 0) and mse[-1] < mse[0]
    mse, x = ex.ista_trial(n=32, iterations=6, lam=1e9, backend="direct")
    assert np.linalg.norm(x) == 0.0 and np.all(mse == mse[0])
    c = ex.ista_curves(n=48, iterations=8, trials=4)
    per = [ex.ista_trial(n=48, iterations=8, trial=i)[0] for i in range(4)]
    for t in range(8):
        col = [p[t] for p in per]
        assert c["mse_mean"][t] == ex.mean_of(col) and c["mse_stderr"][t] == ex.stderr_of_mean(col)


def test_oracle_spectral_matches_dense_diagonalisation():
    # test_experiments.cpp:227-245: direct backend vs dense eigendecomposition
    n, alpha = 64, 2.0
    m = int(alpha * n)
    for trial in (0, 1):
        got = ex.spectral_trial(n, alpha, 1, trial, "direct", "krylov", tol=1e-12)
        base = ex.orc.derive_seed(1, 2 * trial + 1)
        data = ex.orc.RandomSource(base, 1)
        a = ex.sample_dense_haar(m, ex.orc.RandomSource(base, 0))[:n]
        xi = data.normal_vector(n)
        xi *= math.sqrt(n) / np.linalg.norm(xi)
        y = np.tanh(np.abs(a.T @ xi))
        w, v = np.linalg.eigh((a * y[None, :]) @ a.T / m)
        cos = xi @ v[:, -1] / (np.linalg.norm(xi) * np.linalg.norm(v[:, -1]))
        assert got["converged"] and got["residual"] <= 1e-12 and got["matvecs"] <= (m - 1) // 2
        assert abs(got["lambda_max"] - w[-1]) <= 1e-8 * abs(w[-1])
        assert abs(got["rho"] - cos * cos) <= 1e-8 * cos * cos
    for backend in ("hd", "direct"):  # test_experiments.cpp:247-261
        r = ex.spectral_trial(48, 2.0, 1, 0, backend, "krylov")
        assert r["lambda_max"] > 0 and 0.2 < r["rho"] <= 1.0


def test_oracle_operator_contracts_and_mutations():
    # verify.cpp:87-121 restated over the oracle operators: clean operators
    # satisfy every algebraic contract; the planted construction defects break some
    ok = ex.all_operator_contracts(96, 64, ex.orc.derive_seed(9, 0))
    assert len(ok) == 26 and all(p for _, p in ok)
    for mut in ("skip_reflector", "sign_convention"):
        res = ex.all_operator_contracts(96, 64, ex.orc.derive_seed(9, 0), mut)
        assert not all(p for _, p in res), mut
