"""The two-pass Ginibre / GOE kernels (k_nt) in every shape and
schedule the host can pick, each checked against the CPU oracle:

* sub-tiles taller than 64 rows (run as blocks of 64 rows) are only taken when
  every CTA still gets >= 16 sub-tiles, i.e. at n >= ~6e5 — the config-4/5 sizes
  — so a 6.5e5 run covers them, against the same run with HD_NT_MAX_RS=64;
* the two-slot schedule (T phase of sub-tile j in slot j, after the epilogue's
  mbarrier) is the default only with 4 stages; HD_NT_SCHED forces either
  schedule on every launch of an AMP run (config 4's epilogues);
* fp32 passes keep 32-row sub-tiles (TMA writes each panel's columns at a 128-B
  aligned stage offset), so runs whose passes grow past 256 columns take the
  three-pass sequence: a spiked-GOE fp32 run that crosses that width, against
  the fp64 oracle (the power method converges, so fp32 tracks it to ~1e-5).
References: ginibre.hpp:58-106, ensembles.hpp:117-127."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel_rows(a, b):
    a = np.asarray(a)
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


@pytest.fixture
def env_flags():
    saved = {}

    def set_(**kv):
        for k, v in kv.items():
            saved.setdefault(k, os.environ.get(k))
            os.environ[k] = v

    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


N_TALL, T_TALL, SEED_TALL = 650_000, 24, 12


@pytest.fixture(scope="module")
def tall_case(orc):
    x1 = orc.RandomSource(SEED_TALL, 1).normal_vector(N_TALL)
    x1 /= np.linalg.norm(x1)
    ref = orc.Operator("ginibre", m=N_TALL, n=N_TALL, sigma=N_TALL ** -0.5, seed=SEED_TALL).run(
        "normalize", "alternate", T_TALL, x1, keep=True)
    return x1, ref


@pytest.mark.parametrize("max_rs", ["256", "64"])
def test_tall_subtiles_match_oracle_every_iterate(lm, tall_case, env_flags, max_rs):
    env_flags(HD_NT_MAX_RS=max_rs)
    x1, ref = tall_case
    op = lm.GinibreOperator(N_TALL, N_TALL, N_TALL ** -0.5, SEED_TALL, draws="reference", capacity=T_TALL)
    traj = op.run(x1, T_TALL, update="normalize", sides="alternate", keep_trajectory=True)
    assert rel_rows(traj, ref).max() < 1e-9


@pytest.mark.parametrize("sched", ["0", "1"])
def test_amp_run_under_either_slot_schedule_matches_oracle(orc, lm, env_flags, sched):
    import torch

    env_flags(HD_NT_SCHED=sched)
    n, T, seed = 20_000, 60, 14
    m = 2 * n
    g = torch.Generator("cuda").manual_seed(seed)
    beta = (torch.rand(n, device="cuda", generator=g, dtype=torch.float64) < 0.1) * torch.randn(
        n, device="cuda", generator=g, dtype=torch.float64)
    w = 0.1 * torch.randn(m, device="cuda", generator=g, dtype=torch.float64)
    op = lm.GinibreOperator(m, n, m ** -0.5, seed, capacity=T + 1)
    x, mse = lm.amp_sparse_regression(op, beta, w, T)
    draws = np.concatenate([lm.philox_normals(seed, k, L).cpu().numpy()
                            for k, L in enumerate([m] + [n, m] * T)])
    ref = orc.Operator("ginibre", m=m, n=n, sigma=m ** -0.5, draws=draws)
    xr, mser = ref.amp(beta.cpu().numpy(), w.cpu().numpy(), T)
    assert rel_rows(x.cpu().numpy(), xr) < 1e-9
    assert np.max(np.abs(mse.cpu().numpy() - mser) / mser) < 1e-9


def test_fp32_wide_runs_track_the_fp64_oracle(orc, lm):
    n, T, seed = 3000, 200, 33  # 400 inner probes: output passes up to ~400 columns
    u = orc.RandomSource(seed, 1).normal_vector(n)
    u /= np.linalg.norm(u)
    x1 = orc.RandomSource(seed, 2).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    xr, ovr = orc.Operator("goe", n=n, sigma=n ** -0.5, seed=seed).spiked_power(u, x1, T)
    op = lm.GOEOperator(n, seed, sigma=n ** -0.5, draws="reference", capacity=T, dtype="f32")
    x, ov = lm.spiked_power(op, u.astype(np.float32), x1.astype(np.float32), T)
    assert np.all(np.isfinite(x))
    assert abs(abs(ovr[-1]) - 0.866) < 0.05  # theta = 2: the overlap converges to sqrt(1 - 1/theta^2)
    assert np.max(np.abs(np.asarray(ov)[-50:] - ovr[-50:])) < 1e-4  # converged part of the curve
