"""The reference's verification harness (verify.hpp / verify.cpp) on the B200
operators: algebraic contract suites over the five lazy
ensembles, and the statistical equivalence fixtures that compare the lazy
construction against dense direct simulation by two-sample KS tests —
Theorem 1/2 of the paper, run here on the production path (device Philox
draws by default) against dense samples drawn from the reference's
RandomSource. Negative controls: a mismatched dense ensemble, and the
planted mutations (skip_reflector, sign_convention, uncorrected_qr) that
must each trip a suite (acceptance.cpp:285-333).

Lazy trials drive device operators; the dense side is batched over all
trials on the GPU (batched cuSOLVER QR for the Haar samples, batched GEMV
dynamics), its randomness drawn per trial from RandomSource exactly as the
reference does (derive_seed(seed, 2 i + 1), stream 0).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .experiments import _torch, ista_on, two_sample_ks

MUTATIONS = ("none", "skip_reflector", "sign_convention", "uncorrected_qr")


def faults_for(mutation: str) -> dict:  # verify.cpp:17-31
    if mutation not in MUTATIONS:
        raise ValueError(f"unknown mutation {mutation!r}")
    if mutation == "skip_reflector":
        return {"skip_reflector": True}
    if mutation == "sign_convention":
        return {"sign_rule": "zero_when_negative"}
    return {}  # none / uncorrected_qr (targets the dense oracle)


def oracle_sign_correction(mutation: str) -> bool:  # verify.cpp:33-35
    return mutation != "uncorrected_qr"


@dataclass
class CheckResult:
    name: str
    passed: bool
    detail: str = ""


@dataclass
class SuiteReport:
    suite: str
    checks: list = field(default_factory=list)

    def passed(self) -> bool:
        return all(c.passed for c in self.checks)

    def summary(self) -> str:  # verify.cpp:36-45
        ok = sum(1 for c in self.checks if c.passed)
        s = f"{self.suite}: {ok}/{len(self.checks)} checks passed"
        for c in self.checks:
            if not c.passed:
                s += f"\n  FAIL {c.name} ({c.detail})"
        return s


# -------------------------------------------------------- algebraic suites
def _norm_scale(a: float, b: float) -> float:
    s = a + b
    return s if s > 0 else 1.0


def consistency_suite(op, src, rel_tol: float = 1e-10, isometric: bool = False) -> SuiteReport:
    """verify.hpp:100-160: repeat-probe identity on both sides, span linearity,
    the adjoint bilinear identity (twice) and optionally isometry; 11 probes."""
    rep = SuiteReport("consistency")
    if op.remaining_probes < 11:
        raise ValueError("consistency_suite: needs 11 probes")
    m, n = op.rows, op.cols
    nrm = np.linalg.norm

    def record(name, err, tol):
        rep.checks.append(CheckResult(name, bool(err <= tol), f"err {err:.6g} tol {tol:.6g}"))

    x = src.normal_vector(n)
    y1, y2 = op.probe(x, "right"), op.probe(x, "right")
    record("repeat-probe-right", nrm(y1 - y2) / _norm_scale(nrm(y1), nrm(y2)), rel_tol)
    if isometric:
        record("isometry", abs(nrm(y1) - nrm(x)) / nrm(x), rel_tol)
    z = src.normal_vector(m)
    y1, y2 = op.probe(z, "left"), op.probe(z, "left")
    record("repeat-probe-left", nrm(y1 - y2) / _norm_scale(nrm(y1), nrm(y2)), rel_tol)
    x1, x2 = src.normal_vector(n), src.normal_vector(n)
    a, b = src.normal_vector(1)[0], src.normal_vector(1)[0]
    y1, y2 = op.probe(x1, "right"), op.probe(x2, "right")
    yc = op.probe(a * x1 + b * x2, "right")
    pred = a * y1 + b * y2
    record("span-linearity", nrm(yc - pred) / _norm_scale(nrm(pred), nrm(yc)), rel_tol)
    for rnd in range(2):
        x, z = src.normal_vector(n), src.normal_vector(m)
        qx, qtz = op.probe(x, "right"), op.probe(z, "left")
        s1, s2 = float(z @ qx), float(qtz @ x)
        scale = _norm_scale(nrm(z) * nrm(qx), nrm(qtz) * nrm(x))
        record(f"adjoint-bilinear-{rnd + 1}", abs(s1 - s2) / scale, rel_tol)
    return rep


def make_lazy_operator(kind: str, m: int, n: int, seed: int, mutation: str = "none", draws: str = "reference"):
    """verify.cpp:47-85 on device operators."""
    from . import (GinibreOperator, GOEOperator, HaarOperator, RandomSource, SubsampledHaarOperator, USVOperator,
                   derive_seed)

    f = faults_for(mutation)
    if kind == "ginibre":
        return GinibreOperator(m, n, 1.0, seed, draws=draws, **f)
    if kind == "haar":
        if m != n:
            raise ValueError("make_lazy_operator: haar wants square dims")
        return HaarOperator(n, seed=seed, draws=draws, **f)
    if kind == "goe":
        if m != n:
            raise ValueError("make_lazy_operator: goe wants square dims")
        return GOEOperator(n, seed, draws=draws, **f)
    if kind == "usv":
        u = HaarOperator(m, seed=derive_seed(seed, 1), draws=draws, **f)
        v = HaarOperator(n, seed=derive_seed(seed, 2), draws=draws, **f)
        sv_src = RandomSource(derive_seed(seed, 3))
        sv = np.array([0.5 + sv_src.uniform() for _ in range(min(m, n))])
        return USVOperator(u, v, sv)
    if kind == "subsampled_haar":
        if m > n:
            raise ValueError("make_lazy_operator: subsampled wants rows <= cols")
        return SubsampledHaarOperator(HaarOperator(n, seed=derive_seed(seed, 1), draws=draws, **f), m)
    raise ValueError("make_lazy_operator: unknown ensemble kind")


def all_operator_contracts(m: int, n: int, seed: int, mutation: str = "none", draws: str = "reference") -> SuiteReport:
    """verify.cpp:87-121: consistency_suite over all five lazy ensembles."""
    from . import RandomSource, derive_seed

    if not (m >= n >= 22):
        raise ValueError("all_operator_contracts: want m >= n >= 22")
    rep = SuiteReport("operator-contracts")
    entries = [("ginibre", "ginibre", m, n, False), ("haar", "haar", n, n, True), ("goe", "goe", n, n, False),
               ("usv", "usv", m, n, False), ("subsampled-haar", "subsampled_haar", n, m, False)]
    for idx, (name, kind, rows, cols, iso) in enumerate(entries):
        op = make_lazy_operator(kind, rows, cols, derive_seed(seed, 16 + idx), mutation, draws)
        sub = consistency_suite(op, RandomSource(derive_seed(seed, 32 + idx), 1), 1e-10, iso)
        for c in sub.checks:
            c.name = f"{name}/{c.name}"
            rep.checks.append(c)
    return rep


# ------------------------------------------------------- statistical suites
def _ks_check(name: str, a, b, alpha: float) -> CheckResult:  # verify.cpp:138-145
    r = two_sample_ks(a, b)
    return CheckResult(name, bool(r["p_value"] >= alpha),
                       f"D={r['statistic']:.4g} p={r['p_value']:.4g} alpha={alpha:.4g} (n={len(a)} vs {len(b)})")


def _soft(x, th):
    torch = _torch()
    mag = x.abs() - th
    return torch.where(mag > 0.0, torch.where(x > 0.0, mag, -mag), torch.zeros_like(x))


def ista_equivalence_suite(trials: int = 10000, significance: float = 1e-3, seed: int = 1, mutation: str = "none",
                           draws: str = "philox") -> SuiteReport:
    """verify.cpp:147-196: ISTA fixture n = 64, m = 32, T = 15; lazy (device
    operator with the mutation's faults) vs dense design with independent
    randomness; KS on the final MSE and final coordinates 0 and 32."""
    from . import GinibreOperator, RandomSource, derive_seed

    torch = _torch()
    if trials < 2:
        raise ValueError("ista_equivalence_suite: need at least 2 trials")
    n, m, T, lam, tau, rho, ss, sw = 64, 32, 15, 2.0, 0.3, 0.2, 2.0, 0.1
    mid = n // 2
    rep = SuiteReport("ista-equivalence")
    hd_mse, hd_c0, hd_cm = [], [], []
    try:
        op = None
        for i in range(trials):
            base = derive_seed(seed, 2 * i)
            if op is None or draws == "injected":
                op = GinibreOperator(m, n, 1.0 / math.sqrt(m), base, draws=draws, capacity=2 * T + 1,
                                     **faults_for(mutation))
            else:
                op.reseed(base)  # fresh operator state, new matrix seed
            mse, x = ista_on(op, RandomSource(base, 1), T, lam, tau, rho, ss, sw)
            xs = x.cpu().numpy()
            hd_mse.append(mse[-1])
            hd_c0.append(xs[0])
            hd_cm.append(xs[mid])
    except Exception as e:  # noqa: BLE001 — a trial that cannot finish is a detected deviation
        rep.checks.append(CheckResult("trials-completed", False, str(e)))
        return rep
    # dense backend, batched over trials: design from RandomSource(base', 0),
    # data from RandomSource(base', 1), base' = derive_seed(seed, 2 i + 1)
    A, beta, noise = [], [], []
    for i in range(trials):
        base = derive_seed(seed, 2 * i + 1)
        A.append(RandomSource(base, 0).normal_vector(m * n).reshape(n, m).T / math.sqrt(m))
        d = RandomSource(base, 1)
        beta.append(d.bernoulli_gaussian(n, rho, ss))
        noise.append(d.normal_vector(m) * sw)
    A = torch.from_numpy(np.stack(A)).cuda()
    beta = torch.from_numpy(np.stack(beta)).cuda()
    y_obs = torch.bmm(A, beta[:, :, None])[:, :, 0] + torch.from_numpy(np.stack(noise)).cuda()
    x = torch.zeros_like(beta)
    At = A.transpose(1, 2)
    for _ in range(T):
        r = y_obs - torch.bmm(A, x[:, :, None])[:, :, 0]
        x = _soft(x + tau * torch.bmm(At, r[:, :, None])[:, :, 0], lam * tau)
    di_mse = (((x - beta) ** 2).sum(1) / n).cpu().numpy()
    xs = x.cpu().numpy()
    alpha = significance / 3
    rep.checks.append(_ks_check("final-mse", hd_mse, di_mse, alpha))
    rep.checks.append(_ks_check("final-coord-0", hd_c0, xs[:, 0], alpha))
    rep.checks.append(_ks_check(f"final-coord-{mid}", hd_cm, xs[:, mid], alpha))
    return rep


HAAR_FIXTURE_DIM = 32
_STEPS = 6


def _haar_fixture_lazy(op, n: int):
    """verify.cpp:206-237: 6 steps of x <- tanh(y) + 0.1 x from e_1, alternating
    sides; (first probe's leading entry, final coord 0, final ||x||^2, ||Q e_1||^2)."""
    torch = _torch()
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    x[0] = 1.0
    first = fsq = 0.0
    for t in range(1, _STEPS + 1):
        y = op.probe(x, "right" if t % 2 == 1 else "left")
        if t == 1:
            first, fsq = float(y[0]), float(torch.dot(y, y))
        x = torch.tanh(y) + 0.1 * x
    return first, float(x[0]), float(torch.dot(x, x)), fsq


def _haar_fixture_dense(Q):
    torch = _torch()
    B, n, _ = Q.shape
    x = torch.zeros((B, n), dtype=torch.float64, device="cuda")
    x[:, 0] = 1.0
    Qt = Q.transpose(1, 2)
    first = fsq = None
    for t in range(1, _STEPS + 1):
        y = torch.bmm(Q if t % 2 == 1 else Qt, x[:, :, None])[:, :, 0]
        if t == 1:
            first, fsq = y[:, 0].clone(), (y * y).sum(1)
        x = torch.tanh(y) + 0.1 * x
    return first.cpu().numpy(), x[:, 0].cpu().numpy(), (x * x).sum(1).cpu().numpy(), fsq.cpu().numpy()


def _haar_fixture_comparison(trials, significance, seed, mutation, draws, mismatched, suite, with_isometry):
    """verify.cpp:241-312."""
    from . import HaarOperator, RandomSource, derive_seed

    torch = _torch()
    if trials < 2:
        raise ValueError("haar fixture: need at least 2 trials")
    n = HAAR_FIXTURE_DIM
    rep = SuiteReport(suite)
    hd = []
    try:
        op = None
        for i in range(trials):
            base = derive_seed(seed, 2 * i)
            if op is None or draws == "injected":
                op = HaarOperator(n, seed=base, draws=draws, capacity=_STEPS, **faults_for(mutation))
            else:
                op.reseed(base)
            hd.append(_haar_fixture_lazy(op, n))
    except Exception as e:  # noqa: BLE001
        rep.checks.append(CheckResult("trials-completed", False, str(e)))
        return rep
    G = np.stack([RandomSource(derive_seed(seed, 2 * i + 1), 0).normal_vector(n * n).reshape(n, n).T
                  for i in range(trials)])
    G = torch.from_numpy(G).cuda()
    if mismatched:  # the wrong ensemble on purpose: N(0, 1/n) entries
        Q = G / math.sqrt(n)
    else:
        Q, R = torch.linalg.qr(G)  # batched cuSOLVER QR
        if oracle_sign_correction(mutation):
            d = torch.diagonal(R, dim1=1, dim2=2)
            Q = Q * torch.where(d == 0, torch.ones_like(d), torch.sign(d))[:, None, :]
    di = _haar_fixture_dense(Q)
    hd = np.array(hd)
    alpha = significance / (4 if with_isometry else 3)
    rep.checks.append(_ks_check("first-probe-entry", hd[:, 0], di[0], alpha))
    rep.checks.append(_ks_check("final-coord-0", hd[:, 1], di[1], alpha))
    rep.checks.append(_ks_check("final-sqnorm", hd[:, 2], di[2], alpha))
    if with_isometry:
        rep.checks.append(_ks_check("first-probe-sqnorm", hd[:, 3], di[3], alpha))
    return rep


def haar_equivalence_suite(trials: int = 10000, significance: float = 1e-3, seed: int = 1, mutation: str = "none",
                           draws: str = "philox") -> SuiteReport:
    return _haar_fixture_comparison(trials, significance, seed, mutation, draws, False, "haar-equivalence", False)


def mismatched_ensemble_control(trials: int = 10000, significance: float = 1e-3, seed: int = 1,
                                draws: str = "philox") -> SuiteReport:
    """A control that must FAIL: the dense side samples the wrong ensemble."""
    return _haar_fixture_comparison(trials, significance, seed, "none", draws, True,
                                    "mismatched-ensemble-control", True)


def with_retry(run, seed: int) -> SuiteReport:
    """verify.cpp:314-342: one re-run with a fresh derived seed before failing."""
    from . import derive_seed

    def guarded(s):
        try:
            return run(s)
        except Exception as e:  # noqa: BLE001
            return SuiteReport("aborted", [CheckResult("completed-without-error", False, str(e))])

    first = guarded(seed)
    if first.passed():
        return first
    second = guarded(derive_seed(seed, 0x7E7A))
    second.suite += " (after retry)"
    return second
