"""TEST INFRASTRUCTURE ONLY — restatement of the reference's application
drivers (experiments.cpp, eigensolve.hpp, stats.cpp, ensembles.hpp:40-91)
on top of the C++ oracle operators (oracle.py). Used by tests/ to pin
lazymat.ista_curves / spectral_summary / sample_dense_haar / two_sample_ks.

Vectors are numpy fp64; the lazy ("hd") backend is the oracle's own
Ginibre / Haar operator seeded exactly like the reference
(derive_seed(seed, 2*trial + backend), matrix stream 0, data stream 1,
experiments.cpp:122-125,183-187); the "direct" backend materialises the
dense sample from the same stream (ensembles.hpp:50-81).
"""
from __future__ import annotations

import math

import numpy as np

from . import oracle as orc


# ------------------------------------------------------------------ stats.cpp
def mean_of(x):  # stats.cpp:86-91
    if len(x) == 0:
        return 0.0
    s = 0.0
    for v in x:
        s += v
    return s / len(x)


def stderr_of_mean(x):  # stats.cpp:93-106
    if len(x) == 0:
        return 0.0
    if len(x) < 2:
        return 0.0
    m = mean_of(x)
    s = 0.0
    for v in x:
        s += (v - m) * (v - m)
    return math.sqrt(s / (len(x) - 1) / len(x))


def ks_survival(lam):  # stats.cpp:8-22
    if lam <= 0.0:
        return 1.0
    a = -2.0 * lam * lam
    total, sign = 0.0, 1.0
    for k in range(1, 201):
        term = sign * math.exp(a * k * k)
        total += term
        if abs(term) <= 1e-12 * abs(total):
            return min(max(2.0 * total, 0.0), 1.0)
        sign = -sign
    return 1.0


def two_sample_ks(a, b):  # stats.cpp:33-56
    a, b = sorted(a), sorted(b)
    if not a or not b:
        return {"statistic": 0.0, "p_value": 1.0}
    n1, n2 = float(len(a)), float(len(b))
    i = j = 0
    d = 0.0
    while i < len(a) and j < len(b):
        v = min(a[i], b[j])
        while i < len(a) and a[i] == v:
            i += 1
        while j < len(b) and b[j] == v:
            j += 1
        d = max(d, abs(i / n1 - j / n2))
    ne = n1 * n2 / (n1 + n2)
    rn = math.sqrt(ne)
    return {"statistic": d, "p_value": ks_survival((rn + 0.12 + 0.11 / rn) * d)}


# ------------------------------------------------------ ensembles.hpp:40-91
def sample_dense_ginibre(m, n, sigma, rs):  # column j = normals(m)
    return rs.normal_vector(m * n).reshape(n, m).T * sigma


def sample_dense_haar(n, rs):
    """QR of a column-filled normal sample with R's diagonal phases absorbed
    into Q (ensembles.hpp:59-81): the unique Q of the positive-diagonal QR."""
    g = rs.normal_vector(n * n).reshape(n, n).T
    q, r = np.linalg.qr(g)
    d = np.diag(r)
    ph = np.where(np.abs(d) == 0, 1.0, d / np.abs(d))
    return q * ph[None, :]


class Dense:
    def __init__(self, a):
        self.a = a

    def probe(self, x, side="right"):
        return self.a @ x if side == "right" else self.a.T @ x


class Subsampled:
    """SubsampledHaarOperator (ensembles.hpp:182-215): the first `rows` rows."""

    def __init__(self, inner, rows):
        self.inner, self.rows_, self.n = inner, rows, inner.cols

    def probe(self, x, side="right"):
        if side == "right":
            return self.inner.probe(x, "right")[: self.rows_]
        pad = np.zeros(self.n)
        pad[: self.rows_] = x
        return self.inner.probe(pad, "left")


# --------------------------------------------------------- experiments.cpp
def sample_bernoulli_gaussian(n, rho, sigma_s, rs):  # experiments.cpp:19-29
    out = np.empty(n)
    for i in range(n):
        out[i] = 0.0 if rs.uniform() < rho else sigma_s * rs.normal()
    return out


def soft_threshold(x, theta):  # experiments.cpp:31-39
    mag = np.abs(x) - theta
    return np.where(mag > 0.0, np.where(x > 0.0, mag, -mag), 0.0)


def ista_trial(n=256, m_ratio=0.5, iterations=50, lam=2.0, tau=0.3, rho=0.2, sigma_s=2.0, sigma_w=0.1, seed=1,
               trial=0, backend="hd"):
    """experiments.cpp:73-151 (ista_trial_on + ista_trial)."""
    m = int(math.floor(n * m_ratio))
    base = orc.derive_seed(seed, 2 * trial + (1 if backend == "direct" else 0))
    data = orc.RandomSource(base, 1)
    sigma = 1.0 / math.sqrt(m)
    if backend == "hd":
        op = orc.Operator("ginibre", m=m, n=n, sigma=sigma, seed=base)
    else:
        op = Dense(sample_dense_ginibre(m, n, sigma, orc.RandomSource(base, 0)))
    beta = sample_bernoulli_gaussian(n, rho, sigma_s, data)
    noise = data.normal_vector(m) * sigma_w
    y_obs = op.probe(beta, "right") + noise
    # run_dynamics with 2T steps, depth 1, initial {0, 0}, odd t right: the
    # odd step forms the residual, the even step thresholds (experiments.cpp:88-104)
    x = np.zeros(n)
    mse = []
    for _ in range(iterations):
        r = y_obs - op.probe(x, "right")
        x = soft_threshold(x + tau * op.probe(r, "left"), lam * tau)
        mse.append(float(np.dot(x - beta, x - beta)) / n)
    return np.array(mse), x


def ista_curves(n=256, m_ratio=0.5, iterations=50, lam=2.0, tau=0.3, rho=0.2, sigma_s=2.0, sigma_w=0.1, trials=1,
                seed=1, backend="hd"):
    curves = [ista_trial(n, m_ratio, iterations, lam, tau, rho, sigma_s, sigma_w, seed, i, backend)[0]
              for i in range(trials)]
    cols = [[c[t] for c in curves] for t in range(iterations)]
    return {"mse_mean": [mean_of(c) for c in cols], "mse_stderr": [stderr_of_mean(c) for c in cols]}


# ------------------------------------------------------------ eigensolve.hpp
def power_iteration(apply, start, max_matvecs=300, tol=1e-8):  # eigensolve.hpp:28-52
    res = {"lambda": 0.0, "vector": None, "matvecs": 0, "residual": 0.0, "converged": False}
    x = start / np.linalg.norm(start)
    while res["matvecs"] < max_matvecs:
        z = apply(x)
        res["matvecs"] += 1
        lam = float(x @ z)
        rnorm = float(np.linalg.norm(z - lam * x))
        res.update(vector=x, residual=rnorm if lam == 0.0 else rnorm / abs(lam))
        res["lambda"] = lam
        if rnorm <= tol * abs(lam):
            res["converged"] = True
            return res
        zn = float(np.linalg.norm(z))
        if zn == 0.0:
            return res
        x = z / zn
    return res


def restarted_krylov(apply, start, max_matvecs=300, tol=1e-8, basis=24):  # eigensolve.hpp:54-124
    n = start.size
    mb = min(basis, n)
    res = {"lambda": 0.0, "vector": None, "matvecs": 0, "residual": 0.0, "converged": False}
    v0 = start / np.linalg.norm(start)
    while res["matvecs"] < max_matvecs:
        V = np.zeros((n, mb))
        h = np.zeros((mb, mb))
        V[:, 0] = v0
        grown, beta, breakdown = 0, 0.0, False
        while grown < mb and res["matvecs"] < max_matvecs:
            j = grown
            w = apply(V[:, j])
            res["matvecs"] += 1
            for p in range(2):  # full reorthogonalisation, two passes
                for i in range(j + 1):
                    c = float(V[:, i] @ w)
                    if p == 0:
                        h[i, j] += c
                    w = w - c * V[:, i]
            beta = float(np.linalg.norm(w))
            grown = j + 1
            if beta <= 1e-14:
                breakdown = True
                break
            if grown < mb:
                h[j + 1, j] = h[j, j + 1] = beta
                V[:, j + 1] = w / beta
        evals, evecs = np.linalg.eigh(h[:grown, :grown])
        best = int(np.argmax(np.abs(evals)))
        theta, s = float(evals[best]), evecs[:, best]
        u = V[:, :grown] @ s
        u = u / np.linalg.norm(u)
        rnorm = 0.0 if breakdown else beta * abs(float(s[grown - 1]))
        res.update(vector=u, residual=rnorm if theta == 0.0 else rnorm / abs(theta))
        res["lambda"] = theta
        if breakdown or rnorm <= tol * abs(theta):
            res["converged"] = True
            return res
        v0 = u
    return res


def spectral_trial(n=256, alpha=2.0, seed=1, trial=0, backend="hd", solver="power", max_matvecs=300, tol=1e-8,
                   basis=24, start_perturb=0.0):
    """experiments.cpp:171-258 (spectral_instance + spectral_trial).
    start_perturb (test aid, not in the reference): relative perturbation of
    the start vector, to measure how far rounding-level changes move the
    result (the conditioning the device parity tolerance is set against)."""
    m = int(math.floor(alpha * n))
    base = orc.derive_seed(seed, 2 * trial + (1 if backend == "direct" else 0))
    data = orc.RandomSource(base, 1)
    if backend == "hd":
        op = Subsampled(orc.Operator("haar", n=m, seed=base), n)
    else:
        op = Dense(sample_dense_haar(m, orc.RandomSource(base, 0))[:n, :])
    xi = data.normal_vector(n)
    xi = xi * (math.sqrt(n) / np.linalg.norm(xi))
    y = np.tanh(np.abs(op.probe(xi, "left")))
    assert np.all((y > 0) & (y < 1)), "spectral: measurement left (0,1)"
    start = data.normal_vector(n)
    start = start / np.linalg.norm(start)
    if start_perturb:
        start = start * (1.0 + start_perturb * np.random.default_rng(7).standard_normal(n))
    inv_m = 1.0 / m

    def apply(v):
        return op.probe(op.probe(v, "left") * y, "right") * inv_m

    cap = min(max_matvecs, (m - 1) // 2)
    eig = (restarted_krylov(apply, start, cap, tol, basis) if solver == "krylov"
           else power_iteration(apply, start, cap, tol))
    v = eig["vector"]
    cos = float(xi @ v) / (np.linalg.norm(xi) * np.linalg.norm(v))
    return {"lambda_max": eig["lambda"], "rho": cos * cos, "matvecs": eig["matvecs"], "residual": eig["residual"],
            "converged": eig["converged"]}


def spectral_summary(n=256, alpha=2.0, trials=1, seed=1, backend="hd", solver="power", max_matvecs=300, tol=1e-8):
    tr = [spectral_trial(n, alpha, seed, i, backend, solver, max_matvecs, tol) for i in range(trials)]
    rhos = [t["rho"] for t in tr]
    return {"rho_mean": mean_of(rhos), "rho_stderr": stderr_of_mean(rhos),
            "lambda_max_mean": mean_of([t["lambda_max"] for t in tr]), "trials": tr}


# ----------------------------------------------------- verify.hpp / verify.cpp
class USV:
    """USVOperator (ensembles.hpp:133-180) over two oracle Haar operators."""

    def __init__(self, u, v, sv):
        self.u, self.v, self.sv = u, v, np.asarray(sv, dtype=np.float64)
        self.rows, self.cols = u.rows, v.cols

    def probe(self, x, side="right"):
        k = self.sv.size
        if side == "right":
            w = np.zeros(self.rows)
            w[:k] = self.sv * self.v.probe(x, "right")[:k]
            return self.u.probe(w, "right")
        w = np.zeros(self.cols)
        w[:k] = self.sv * self.u.probe(x, "left")[:k]
        return self.v.probe(w, "left")


def consistency_suite(op, m, n, src, rel_tol=1e-10, isometric=False):
    """verify.hpp:100-160 restated; returns [(name, passed)]."""
    out = []
    nrm = np.linalg.norm

    def scale(a, b):
        return a + b if a + b > 0 else 1.0

    x = src.normal_vector(n)
    y1, y2 = op.probe(x, "right"), op.probe(x, "right")
    out.append(("repeat-probe-right", nrm(y1 - y2) / scale(nrm(y1), nrm(y2)) <= rel_tol))
    if isometric:
        out.append(("isometry", abs(nrm(y1) - nrm(x)) / nrm(x) <= rel_tol))
    z = src.normal_vector(m)
    y1, y2 = op.probe(z, "left"), op.probe(z, "left")
    out.append(("repeat-probe-left", nrm(y1 - y2) / scale(nrm(y1), nrm(y2)) <= rel_tol))
    x1, x2 = src.normal_vector(n), src.normal_vector(n)
    a, b = src.normal_vector(1)[0], src.normal_vector(1)[0]
    y1, y2 = op.probe(x1, "right"), op.probe(x2, "right")
    yc = op.probe(a * x1 + b * x2, "right")
    pred = a * y1 + b * y2
    out.append(("span-linearity", nrm(yc - pred) / scale(nrm(pred), nrm(yc)) <= rel_tol))
    for rnd in range(2):
        x, z = src.normal_vector(n), src.normal_vector(m)
        qx, qtz = op.probe(x, "right"), op.probe(z, "left")
        err = abs(float(z @ qx) - float(qtz @ x)) / scale(nrm(z) * nrm(qx), nrm(qtz) * nrm(x))
        out.append((f"adjoint-bilinear-{rnd + 1}", err <= rel_tol))
    return out


def all_operator_contracts(m, n, seed, mutation="none"):
    """verify.cpp:47-121 over the oracle operators; returns [(name, passed)]."""
    kw = {"skip_reflector": mutation == "skip_reflector",
          "sign_rule": "zero_when_negative" if mutation == "sign_convention" else "stable"}
    res = []
    for idx, (name, rows, cols, iso) in enumerate([("ginibre", m, n, False), ("haar", n, n, True),
                                                   ("goe", n, n, False), ("usv", m, n, False),
                                                   ("subsampled-haar", n, m, False)]):
        s = orc.derive_seed(seed, 16 + idx)
        if name == "ginibre":
            op = orc.Operator("ginibre", m=rows, n=cols, sigma=1.0, seed=s, **kw)
        elif name == "haar":
            op = orc.Operator("haar", n=cols, seed=s, **kw)
        elif name == "goe":
            op = orc.Operator("goe", n=cols, sigma=1.0, seed=s, **kw)
        elif name == "usv":
            sv_src = orc.RandomSource(orc.derive_seed(s, 3))
            sv = [0.5 + sv_src.uniform() for _ in range(min(rows, cols))]
            op = USV(orc.Operator("haar", n=rows, seed=orc.derive_seed(s, 1), **kw),
                     orc.Operator("haar", n=cols, seed=orc.derive_seed(s, 2), **kw), sv)
        else:
            op = Subsampled(orc.Operator("haar", n=cols, seed=orc.derive_seed(s, 1), **kw), rows)
        for cname, ok in consistency_suite(op, rows, cols, orc.RandomSource(orc.derive_seed(seed, 32 + idx), 1),
                                           1e-10, iso):
            res.append((f"{name}/{cname}", ok))
    return res
