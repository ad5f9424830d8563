"""The reference's application drivers on the B200 operators:
ista_curves (experiments.cpp:73-151), spectral_summary (experiments.cpp:153-300
with eigensolve.hpp power / restarted Krylov), sample_dense_haar
(ensembles.hpp:55-81) and two_sample_ks (stats.cpp:8-56), with the reference
Python signatures (bindings/module.cpp:113-194).

Every matrix-vector product runs on the GPU: the lazy "hd" backend through
the device operators (probes on CUDA tensors), the "direct" backend as a
dense matrix resident in HBM (cuBLAS GEMV; the dense Haar sample is a
cuSOLVER QR with the phase correction). Seeding follows the reference:
trial i of backend b uses base = derive_seed(seed, 2 i + b), the matrix from
RandomSource(base, 0) and the data from RandomSource(base, 1)
(experiments.cpp:122-125,183-187). With ``draws="reference"`` (default) the
lazy operators draw that exact stream, so the curves are the reference's up
to floating-point reduction order; ``draws="philox"`` switches the matrix
draws to device Philox (same distribution, no host generation).
"""
from __future__ import annotations

import math
import os

import numpy as np

from .._native import BudgetExhausted, ResourceCapExceeded


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("lazymat: the B200 drivers need a CUDA device (there is no CPU fallback)")
    return torch


def _backend(name: str) -> int:  # module.cpp:30-34
    if name == "hd":
        return 0
    if name == "direct":
        return 1
    raise ValueError("backend must be 'hd' or 'direct'")


# ----------------------------------------------------------------- stats.cpp
def mean_of(x) -> float:  # stats.cpp:86-91 (sequential sum, like the reference)
    if len(x) == 0:
        return 0.0
    s = 0.0
    for v in x:
        s += float(v)
    return s / len(x)


def stderr_of_mean(x) -> float:  # stats.cpp:93-106
    if len(x) < 2:
        return 0.0
    m = mean_of(x)
    s = 0.0
    for v in x:
        s += (float(v) - m) * (float(v) - m)
    return math.sqrt(s / (len(x) - 1) / len(x))


def ks_survival(lam: float) -> float:  # stats.cpp:8-22
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


def two_sample_ks(a, b) -> dict:
    """Two-sample Kolmogorov-Smirnov statistic with the asymptotic p-value
    (stats.cpp:33-56): sup over the merged distinct values of the ECDF gap,
    ties advancing both ECDFs first; Stephens' effective-n correction."""
    a = np.sort(np.asarray(a, dtype=np.float64).reshape(-1))
    b = np.sort(np.asarray(b, dtype=np.float64).reshape(-1))
    if a.size == 0 or b.size == 0:
        return {"statistic": 0.0, "p_value": 1.0}
    n1, n2 = float(a.size), float(b.size)
    vals = np.unique(np.concatenate([a, b]))
    i = np.searchsorted(a, vals, side="right")
    j = np.searchsorted(b, vals, side="right")
    d = float(np.max(np.abs(i / n1 - j / n2)))
    rn = math.sqrt(n1 * n2 / (n1 + n2))
    return {"statistic": d, "p_value": ks_survival((rn + 0.12 + 0.11 / rn) * d)}


# ------------------------------------------------- dense samples (direct)
def _oracle_cap() -> int:  # ensembles.hpp:22-28
    s = os.environ.get("LAZYMAT_ORACLE_DIM_CAP")
    if s:
        try:
            v = int(s)
        except ValueError:
            v = 0
        if v >= 1:
            return v
    return 2048


def _check_cap(rows: int, cols: int) -> None:  # ensembles.hpp:30-38
    cap = _oracle_cap()
    if max(rows, cols) > cap:
        raise ResourceCapExceeded(f"dense oracle: dimension {max(rows, cols)} exceeds cap {cap} "
                                  "(set LAZYMAT_ORACLE_DIM_CAP to raise)")


def _column_filled(rs, rows: int, cols: int):
    """Column j = normals(rows), j = 0..cols-1 (ensembles.hpp:47,64), on the GPU."""
    torch = _torch()
    g = rs.normal_vector(rows * cols).reshape(cols, rows)
    return torch.from_numpy(g).cuda().t().contiguous()


def _dense_ginibre(m: int, n: int, sigma: float, rs):
    if not (m >= 1 and n >= 1):
        raise ValueError("sample_dense_ginibre: dims must be positive")
    if not sigma > 0:
        raise ValueError("sample_dense_ginibre: sigma must be positive")
    _check_cap(m, n)
    return _column_filled(rs, m, n) * sigma


def _dense_haar(n: int, rs):
    """Q of QR(G) with R's diagonal signs absorbed (ensembles.hpp:59-81): the
    unique orthogonal factor with a positive-diagonal R, so it does not depend
    on the QR routine (cuSOLVER here, Eigen's HouseholderQR in the reference)."""
    torch = _torch()
    if n < 1:
        raise ValueError("sample_dense_haar: n must be positive")
    _check_cap(n, n)
    q, r = torch.linalg.qr(_column_filled(rs, n, n))
    d = torch.diagonal(r)
    ph = torch.where(d == 0, torch.ones_like(d), torch.sign(d))
    return q * ph[None, :]


def sample_dense_haar(n: int, seed: int = 1) -> np.ndarray:
    """module.cpp:113-120: materialised orthogonal sample from RandomSource(seed)."""
    from . import RandomSource

    return _dense_haar(int(n), RandomSource(seed, 0)).cpu().numpy()


class _Dense:
    """DenseOperator: the materialised matrix resident in HBM."""

    def __init__(self, a):
        self.a = a
        self.rows, self.cols = a.shape

    def probe(self, x, side: str = "right"):
        return self.a @ x if side == "right" else self.a.t() @ x


# ------------------------------------------------------------- ISTA (f3)
def _ista_validate(n, m_ratio, iterations, lam, tau, rho, sigma_s, sigma_w, trials):  # experiments.cpp:45-56
    if n < 2:
        raise ValueError("ista: n must be at least 2")
    if int(math.floor(n * m_ratio)) < 1:
        raise ValueError("ista: m_ratio gives an empty design")
    if iterations < 1:
        raise ValueError("ista: need at least one iteration")
    if not (lam > 0.0 and tau > 0.0):
        raise ValueError("ista: lambda, tau must be positive")
    if not (0.0 < rho < 1.0):
        raise ValueError("ista: rho must lie in (0,1)")
    if not (sigma_s > 0.0 and sigma_w > 0.0):
        raise ValueError("ista: sigma_s, sigma_w must be positive")
    if trials < 1:
        raise ValueError("ista: trials must be positive")


def soft_threshold(x, theta: float):
    """experiments.cpp:31-39 on a device tensor: sign(x) max(|x| - theta, 0)."""
    torch = _torch()
    if theta < 0.0:
        raise ValueError("soft_threshold: threshold must be nonnegative")
    mag = x.abs() - theta
    return torch.where(mag > 0.0, torch.where(x > 0.0, mag, -mag), torch.zeros_like(x))


def ista_trial(n: int = 256, m_ratio: float = 0.5, iterations: int = 50, lambda_: float = 2.0, tau: float = 0.3,
               rho: float = 0.2, sigma_s: float = 2.0, sigma_w: float = 0.1, seed: int = 1, trial: int = 0,
               backend: str = "hd", *, draws: str = "reference"):
    """One trial (experiments.cpp:73-131): returns (mse[T] numpy, x_T device tensor).

    x^0 = 0; per iteration r = y - A x (right probe), x = soft(x + tau A^T r,
    lambda tau) (left probe): the reference's 2T-step run_dynamics with history
    depth 1 (experiments.cpp:88-104), whose first probe is A 0."""
    from . import GinibreOperator, RandomSource, derive_seed

    _torch()
    b = _backend(backend)
    _ista_validate(n, m_ratio, iterations, lambda_, tau, rho, sigma_s, sigma_w, 1)
    m = int(math.floor(n * m_ratio))
    if b == 0 and 2 * iterations + 1 > min(m, n):
        raise BudgetExhausted("ista: data generation plus 2T probes exceed the min(m, n) budget")
    base = derive_seed(seed, 2 * trial + b)
    sigma = 1.0 / math.sqrt(m)
    if b == 0:
        op = GinibreOperator(m, n, sigma, base, draws=draws, capacity=iterations + 1)
    else:
        op = _Dense(_dense_ginibre(m, n, sigma, RandomSource(base, 0)))
    return ista_on(op, RandomSource(base, 1), iterations, lambda_, tau, rho, sigma_s, sigma_w)


def ista_on(op, data, iterations: int, lambda_: float = 2.0, tau: float = 0.3, rho: float = 0.2,
            sigma_s: float = 2.0, sigma_w: float = 0.1):
    """ista_trial_on (experiments.cpp:73-111) over a caller-supplied design
    operator (lazy or dense) and data source: (mse[T] numpy, x_T device)."""
    torch = _torch()
    m, n = op.rows, op.cols
    beta = torch.from_numpy(data.bernoulli_gaussian(n, rho, sigma_s)).cuda()
    noise = torch.from_numpy(data.normal_vector(m)).cuda() * sigma_w
    y_obs = op.probe(beta, "right") + noise
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    shrink = lambda_ * tau
    mse = torch.empty(iterations, dtype=torch.float64, device="cuda")
    for t in range(iterations):
        r = y_obs - op.probe(x, "right")
        x = soft_threshold(x + tau * op.probe(r, "left"), shrink)
        d = x - beta
        mse[t] = torch.dot(d, d) / n
    return mse.cpu().numpy(), x


def ista_curves(n: int = 256, m_ratio: float = 0.5, iterations: int = 50, lambda_: float = 2.0, tau: float = 0.3,
                rho: float = 0.2, sigma_s: float = 2.0, sigma_w: float = 0.1, trials: int = 1, seed: int = 1,
                threads: int = 1, backend: str = "hd", *, draws: str = "reference", **kw) -> dict:
    """module.cpp:122-151 / experiments.cpp:133-151: trial-averaged MSE curve of
    ISTA on a lazily served ('hd') or materialised ('direct') design. The
    reference's keyword ``lambda`` is accepted (``lambda_`` positionally);
    ``threads`` is accepted for signature parity (trials run on the GPU)."""
    if "lambda" in kw:
        lambda_ = kw.pop("lambda")
    if kw:
        raise TypeError(f"ista_curves() got unexpected keyword arguments {sorted(kw)}")
    _backend(backend)
    _ista_validate(n, m_ratio, iterations, lambda_, tau, rho, sigma_s, sigma_w, trials)
    curves = [ista_trial(n, m_ratio, iterations, lambda_, tau, rho, sigma_s, sigma_w, seed, i, backend,
                         draws=draws)[0] for i in range(trials)]
    mean = [mean_of([c[t] for c in curves]) for t in range(iterations)]
    err = [stderr_of_mean([c[t] for c in curves]) for t in range(iterations)]
    return {"mse_mean": mean, "mse_stderr": err}


# ------------------------------------------------------- eigensolve.hpp
def power_iteration(apply, start, max_matvecs: int = 300, tol: float = 1e-8) -> dict:
    """eigensolve.hpp:28-52 on device vectors: Rayleigh quotient + residual test."""
    torch = _torch()
    if start.numel() < 1:
        raise ValueError("power_iteration: empty start vector")
    nrm = float(torch.linalg.vector_norm(start))
    if not nrm > 0:
        raise ValueError("power_iteration: zero start vector")
    res = {"lambda": 0.0, "vector": None, "matvecs": 0, "residual": 0.0, "converged": False}
    x = start / nrm
    while res["matvecs"] < max_matvecs:
        z = apply(x)
        res["matvecs"] += 1
        lam = float(torch.dot(x, z))
        rnorm = float(torch.linalg.vector_norm(z - lam * x))
        res["lambda"], res["vector"] = lam, x
        res["residual"] = rnorm if lam == 0.0 else rnorm / abs(lam)
        if rnorm <= tol * abs(lam):
            res["converged"] = True
            return res
        zn = float(torch.linalg.vector_norm(z))
        if zn == 0.0:
            return res  # start lies in the kernel
        x = z / zn
    return res


def restarted_krylov(apply, start, max_matvecs: int = 300, tol: float = 1e-8, basis: int = 24) -> dict:
    """eigensolve.hpp:54-124: Lanczos basis with two-pass full
    reorthogonalisation on the device, Rayleigh-Ritz of the small projected
    matrix on the host, restart from the best Ritz vector; the residual comes
    from the Arnoldi relation (no extra matvec)."""
    torch = _torch()
    if start.numel() < 1:
        raise ValueError("restarted_krylov: empty start vector")
    nrm = float(torch.linalg.vector_norm(start))
    if not nrm > 0:
        raise ValueError("restarted_krylov: zero start vector")
    if basis < 2:
        raise ValueError("restarted_krylov: basis must be >= 2")
    n = start.numel()
    mb = min(basis, n)
    res = {"lambda": 0.0, "vector": None, "matvecs": 0, "residual": 0.0, "converged": False}
    v0 = start / nrm
    while res["matvecs"] < max_matvecs:
        V = torch.zeros((mb, n), dtype=start.dtype, device=start.device)  # row j = basis vector j
        h = np.zeros((mb, mb))
        V[0] = v0
        grown, beta, breakdown = 0, 0.0, False
        while grown < mb and res["matvecs"] < max_matvecs:
            j = grown
            w = apply(V[j])
            res["matvecs"] += 1
            for p in range(2):
                for i in range(j + 1):
                    c = torch.dot(V[i], w)
                    if p == 0:
                        h[i, j] += float(c)
                    w = w - c * V[i]
            beta = float(torch.linalg.vector_norm(w))
            grown = j + 1
            if beta <= 1e-14:
                breakdown = True  # exact invariant subspace
                break
            if grown < mb:
                h[j + 1, j] = h[j, j + 1] = beta
                V[j + 1] = w / beta
        evals, evecs = np.linalg.eigh(h[:grown, :grown])
        best = int(np.argmax(np.abs(evals)))
        theta = float(evals[best])
        s = evecs[:, best]
        u = torch.from_numpy(np.ascontiguousarray(s)).to(V) @ V[:grown]
        u = u / torch.linalg.vector_norm(u)
        rnorm = 0.0 if breakdown else beta * abs(float(s[grown - 1]))
        res["lambda"], res["vector"] = theta, u
        res["residual"] = rnorm if theta == 0.0 else rnorm / abs(theta)
        if breakdown or rnorm <= tol * abs(theta):
            res["converged"] = True
            return res
        v0 = u
    return res


# ------------------------------------------------------------ spectral (f3)
def _spectral_validate(n, alpha, tol, max_matvecs, krylov_basis, trials):  # experiments.cpp:157-164
    if n < 2:
        raise ValueError("spectral: n must be at least 2")
    if not alpha > 1.0:
        raise ValueError("spectral: alpha must exceed 1")
    if not tol > 0.0:
        raise ValueError("spectral: tol must be positive")
    if max_matvecs < 1:
        raise ValueError("spectral: need a positive matvec budget")
    if krylov_basis < 2:
        raise ValueError("spectral: krylov basis must be >= 2")
    if trials < 1:
        raise ValueError("spectral: trials must be positive")


def spectral_trial(n: int = 256, alpha: float = 2.0, seed: int = 1, trial: int = 0, backend: str = "hd",
                   solver: str = "power", max_matvecs: int = 300, tol: float = 1e-8, krylov_basis: int = 24, *,
                   draws: str = "reference") -> dict:
    """experiments.cpp:171-258: planted direction xi (norm sqrt(n)), measurements
    y = tanh(|A^T xi|) over the first n rows A of an m x m Haar matrix
    (m = floor(alpha n)), leading eigenpair of D = A diag(y) A^T / m."""
    from . import HaarOperator, RandomSource, SubsampledHaarOperator, derive_seed

    torch = _torch()
    b = _backend(backend)
    _spectral_validate(n, alpha, tol, max_matvecs, krylov_basis, 1)
    m = int(math.floor(alpha * n))
    base = derive_seed(seed, 2 * trial + b)
    data = RandomSource(base, 1)
    if b == 0:
        cap_probes = min(max_matvecs, (m - 1) // 2)
        op = SubsampledHaarOperator(HaarOperator(m, seed=base, draws=draws, capacity=2 * max(cap_probes, 0) + 1), n)
    else:
        op = _Dense(_dense_haar(m, RandomSource(base, 0))[:n].contiguous())
    xi = torch.from_numpy(data.normal_vector(n)).cuda()
    xi = xi * (math.sqrt(n) / float(torch.linalg.vector_norm(xi)))
    y = torch.tanh(op.probe(xi, "left").abs())
    if not bool(((y > 0.0) & (y < 1.0)).all()):
        raise ValueError("spectral: measurement left (0,1)")
    start = torch.from_numpy(data.normal_vector(n)).cuda()
    start = start / torch.linalg.vector_norm(start)
    inv_m = 1.0 / m

    def apply(v):
        return op.probe(op.probe(v, "left") * y, "right") * inv_m

    cap = min(max_matvecs, (m - 1) // 2)  # experiments.cpp:232-238
    if cap < 1:
        raise ValueError("spectral: m too small for even one matvec")
    eig = (restarted_krylov(apply, start, cap, tol, krylov_basis) if solver == "krylov"
           else power_iteration(apply, start, cap, tol))
    v = eig["vector"]
    cos = float(torch.dot(xi, v)) / (float(torch.linalg.vector_norm(xi)) * float(torch.linalg.vector_norm(v)))
    return {"lambda_max": eig["lambda"], "rho": cos * cos, "matvecs": eig["matvecs"], "residual": eig["residual"],
            "converged": eig["converged"]}


def spectral_summary(n: int = 256, alpha: float = 2.0, trials: int = 1, seed: int = 1, threads: int = 1,
                     backend: str = "hd", solver: str = "power", max_matvecs: int = 300, tol: float = 1e-8, *,
                     draws: str = "reference") -> dict:
    """module.cpp:153-181 / experiments.cpp:278-298."""
    _backend(backend)
    _spectral_validate(n, alpha, tol, max_matvecs, 24, trials)
    tr = [spectral_trial(n, alpha, seed, i, backend, solver, max_matvecs, tol, draws=draws) for i in range(trials)]
    rhos = [t["rho"] for t in tr]
    return {"rho_mean": mean_of(rhos), "rho_stderr": stderr_of_mean(rhos),
            "lambda_max_mean": mean_of([t["lambda_max"] for t in tr])}
