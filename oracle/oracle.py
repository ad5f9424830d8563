"""TEST INFRASTRUCTURE ONLY — ctypes view of the CPU oracle (oracle/hd_oracle.cpp).

The oracle restates the reference hot path (/root/reference/proj: random.cpp,
reflect.hpp, ginibre.hpp, haar.hpp, ensembles.hpp:93-131, dynamics.hpp) in
plain C++. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package
(paper_2101_07464_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


class BudgetExhausted(OracleError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (needs g++)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.or_last_error.restype = C.c_char_p
        L.or_derive_seed.restype = C.c_uint64
        L.or_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.or_rs_new.restype = C.c_void_p
        L.or_rs_new.argtypes = [C.c_uint64, C.c_uint64]
        L.or_rs_free.argtypes = [C.c_void_p]
        L.or_rs_next_u64.restype = C.c_uint64
        L.or_rs_next_u64.argtypes = [C.c_void_p]
        L.or_rs_uniform.restype = C.c_double
        L.or_rs_uniform.argtypes = [C.c_void_p]
        L.or_rs_normal.restype = C.c_double
        L.or_rs_normal.argtypes = [C.c_void_p]
        L.or_rs_normal_vector.argtypes = [C.c_void_p, C.c_int64, _dp]
        L.or_rs_normal_complex_vector.argtypes = [C.c_void_p, C.c_int64, _dp]
        L.or_make_reflector.argtypes = [_dp, C.c_int64, C.c_int64, C.c_double, C.c_int, _dp,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.or_reflector_apply.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int, _dp, _dp]
        L.or_op_new.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_uint64,
                                C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.or_op_free.argtypes = [C.c_void_p]
        L.or_op_remaining.restype = C.c_int64
        L.or_op_remaining.argtypes = [C.c_void_p]
        L.or_op_rows.restype = C.c_int64
        L.or_op_rows.argtypes = [C.c_void_p]
        L.or_op_cols.restype = C.c_int64
        L.or_op_cols.argtypes = [C.c_void_p]
        L.or_op_counts.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.or_op_chain_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.or_op_probe.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_int, _dp, C.c_int64]
        L.or_run_builtin.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, _dp, C.c_void_p,
                                     C.c_int64, C.c_int, _dp]
        L.or_amp.argtypes = [C.c_void_p, _dp, _dp, C.c_int64, C.c_double, _dp, _dp]
        L.or_spiked_power.argtypes = [C.c_void_p, _dp, _dp, C.c_int64, C.c_double, _dp, _dp]
        L.or_c_last_error.restype = C.c_char_p
        L.or_c_make_reflector.argtypes = [_dp, C.c_int64, C.c_int64, _dp, C.POINTER(C.c_double), _dp,
                                          C.POINTER(C.c_int)]
        L.or_c_reflector_apply.argtypes = [_dp, C.c_int64, C.c_int64, _dp, C.c_int, _dp]
        L.or_c_chain_apply.argtypes = [_dp, C.c_int64, C.c_int64, _dp, C.c_int, C.c_int, _dp]
        L.or_c_op_new.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_uint64, C.c_int,
                                  C.POINTER(C.c_void_p)]
        L.or_c_op_free.argtypes = [C.c_void_p]
        L.or_c_op_remaining.restype = C.c_int64
        L.or_c_op_remaining.argtypes = [C.c_void_p]
        L.or_c_op_probe.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_int, _dp, C.c_int64]
        L.or_op_new_queued.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, _dp, C.c_int64,
                                       C.POINTER(C.c_void_p)]
        L.or_bench_app.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_int,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.or_bench_workload.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_int, C.c_int,
                                        C.c_int64, C.c_uint64, C.c_int, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().or_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise BudgetExhausted(msg)
    raise OracleError(msg)


SIDES = {"right": 0, "left": 1}
ENSEMBLES = {"ginibre": 0, "haar": 1, "goe": 2}
UPDATES = {"identity": 0, "normalize": 1, "tanh_mix": 2}
SIDE_RULES = {"alternate": 0, "right": 1, "left": 2}
SIGN_RULES = {"stable": 0, "negative_at_zero": 1, "zero_when_negative": 2}


def derive_seed(base: int, index: int) -> int:
    return int(lib().or_derive_seed(base, index))


class RandomSource:
    """random.hpp:55-112 restated."""

    def __init__(self, seed: int, stream: int = 0):
        self._h = lib().or_rs_new(seed, stream)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_rs_free(self._h)
            self._h = None

    def next_u64(self) -> int:
        return int(lib().or_rs_next_u64(self._h))

    def uniform(self) -> float:
        return float(lib().or_rs_uniform(self._h))

    def normal(self) -> float:
        return float(lib().or_rs_normal(self._h))

    def normal_vector(self, n: int) -> np.ndarray:
        out = np.empty(max(n, 1), dtype=np.float64)
        _check(lib().or_rs_normal_vector(self._h, n, out))
        return out

    def normal_complex_vector(self, n: int) -> np.ndarray:
        out = np.empty(2 * max(n, 1), dtype=np.float64)
        _check(lib().or_rs_normal_complex_vector(self._h, n, out))
        return out[0::2] + 1j * out[1::2]


def make_reflector(p, offset: int = 0, zero_tol: float = 0.0, rule: str = "stable"):
    """Returns (w, c, s, identity) per reflect.hpp:120-176."""
    p = np.ascontiguousarray(p, dtype=np.float64)
    n = p.size
    w = np.zeros(max(n - offset, 1), dtype=np.float64)
    c, s, ident = C.c_double(), C.c_double(), C.c_int()
    _check(lib().or_make_reflector(p, n, offset, zero_tol, SIGN_RULES[rule], w, C.byref(c), C.byref(s),
                                   C.byref(ident)))
    return w[: n - offset], c.value, s.value, bool(ident.value)


def reflector_apply(p, offset, x, rule: str = "stable"):
    p = np.ascontiguousarray(p, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    _check(lib().or_reflector_apply(p, p.size, offset, SIGN_RULES[rule], x, y))
    return y


class Operator:
    """ProbeOperator (operators.hpp:29-49) over Ginibre / Haar / GOE."""

    def __init__(self, ensemble: str, m: int = 0, n: int = 0, sigma: float = 1.0, seed: int = 1,
                 stream: int = 0, skip_reflector: bool = False, sign_rule: str = "stable", draws=None):
        """draws: optional fp64 array; the operator's matrix stream then serves
        these values (one normal_vector per probe, in order) instead of
        RandomSource(seed, stream) — the checker for device Philox runs."""
        h = C.c_void_p()
        if draws is not None:
            d = np.ascontiguousarray(draws, dtype=np.float64).reshape(-1)
            _check(lib().or_op_new_queued(ENSEMBLES[ensemble], m, n, sigma, d, d.size, C.byref(h)))
        else:
            _check(lib().or_op_new(ENSEMBLES[ensemble], m, n, sigma, seed, stream, int(skip_reflector),
                                   SIGN_RULES[sign_rule], C.byref(h)))
        self._h = h.value
        self.ensemble = ensemble

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_op_free(self._h)
            self._h = None

    @property
    def rows(self) -> int:
        return int(lib().or_op_rows(self._h))

    @property
    def cols(self) -> int:
        return int(lib().or_op_cols(self._h))

    @property
    def remaining_probes(self) -> int:
        return int(lib().or_op_remaining(self._h))

    def counts(self):
        r, l = C.c_int64(), C.c_int64()
        lib().or_op_counts(self._h, C.byref(r), C.byref(l))
        return r.value, l.value

    def chain_sizes(self):
        r, l = C.c_int64(), C.c_int64()
        lib().or_op_chain_sizes(self._h, C.byref(r), C.byref(l))
        return r.value, l.value

    def probe(self, x, side: str = "right") -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out_len = self.rows if side == "right" else self.cols
        y = np.empty(out_len, dtype=np.float64)
        _check(lib().or_op_probe(self._h, x, x.size, SIDES[side], y, out_len))
        return y

    def amp(self, beta, w, T: int, alpha: float = 1.5):
        """AMP for sparse regression (BASELINE config 4, defined in or_amp)."""
        beta = np.ascontiguousarray(beta, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        x = np.empty(self.cols, dtype=np.float64)
        mse = np.empty(max(T, 1), dtype=np.float64)
        _check(lib().or_amp(self._h, beta, w, T, alpha, x, mse))
        return x, mse[:T]

    def spiked_power(self, u, x1, T: int, theta: float = 2.0):
        """Spiked-GOE power method (BASELINE config 5, or_spiked_power)."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        x1 = np.ascontiguousarray(x1, dtype=np.float64)
        x = np.empty(self.cols, dtype=np.float64)
        ov = np.empty(max(T, 1), dtype=np.float64)
        _check(lib().or_spiked_power(self._h, u, x1, T, theta, x, ov))
        return x, ov[:T]

    def run(self, kind: str, side_rule: str, T: int, x1, x0=None, keep: bool = True) -> np.ndarray:
        x1 = np.ascontiguousarray(x1, dtype=np.float64)
        dim = x1.size
        out = np.empty(((T + 1) if keep else 1, dim), dtype=np.float64)
        x0p = None
        if x0 is not None:
            x0a = np.ascontiguousarray(x0, dtype=np.float64)
            x0p = x0a.ctypes.data_as(C.c_void_p)
        _check(lib().or_run_builtin(self._h, UPDATES[kind], SIDE_RULES[side_rule], T, x1, x0p, dim,
                                    int(keep), out.reshape(-1)))
        return out


# ------------------------------------------------ complex field
def _c_check(rc: int):
    if rc == 0:
        return
    msg = lib().or_c_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise BudgetExhausted(msg)
    raise OracleError(msg)


def _ileave(z) -> np.ndarray:
    z = np.ascontiguousarray(np.asarray(z, dtype=np.complex128).reshape(-1))
    return np.ascontiguousarray(z.view(np.float64))


def _cplx(a: np.ndarray) -> np.ndarray:
    return a.view(np.complex128).copy()


def c_make_reflector(p, offset: int = 0):
    """Complex make_reflector (reflect.hpp:142-153): (w, c, s, identity)."""
    pi = _ileave(p)
    n = pi.size // 2
    w = np.zeros(2 * max(n - offset, 1))
    c, ident = C.c_double(), C.c_int()
    s = np.zeros(2)
    _c_check(lib().or_c_make_reflector(pi, n, offset, w, C.byref(c), s, C.byref(ident)))
    return _cplx(w)[: n - offset], c.value, complex(s[0], s[1]), bool(ident.value)


def c_reflector_apply(p, offset: int, x, adjoint: bool = False) -> np.ndarray:
    pi, xi = _ileave(p), _ileave(x)
    y = np.empty_like(xi)
    _c_check(lib().or_c_reflector_apply(pi, pi.size // 2, offset, xi, int(adjoint), y))
    return _cplx(y)


def c_chain_apply(ps, x, reverse: bool = False, adjoint: bool = False) -> np.ndarray:
    """Chain of reflectors built from rows ps[k] at offsets k (reflect.hpp:193-231)."""
    ps = np.asarray(ps, dtype=np.complex128)
    k, n = ps.shape
    xi = _ileave(x)
    y = np.empty_like(xi)
    _c_check(lib().or_c_chain_apply(_ileave(ps), k, n, xi, int(reverse), int(adjoint), y))
    return _cplx(y)


class COperator:
    """GinibreOperator<complex<double>> / HaarOperator<complex<double>>."""

    def __init__(self, ensemble: str, m: int = 0, n: int = 0, sigma: float = 1.0, seed: int = 1, stream: int = 0,
                 skip_reflector: bool = False):
        h = C.c_void_p()
        _c_check(lib().or_c_op_new({"ginibre": 0, "haar": 1}[ensemble], m if ensemble == "ginibre" else n, n, sigma,
                                   seed, stream, int(skip_reflector), C.byref(h)))
        self._h, self.ensemble = h.value, ensemble
        self.rows, self.cols = (m if ensemble == "ginibre" else n), n

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_c_op_free(self._h)
            self._h = None

    @property
    def remaining_probes(self) -> int:
        return int(lib().or_c_op_remaining(self._h))

    def probe(self, x, side: str = "right") -> np.ndarray:
        xi = _ileave(x)
        out = self.rows if side == "right" else self.cols
        y = np.empty(2 * out)
        _c_check(lib().or_c_op_probe(self._h, xi, xi.size // 2, SIDES[side], y, out))
        return _cplx(y)


def complex_draws_for(seed: int, lengths, stream: int = 0) -> np.ndarray:
    """The complex draw sequence (normal_complex_vector per probe) as interleaved (re, im) fp64."""
    rs = RandomSource(seed, stream)
    return np.concatenate([rs.normal_complex_vector(int(L)) for L in lengths]).view(np.float64).copy()


def draws_for(seed: int, lengths, stream: int = 0) -> np.ndarray:
    """The exact per-probe draw sequence an operator seeded with (seed, stream)
    consumes: one normal_vector(len) per probe (ginibre.hpp:67,86; haar.hpp:48)."""
    rs = RandomSource(seed, stream)
    return np.concatenate([rs.normal_vector(int(L)) for L in lengths]) if len(lengths) else np.zeros(0)


def bench_workload(ensemble: str, m: int, n: int, sigma: float, kind: str, side_rule: str, T: int,
                   seed: int, trials: int, threads: int):
    secs, chk = C.c_double(), C.c_double()
    _check(lib().or_bench_workload(ENSEMBLES[ensemble], m, n, sigma, UPDATES[kind], SIDE_RULES[side_rule],
                                   T, seed, trials, threads, C.byref(secs), C.byref(chk)))
    return secs.value, chk.value


def bench_app(kind: str, n: int, T: int, seed: int, trials: int, threads: int):
    """Wall time of `trials` independent config-4 ('amp', m = 2n) or config-5
    ('spiked', GOE) trials on `threads` threads, from operator construction
    (or_bench_app). Returns (seconds, checksum)."""
    secs, chk = C.c_double(), C.c_double()
    _check(lib().or_bench_app({"amp": 0, "spiked": 1}[kind], n, T, seed, trials, threads, C.byref(secs),
                              C.byref(chk)))
    return secs.value, chk.value
