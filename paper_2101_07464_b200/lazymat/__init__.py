"""Drop-in mirror of the reference's ``lazymat`` Python module on the B200 path.

Same names, argument names, defaults and exceptions as the reference bindings
(/root/reference/proj/bindings/module.cpp:38-194, python/lazymat/__init__.py):

    GinibreOperator(m, n, sigma=1.0, seed=1).probe(x, side="right")
    HaarOperator(n, seed=1).probe(x, side="right"); .reconstruct()
    derive_seed(base, index); BudgetExhausted; ResourceCapExceeded

plus the B200 extensions (keyword-only): ``dtype`` ("f64"/"f32"), ``draws``
("philox" device draws, or "injected" for parity runs fed by
``push_draws``), ``capacity`` (panel width hint), ``stream``, fault flags,
``GOEOperator`` (ensembles.hpp:93-131) and device dynamics ``run(...)``.

Inputs may be numpy arrays (host, like the reference) or CUDA torch tensors
(zero-copy device path; the result is then a CUDA tensor). Everything runs
through the C-ABI of libhd_b200.so; there is no CPU fallback.

make_reflector / Reflector (module.cpp:48-66) build and apply the reflector
on the device through hd_reflector_apply. ista_curves, spectral_summary,
sample_dense_haar and two_sample_ks (module.cpp:113-194) run the reference's
application drivers on the device operators (lazymat/experiments.py).
``draws="reference"`` makes an operator draw the reference's own
RandomSource(seed) stream, i.e. the same matrix as the reference's for the
same seed; ``RandomSource`` is that generator on the host.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .. import _native as N
from .._native import BudgetExhausted, ResourceCapExceeded

__all__ = [
    "BudgetExhausted", "GinibreOperator", "HaarOperator", "GOEOperator", "Reflector", "ResourceCapExceeded",
    "RandomSource", "SubsampledHaarOperator", "USVOperator", "derive_seed", "Exchange", "shard_plan",
    "DynamicsSpec", "run_dynamics",
    "share_nccl_id", "nccl_exchange", "ista_curves", "make_reflector", "run_trials", "amp_sparse_regression", "spiked_power",
    "sample_dense_haar", "ista_trial", "spectral_trial", "power_iteration", "restarted_krylov", "soft_threshold",
    "spectral_summary", "two_sample_ks",
]

__version__ = "0.1.0"

_MASK = (1 << 64) - 1


def derive_seed(base: int, index: int) -> int:
    """random.cpp:73-76: splitmix64(base + index * golden_gamma)."""
    return int(N.lib().hd_derive_seed(int(base) & _MASK, int(index) & _MASK))


def philox_normals(seed: int, probe: int, n: int, stream: int = 0, device=None):
    """The device draw stream of ``draws="philox"`` operators: the length-n
    Gaussian draw with probe index ``probe`` of an operator built with
    (seed, stream), as a CUDA float64 tensor (Philox4x32-10, key = seed,
    counter = (row pair, probe, stream); Box-Muller on 53-bit uniforms)."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
    out = torch.empty(int(n), dtype=torch.float64, device=dev)
    N.check(N.lib().hd_philox_normals(int(seed) & _MASK, int(stream) & _MASK, int(probe), int(n),
                                      C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return out


class RandomSource:
    """The reference's RandomSource(seed, stream) (random.hpp:55-112): xoshiro256++,
    stream k = k jumps of 2^128, polar normal(), ziggurat normal_vector().
    Runs on the host inside libhd_b200.so (hd_rs_*)."""

    def __init__(self, seed: int = 1, stream: int = 0):
        h = C.c_void_p()
        N.check(N.lib().hd_rs_create(int(seed) & _MASK, int(stream) & _MASK, C.byref(h)))
        self._h = h.value

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and N is not None and N._lib is not None:
            N._lib.hd_rs_destroy(h)

    def next_u64(self) -> int:
        return int(N.lib().hd_rs_next_u64(self._h))

    def uniform(self) -> float:
        return float(N.lib().hd_rs_uniform(self._h))

    def normal(self) -> float:
        return float(N.lib().hd_rs_normal(self._h))

    def normal_vector(self, n: int) -> np.ndarray:
        out = np.empty(max(int(n), 1), dtype=np.float64)
        N.check(N.lib().hd_rs_normal_vector(self._h, int(n), out.ctypes.data_as(C.c_void_p)))
        return out

    def bernoulli_gaussian(self, n: int, rho: float, sigma_s: float) -> np.ndarray:
        """sample_bernoulli_gaussian (experiments.cpp:19-29) from this source."""
        out = np.empty(max(int(n), 1), dtype=np.float64)
        N.check(N.lib().hd_rs_bernoulli_gaussian(self._h, int(n), float(rho), float(sigma_s),
                                                 out.ctypes.data_as(C.c_void_p)))
        return out


def _side(side: str) -> int:
    if side == "right":
        return N.HD_RIGHT
    if side == "left":
        return N.HD_LEFT
    raise ValueError("side must be 'right' or 'left'")  # module.cpp:24-28


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


class Exchange:
    """The exchange of a row-sharded operator group (hd_exchange_*).

    ``Exchange.local(k)``: k virtual shards in this process, each driven from
    its own host thread (tests, one GPU). ``Exchange.nccl(uid, world, rank,
    device)``: one rank per GPU over NCCL; ``Exchange.nccl_id()`` makes the
    128-byte id on one rank (share it, e.g. with torch.distributed)."""

    def __init__(self, handle: int, size: int):
        self._h, self.size = handle, size

    @classmethod
    def local(cls, nshards: int) -> "Exchange":
        h = C.c_void_p()
        N.check(N.lib().hd_exchange_create_local(int(nshards), C.byref(h)))
        return cls(h.value, int(nshards))

    @staticmethod
    def nccl_id() -> bytes:
        buf = C.create_string_buffer(128)
        N.check(N.lib().hd_exchange_nccl_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, uid: bytes, world: int, rank: int, device: int = 0) -> "Exchange":
        if len(uid) != 128:
            raise ValueError("Exchange.nccl: uid must be the 128-byte NCCL id")
        h = C.c_void_p()
        N.check(N.lib().hd_exchange_create_nccl(C.c_char_p(uid), int(world), int(rank), int(device), C.byref(h)))
        return cls(h.value, int(world))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and N is not None and N._lib is not None:
            N._lib.hd_exchange_destroy(h)


def share_nccl_id(group=None) -> bytes:
    """Rank 0 of the torch.distributed group makes the NCCL id; every rank
    receives it (any backend, gloo included)."""
    import torch.distributed as dist

    obj = [Exchange.nccl_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def nccl_exchange(group=None, device: int = None) -> Exchange:
    """The NCCL exchange of a row-sharded operator spanning the ranks of a
    torch.distributed group (one rank per GPU, launched with torchrun)."""
    import torch
    import torch.distributed as dist

    uid = share_nccl_id(group)
    dev = torch.cuda.current_device() if device is None else int(device)
    return Exchange.nccl(uid, dist.get_world_size(group), dist.get_rank(group), dev)


def shard_plan(N_rows: int, count: int, rank: int, head_rows: int = 0):
    """Rows [begin, end) that shard `rank` of `count` owns (hd_shard_plan)."""
    b, e = C.c_int64(), C.c_int64()
    N.check(N.lib().hd_shard_plan(int(N_rows), int(count), int(rank), int(head_rows), C.byref(b), C.byref(e)))
    return b.value, e.value


class _Operator:
    _ensemble = -1

    def __init__(self, m: int, n: int, sigma: float, seed: int, *, dtype: str = "f64", draws: str = "philox",
                 capacity: int = 0, stream: int = 0, skip_reflector: bool = False, sign_rule: str = "stable",
                 device: int = 0, shard: tuple = None, exchange: "Exchange" = None):
        cfg = N.hd_config()
        cfg.ensemble = self._ensemble
        if dtype not in ("f64", "f32", "c128"):
            raise ValueError("dtype must be 'f64', 'f32' or 'c128'")
        cfg.dtype = {"f64": N.HD_F64, "f32": N.HD_F32, "c128": N.HD_C128}[dtype]
        cfg.m, cfg.n = int(m), int(n)
        cfg.sigma = float(sigma)
        cfg.seed = int(seed) & _MASK
        cfg.stream = int(stream)
        cfg.capacity = int(capacity)
        if draws not in N.DRAW_MODES:
            raise ValueError("draws must be 'philox', 'injected' or 'reference'")
        cfg.draw_mode = N.DRAW_MODES[draws]
        cfg.skip_reflector = int(bool(skip_reflector))
        cfg.sign_rule = N.SIGN_RULES[sign_rule]
        cfg.device = int(device)
        if shard is not None:  # (rank, count): this handle is one row shard of the operator
            cfg.shard_rank, cfg.shard_count = int(shard[0]), int(shard[1])
            cfg.exchange = exchange._h if exchange is not None else None
        h = C.c_void_p()
        N.check(N.lib().hd_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._exchange = exchange  # keep the group's exchange alive
        self._np_dtype = {"f64": np.float64, "f32": np.float32, "c128": np.complex128}[dtype]
        self.dtype = dtype
        self.device = int(device)
        self._ranges = [self._range(0), self._range(1)]

    def _range(self, dim: int):
        b, e = C.c_int64(), C.c_int64()
        N.check(N.lib().hd_shard_range(self._h, dim, C.byref(b), C.byref(e)))
        return b.value, e.value

    def shard_range(self, dim: str = "cols"):
        """Global rows [begin, end) of x (dim 'cols', the right-probe input) or
        of y (dim 'rows') that this handle owns; the whole range when unsharded."""
        return self._ranges[0 if dim == "cols" else 1]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                N.lib().hd_destroy(h)
            except Exception:
                pass
            self._h = None

    # ProbeOperator interface (operators.hpp:29-49)
    @property
    def rows(self) -> int:
        r, c = C.c_int64(), C.c_int64()
        N.check(N.lib().hd_shape(self._h, C.byref(r), C.byref(c)))
        return r.value

    @property
    def cols(self) -> int:
        r, c = C.c_int64(), C.c_int64()
        N.check(N.lib().hd_shape(self._h, C.byref(r), C.byref(c)))
        return c.value

    @property
    def remaining_probes(self) -> int:
        v = C.c_int64()
        N.check(N.lib().hd_remaining(self._h, C.byref(v)))
        return v.value

    def probe_counts(self):
        r, l = C.c_int64(), C.c_int64()
        N.check(N.lib().hd_counts(self._h, C.byref(r), C.byref(l)))
        return r.value, l.value

    def chain_sizes(self):
        r, l = C.c_int64(), C.c_int64()
        N.check(N.lib().hd_chain_sizes(self._h, C.byref(r), C.byref(l)))
        return r.value, l.value

    def _out_len(self, side: int) -> int:  # this shard's rows of the output
        b, e = self._ranges[1] if side == N.HD_RIGHT else self._ranges[0]
        return e - b

    def probe(self, x, side: str = "right"):
        """Q @ x ('right') or Q.T @ x ('left'), revealing only the randomness
        the probe requires (module.cpp:79-87)."""
        s = _side(side)
        if _is_torch_cuda(x):
            import torch

            xt = x.contiguous()
            want = {"f64": torch.float64, "f32": torch.float32, "c128": torch.complex128}[self.dtype]
            if xt.dtype != want:
                xt = xt.to(want)
            out = torch.empty(self._out_len(s if self._ensemble != N.HD_GOE else N.HD_RIGHT), dtype=want,
                              device=xt.device)
            stream = torch.cuda.current_stream(xt.device).cuda_stream
            N.check(N.lib().hd_probe(self._h, C.c_void_p(xt.data_ptr()), xt.numel(), C.c_void_p(out.data_ptr()),
                                     out.numel(), s, 1, C.c_void_p(stream)))
            return out
        xa = np.ascontiguousarray(np.asarray(x, dtype=self._np_dtype).reshape(-1))
        out_len = self._out_len(s if self._ensemble != N.HD_GOE else N.HD_RIGHT)
        y = np.empty(out_len, dtype=self._np_dtype)
        N.check(N.lib().hd_probe(self._h, xa.ctypes.data_as(C.c_void_p), xa.size, y.ctypes.data_as(C.c_void_p),
                                 y.size, s, 0, None))
        return y

    # parity mode
    def push_draws(self, g) -> None:
        """Queue the next probes' draws (injected mode): fp64 values, or for a
        complex operator complex values (one normal_complex_vector per probe)."""
        if np.iscomplexobj(g):
            ga = np.ascontiguousarray(np.asarray(g, dtype=np.complex128).reshape(-1)).view(np.float64)
        else:
            ga = np.ascontiguousarray(np.asarray(g, dtype=np.float64).reshape(-1))
        N.check(N.lib().hd_push_draws(self._h, ga.ctypes.data_as(C.c_void_p), ga.size, 0))

    def reset(self) -> None:
        N.check(N.lib().hd_reset(self._h))

    # device dynamics (run_dynamics, dynamics.hpp:42-76, built-in maps)
    def run(self, x1, iterations: int, update: str = "normalize", sides: str = "alternate", x0=None,
            keep_trajectory: bool = False, use_graph: bool = False, out=None):
        """run_dynamics with a built-in update map on the device; returns x_{T+1}
        (or the trajectory). A fresh Haar operator on a fixed side takes the
        two-pass sequence (each panel read once per probe)."""
        a = N.hd_run_args()
        a.update = N.UPDATES[update]
        a.side_rule = N.SIDE_RULES[sides]
        a.iterations = int(iterations)
        a.use_graph = int(bool(use_graph))
        if _is_torch_cuda(x1):
            import torch

            want = torch.float64 if self.dtype == "f64" else torch.float32
            x1t = x1.contiguous().to(want)
            a.x1 = x1t.data_ptr()
            x0t = None
            if x0 is not None:
                x0t = x0.contiguous().to(want)
                a.x0 = x0t.data_ptr()
            a.on_device = 1
            fdim = self._final_dim(iterations, sides, x1t.numel())
            fin = torch.empty(fdim, dtype=want, device=x1t.device)
            a.final_out = fin.data_ptr()
            traj = None
            if keep_trajectory:
                traj = torch.empty((iterations + 1, x1t.numel()), dtype=want, device=x1t.device)
                a.traj = traj.data_ptr()
            a.stream = torch.cuda.current_stream(x1t.device).cuda_stream
            N.check(N.lib().hd_run(self._h, C.byref(a)))
            return traj if keep_trajectory else fin
        x1a = np.ascontiguousarray(np.asarray(x1, dtype=self._np_dtype).reshape(-1))
        a.x1 = x1a.ctypes.data
        x0a = None
        if x0 is not None:
            x0a = np.ascontiguousarray(np.asarray(x0, dtype=self._np_dtype).reshape(-1))
            a.x0 = x0a.ctypes.data
        fdim = self._final_dim(iterations, sides, x1a.size)
        if out is not None:  # caller's host buffer (e.g. pinned) for x_{T+1}
            if out.dtype != self._np_dtype or out.size != fdim or not out.flags.c_contiguous:
                raise ValueError("run: out must be a contiguous host array of the final iterate's size and dtype")
            fin = out
        else:
            fin = np.empty(fdim, dtype=self._np_dtype)
        a.final_out = fin.ctypes.data
        traj = None
        if keep_trajectory:
            traj = np.empty((iterations + 1, x1a.size), dtype=self._np_dtype)
            a.traj = traj.ctypes.data
        N.check(N.lib().hd_run(self._h, C.byref(a)))
        return traj if keep_trajectory else fin

    # ---- asynchronous runs (many handles on their own streams: batched trials)
    def reseed(self, seed: int) -> None:
        """Fresh state with a new seed (Philox key) without host sync."""
        N.check(N.lib().hd_reseed(self._h, int(seed) & _MASK))

    def run_async(self, x1, iterations: int, out, update: str = "normalize", sides: str = "alternate", x0=None,
                  use_graph: bool = True) -> None:
        """Enqueue a whole run on the operator's own stream, ordered after the
        work already queued on torch's current stream; `x1` / `x0` / `out` are
        CUDA tensors of the operator's dtype that must stay alive until wait()."""
        import torch

        a = N.hd_run_args()
        a.update = N.UPDATES[update]
        a.side_rule = N.SIDE_RULES[sides]
        a.iterations = int(iterations)
        a.use_graph = int(bool(use_graph))
        a.x1 = x1.data_ptr()
        if x0 is not None:
            a.x0 = x0.data_ptr()
        a.on_device = 1
        a.final_out = out.data_ptr()
        a.stream = torch.cuda.current_stream(x1.device).cuda_stream
        self._inflight = (x1, x0, out)
        N.check(N.lib().hd_run_async(self._h, C.byref(a)))

    def wait(self) -> None:
        try:
            N.check(N.lib().hd_wait(self._h))
        finally:
            self._inflight = None

    def _final_dim(self, iterations: int, sides: str, dim1: int) -> int:
        if iterations == 0:
            return dim1
        if self._ensemble == N.HD_GOE:
            return self.rows
        last = iterations
        right = sides == "right" or (sides == "alternate" and last % 2 == 1)
        return self.rows if right else self.cols

    # instrumentation
    def set_profiling(self, on: bool = True) -> None:
        N.check(N.lib().hd_set_profiling(self._h, int(on)))

    def kernel_stats(self):
        cnt = C.c_int32()
        N.check(N.lib().hd_get_stats(self._h, None, 0, C.byref(cnt)))
        arr = (N.hd_kernel_stats * max(cnt.value, 1))()
        N.check(N.lib().hd_get_stats(self._h, arr, cnt.value, C.byref(cnt)))
        return {arr[i].name.decode(): {"launches": arr[i].launches, "ms": arr[i].ms, "alg_bytes": arr[i].alg_bytes}
                for i in range(cnt.value)}

    def reset_stats(self) -> None:
        N.check(N.lib().hd_reset_stats(self._h))

    def launch_count(self) -> int:
        v = C.c_int64()
        N.check(N.lib().hd_launch_count(self._h, C.byref(v)))
        return v.value


class GinibreOperator(_Operator):
    """Lazy m x n Gaussian matrix, entries N(0, sigma^2) (ginibre.hpp:26-118)."""

    _ensemble = N.HD_GINIBRE

    def __init__(self, m: int, n: int, sigma: float = 1.0, seed: int = 1, **kw):
        super().__init__(m, n, sigma, seed, **kw)


class HaarOperator(_Operator):
    """Lazy n x n Haar-orthogonal matrix (haar.hpp:21-76)."""

    _ensemble = N.HD_HAAR

    def __init__(self, n: int, seed: int = 1, **kw):
        super().__init__(n, n, 1.0, seed, **kw)

    def reconstruct(self):
        """Materialise Q by right-probing the natural basis; consumes the whole
        budget (haar.hpp:80-91, module.cpp:105-111)."""
        r, _ = self.probe_counts()
        if r != 0:
            raise ValueError("reconstruct: operator already probed")
        n = self.rows
        q = np.empty((n, n), dtype=self._np_dtype)
        for j in range(n):
            e = np.zeros(n, dtype=self._np_dtype)
            e[j] = 1.0
            q[:, j] = self.probe(e, "right")
        return q


class GOEOperator(_Operator):
    """Lazy symmetric Gaussian matrix: (inner right + inner left probe)/sqrt(2)
    over a square Ginibre of entry std ``sigma`` (ensembles.hpp:93-131)."""

    _ensemble = N.HD_GOE

    def __init__(self, n: int, seed: int = 1, sigma: float = 1.0, **kw):
        super().__init__(n, n, sigma, seed, **kw)


class Reflector:
    """Generalised Householder reflector H_k(p) (reflect.hpp:47-104), built and
    applied on the device; exposes dim / offset / is_identity / apply like the
    reference binding (module.cpp:48-57)."""

    def __init__(self, p: np.ndarray, offset: int, info):
        self._p = p
        self._offset = int(offset)
        self._c, self._s, ident = info
        self._identity = bool(ident)

    @property
    def dim(self) -> int:
        return int(self._p.size)

    @property
    def offset(self) -> int:
        return self._offset

    @property
    def is_identity(self) -> bool:
        return self._identity

    def apply(self, x, adjoint: bool = False):
        # real reflectors are self-adjoint (reflect.hpp:80)
        xa = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
        if xa.size != self.dim:
            raise ValueError("Reflector::apply: dimension mismatch")
        y = np.empty_like(xa)
        N.check(N.lib().hd_reflector_apply(self._p.ctypes.data_as(C.c_void_p), self.dim, self._offset, 0.0, 0,
                                           xa.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), 1, 0, None))
        return y


def batch_run(ops, x1, out, seeds, iterations: int, update: str = "normalize", sides: str = "alternate",
              stream=None) -> None:
    """hd_batch_run: operators of one shape run the same dynamics in lockstep
    from fresh states (seed per operator), every kernel launch issued once for
    all of them (include/hd.h). x1 / out: (len(ops), dim) CUDA tensors of the
    operators' dtype; asynchronous on `stream` (default: torch's current)."""
    import torch

    B = len(ops)
    a = N.hd_run_args()
    a.update = N.UPDATES[update]
    a.side_rule = N.SIDE_RULES[sides]
    a.iterations = int(iterations)
    a.on_device = 1
    a.use_graph = 1
    st = stream if stream is not None else torch.cuda.current_stream(x1.device)
    a.stream = st.cuda_stream
    handles = (C.c_void_p * B)(*[op._h for op in ops])
    items = (N.hd_batch_item * B)()
    for b in range(B):
        items[b].x1 = x1[b].data_ptr()
        items[b].out = out[b].data_ptr()
        items[b].seed = int(seeds[b]) & _MASK
    N.check(N.lib().hd_batch_run(handles, B, C.byref(a), items))


def run_trials(ensemble: str, trials: int, n: int, T: int, *, m: int = None, sigma: float = None, seed: int = 1,
               dtype: str = "f64", update: str = "normalize", sides: str = "alternate", concurrency: int = 16,
               x1=None, first_trial: int = 0, device: int = 0, return_ops: bool = False, batch: int = 1,
               ops=None):
    """Independent HD trials (BASELINE config 3: trial b uses seed + b). Keeps
    `concurrency` device operators in flight, each on its own CUDA stream
    replaying one captured run graph (reseeded per trial), so the latency of
    one trial's probe sequence overlaps the HBM streaming of the others.
    batch > 1: `concurrency` groups of `batch` operators, each group's trials
    sharing every kernel launch (batch_run / hd_batch_run) — the separate-graph
    mode is bound by the kernel-dispatch rate at config-3 sizes. A batched
    launch gives each operator floor(SMs / batch) CTAs, so `batch` should
    divide the SM count (148 = 4 x 37: batch 37 / 74 / 148); batch = 0 picks
    half the SM count (config 3: 1.62 s against 1.71 s at batch 32).
    Returns x_{T+1} of every trial as a (trials, dim) CUDA tensor.
    x1: optional (trials, dim) CUDA tensor; default N(0, I) per trial.
    ops: the operators a previous call returned (return_ops=True) with the same
    arguments, reused instead of allocating new ones."""
    import torch

    if batch == 0:
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        batch = max(1, min(trials, sms // 2))
    if batch > 1:
        return _run_trials_batched(ensemble, trials, n, T, m=m, sigma=sigma, seed=seed, dtype=dtype, update=update,
                                   sides=sides, groups=concurrency, batch=batch, x1=x1, first_trial=first_trial,
                                   device=device, return_ops=return_ops, pool=ops)

    m = n if m is None else m
    if sigma is None:
        sigma = 1.0 / float(n) ** 0.5
    tdt = torch.float64 if dtype == "f64" else torch.float32
    dev = torch.device("cuda", device)
    make = {
        "ginibre": lambda: GinibreOperator(m, n, sigma, seed, dtype=dtype, capacity=T, device=device),
        "haar": lambda: HaarOperator(n, seed, dtype=dtype, capacity=T, device=device),
        "goe": lambda: GOEOperator(n, seed, sigma=sigma, dtype=dtype, capacity=T, device=device),
    }[ensemble]
    if ops is None:
        ops = [make() for _ in range(max(1, min(concurrency, trials)))]
    dim1 = n if (ensemble != "ginibre" or sides != "left") else m
    fdim = ops[0]._final_dim(T, sides, dim1)
    if x1 is None:
        x1 = torch.empty((trials, dim1), dtype=tdt, device=dev)
        for b in range(trials):
            g = torch.Generator(device=dev).manual_seed(seed + first_trial + b)
            x1[b] = torch.randn(dim1, dtype=tdt, device=dev, generator=g)
    out = torch.empty((trials, fdim), dtype=tdt, device=dev)
    torch.cuda.synchronize(dev)
    nxt = 0
    busy = []
    for op in ops:
        if nxt >= trials:
            break
        op.reseed(seed + first_trial + nxt)
        op.run_async(x1[nxt], T, out[nxt], update=update, sides=sides)
        busy.append(op)
        nxt += 1
    while busy:
        op = busy.pop(0)
        op.wait()
        if nxt < trials:
            op.reseed(seed + first_trial + nxt)
            op.run_async(x1[nxt], T, out[nxt], update=update, sides=sides)
            busy.append(op)
            nxt += 1
    return (out, ops) if return_ops else out


def _run_trials_batched(ensemble, trials, n, T, *, m, sigma, seed, dtype, update, sides, groups, batch, x1,
                        first_trial, device, return_ops, pool):
    import torch

    m = n if m is None else m
    if sigma is None:
        sigma = 1.0 / float(n) ** 0.5
    tdt = torch.float64 if dtype == "f64" else torch.float32
    dev = torch.device("cuda", device)
    make = {
        "ginibre": lambda: GinibreOperator(m, n, sigma, seed, dtype=dtype, capacity=T, device=device),
        "haar": lambda: HaarOperator(n, seed, dtype=dtype, capacity=T, device=device),
        "goe": lambda: GOEOperator(n, seed, sigma=sigma, dtype=dtype, capacity=T, device=device),
    }[ensemble]
    batch = max(1, min(batch, trials))
    ngroups = max(1, min(groups, -(-trials // batch)))
    tail = trials % batch
    if pool is not None:  # (groups, tail operators, streams) of a previous call
        grp, tail_ops, streams = pool
    else:
        grp = [[make() for _ in range(batch)] for _ in range(ngroups)]
        tail_ops = [make() for _ in range(tail)] if tail else []  # a ragged last chunk: its own group
        streams = [torch.cuda.Stream(device=dev) for _ in range(ngroups)]
    dim1 = n if (ensemble != "ginibre" or sides != "left") else m
    fdim = grp[0][0]._final_dim(T, sides, dim1)
    if x1 is None:
        x1 = torch.empty((trials, dim1), dtype=tdt, device=dev)
        for b in range(trials):
            g = torch.Generator(device=dev).manual_seed(seed + first_trial + b)
            x1[b] = torch.randn(dim1, dtype=tdt, device=dev, generator=g)
    out = torch.empty((trials, fdim), dtype=tdt, device=dev)
    main = torch.cuda.current_stream(dev)
    for st in streams:
        st.wait_stream(main)
    chunk = 0
    for b0 in range(0, trials - tail, batch):
        gi = chunk % ngroups
        with torch.cuda.stream(streams[gi]):
            seeds = [seed + first_trial + b0 + j for j in range(batch)]
            batch_run(grp[gi], x1[b0:b0 + batch], out[b0:b0 + batch], seeds, T, update, sides, stream=streams[gi])
        chunk += 1
    if tail:
        b0 = trials - tail
        with torch.cuda.stream(streams[0]):
            seeds = [seed + first_trial + b0 + j for j in range(tail)]
            batch_run(tail_ops, x1[b0:], out[b0:], seeds, T, update, sides, stream=streams[0])
    for st in streams:
        main.wait_stream(st)
    return (out, (grp, tail_ops, streams)) if return_ops else out


class DynamicsSpec:
    """DynamicsSpec (dynamics.hpp:21-32): T iterations of
    x_{t+1} = update(t, y_t, history) with y_t = M_t x_t, M_t chosen by
    side_of(t) ('right' / 'left'); `initial` holds the d + 1 starting vectors
    newest first; `observer(t, y_t, x_{t+1})` sees the run stream by."""

    def __init__(self, iterations: int = 0, history_depth: int = 0, initial=None, side_of=None, update=None,
                 observer=None, keep_trajectory: bool = True):
        self.iterations, self.history_depth = int(iterations), int(history_depth)
        self.initial = list(initial) if initial is not None else []
        self.side_of, self.update, self.observer = side_of, update, observer
        self.keep_trajectory = bool(keep_trajectory)


def _all_finite(v) -> bool:
    if _is_torch_cuda(v):
        import torch

        return bool(torch.isfinite(v).all())
    return bool(np.all(np.isfinite(np.asarray(v))))


def run_dynamics(op, spec: DynamicsSpec) -> list:
    """run_dynamics (dynamics.hpp:42-76) over a device operator with user
    callbacks: the same validation messages, the history window newest first,
    the non-finite abort and the observer. Vectors are numpy (host) or CUDA
    tensors (device-resident); every probe runs on the GPU. Returns the
    iterates x_1..x_{T+1} (or [x_{T+1}] when keep_trajectory is off)."""
    if spec.iterations < 0:
        raise ValueError("run_dynamics: negative iteration count")
    if spec.history_depth < 0:
        raise ValueError("run_dynamics: negative history depth")
    if len(spec.initial) != spec.history_depth + 1:
        raise ValueError("run_dynamics: initial history must hold d + 1 vectors")
    if spec.side_of is None:
        raise ValueError("run_dynamics: no side schedule")
    if spec.update is None:
        raise ValueError("run_dynamics: no update map")
    if spec.iterations > op.remaining_probes:
        raise ValueError("run_dynamics: iteration count exceeds the operator's probe budget")
    history = list(spec.initial)
    traj = [history[0]] if spec.keep_trajectory else []
    for t in range(1, spec.iterations + 1):
        y = op.probe(history[0], spec.side_of(t))
        nxt = spec.update(t, y, history)
        if not _all_finite(nxt):
            raise RuntimeError(f"run_dynamics: non-finite iterate at step {t}")
        if spec.observer is not None:
            spec.observer(t, y, nxt)
        history.insert(0, nxt)
        history.pop()
        if spec.keep_trajectory:
            traj.append(nxt)
    if not spec.keep_trajectory:
        traj.append(history[0])
    return traj


def _app_io(op, vecs, dims):
    """Inputs of a device app run: (pointers, keep-alive, on_device, stream,
    torch module or None). CUDA tensors stay on the device; anything else is a
    contiguous host array of the operator's dtype."""
    if any(_is_torch_cuda(v) for v in vecs):
        import torch

        want = torch.float64 if op.dtype == "f64" else torch.float32
        dev = next(v.device for v in vecs if _is_torch_cuda(v))
        ts = [torch.as_tensor(v, device=dev).to(want).contiguous().reshape(-1) for v in vecs]
        for t, d in zip(ts, dims):
            if t.numel() != d:
                raise ValueError("run_dynamics: initial history must hold d + 1 vectors")
        return [t.data_ptr() for t in ts], ts, 1, torch.cuda.current_stream(dev).cuda_stream, torch
    arrs = [np.ascontiguousarray(np.asarray(v, dtype=op._np_dtype).reshape(-1)) for v in vecs]
    for a, d in zip(arrs, dims):
        if a.size != d:
            raise ValueError("run_dynamics: initial history must hold d + 1 vectors")
    return [a.ctypes.data for a in arrs], arrs, 0, None, None


def amp_sparse_regression(op, beta, w, T: int, alpha: float = 1.5, use_graph: bool = True, x_out=None,
                          mse_out=None):
    """AMP for sparse regression on a device Ginibre design A (BASELINE config 4;
    not in the reference — the same recurrence is or_amp in the test oracle):
    y = A beta + w (one right probe, experiments.cpp:80-82), x^0 = 0, z^0 = y,
      x^{t+1} = soft(x^t + A^T z^t, alpha ||z^t|| / sqrt(m))   (soft: experiments.cpp:31-39)
      z^{t+1} = y - A x^{t+1} + (nnz(x^{t+1}) / n / delta) z^t,  delta = m / n.
    The whole run (2T + 1 probes, the update maps fused into each output pass)
    is one device-resident CUDA graph (hd_run_amp). CUDA tensors in -> CUDA
    tensors out; host arrays in -> numpy out (optionally into the caller's
    host buffers x_out / mse_out, e.g. pinned). Returns (x^T, mse curve
    ||x^t - beta||^2 / n)."""
    m, n = op.rows, op.cols
    ptrs, keep, on_dev, stream, torch = _app_io(op, [beta, w], [n, m])
    a = N.hd_amp_args()
    a.beta, a.w = ptrs
    a.iterations, a.alpha = int(T), float(alpha)
    a.on_device, a.use_graph = on_dev, int(bool(use_graph))
    a.stream = stream
    if torch is not None:
        x = torch.empty(n, dtype=keep[0].dtype, device=keep[0].device) if x_out is None else x_out
        mse = torch.empty(int(T), dtype=torch.float64, device=keep[0].device) if mse_out is None else mse_out
    else:
        x = np.empty(n, dtype=op._np_dtype) if x_out is None else x_out
        mse = np.empty(int(T), dtype=np.float64) if mse_out is None else mse_out
    a.x_out = x.data_ptr() if torch is not None else x.ctypes.data
    a.mse_out = (mse.data_ptr() if torch is not None else mse.ctypes.data) if int(T) > 0 else None
    N.check(N.lib().hd_run_amp(op._h, C.byref(a)))
    return x, mse


def spiked_power(op, u, x1, T: int, theta: float = 2.0, use_graph: bool = True, x_out=None, overlap_out=None):
    """Power method on Q + theta u u^T with Q a device GOE operator (BASELINE
    config 5): x_{t+1} = (Q x_t + theta <u, x_t> u) / ||.||. One device-resident
    CUDA graph (hd_run_spiked). Returns (x_{T+1}, overlaps <u, x_{t+1}>)."""
    lo, hi = op.shard_range("cols")  # a row shard takes and returns its own rows
    n = hi - lo
    ptrs, keep, on_dev, stream, torch = _app_io(op, [u, x1], [n, n])
    a = N.hd_spiked_args()
    a.u, a.x1 = ptrs
    a.iterations, a.theta = int(T), float(theta)
    a.on_device, a.use_graph = on_dev, int(bool(use_graph))
    a.stream = stream
    if torch is not None:
        x = torch.empty(n, dtype=keep[0].dtype, device=keep[0].device) if x_out is None else x_out
        ov = torch.empty(int(T), dtype=torch.float64, device=keep[0].device) if overlap_out is None else overlap_out
    else:
        x = np.empty(n, dtype=op._np_dtype) if x_out is None else x_out
        ov = np.empty(int(T), dtype=np.float64) if overlap_out is None else overlap_out
    a.x_out = x.data_ptr() if torch is not None else x.ctypes.data
    a.overlap_out = (ov.data_ptr() if torch is not None else ov.ctypes.data) if int(T) > 0 else None
    N.check(N.lib().hd_run_spiked(op._h, C.byref(a)))
    return x, ov


def make_reflector(p, offset: int = 0):
    """Orthogonal reflector sending p[offset:] to +||p[offset:]|| e_1 and fixing
    the first `offset` coordinates (reflect.hpp:120-176, module.cpp:59-66)."""
    pa = np.ascontiguousarray(np.asarray(p, dtype=np.float64).reshape(-1)).copy()
    info = (C.c_double * 3)()
    N.check(N.lib().hd_reflector_apply(pa.ctypes.data_as(C.c_void_p), pa.size, int(offset), 0.0, 0, None, None, 0, 0,
                                       info))
    return Reflector(pa, offset, (info[0], info[1], info[2]))


def _xp_zeros(like, n):
    if _is_torch_cuda(like):
        import torch

        return torch.zeros(n, dtype=like.dtype, device=like.device)
    return np.zeros(n, dtype=np.asarray(like).dtype)


class USVOperator:
    """Q = U S V over two square lazy factors and a fixed rectangular diagonal
    (ensembles.hpp:133-180); one probe of each device factor per probe."""

    def __init__(self, u, v, singular_values):
        if u is None or v is None:
            raise ValueError("USVOperator: null factor")
        if u.rows != u.cols or v.rows != v.cols:
            raise ValueError("USVOperator: factors must be square")
        sv = np.asarray(singular_values, dtype=np.float64).reshape(-1)
        if sv.size != min(u.rows, v.cols):
            raise ValueError("USVOperator: need min(rows, cols) singular values")
        self.u, self.v, self._sv = u, v, sv

    @property
    def rows(self):
        return self.u.rows

    @property
    def cols(self):
        return self.v.cols

    @property
    def remaining_probes(self):
        return min(self.u.remaining_probes, self.v.remaining_probes)

    @property
    def singular_values(self):
        return self._sv.copy()

    def probe(self, x, side: str = "right"):
        s_ = _side(side)
        want = self.cols if s_ == N.HD_RIGHT else self.rows
        if (x.numel() if _is_torch_cuda(x) else np.asarray(x).size) != want:
            raise ValueError("probe: input dimension mismatch")
        if self.remaining_probes == 0:
            raise BudgetExhausted("USVOperator: factor budget spent")
        k = self._sv.size
        if s_ == N.HD_RIGHT:
            t = self.v.probe(x, "right")
            s = _xp_zeros(t, self.rows)
            s[:k] = self._sv_like(t)[:k] * t[:k]
            return self.u.probe(s, "right")
        t = self.u.probe(x, "left")
        s = _xp_zeros(t, self.cols)
        s[:k] = self._sv_like(t)[:k] * t[:k]
        return self.v.probe(s, "left")

    def _sv_like(self, t):
        if _is_torch_cuda(t):
            import torch

            return torch.as_tensor(self._sv, dtype=t.dtype, device=t.device)
        return self._sv.astype(t.dtype)


class SubsampledHaarOperator:
    """A = [I 0] Q: the first `rows` coordinates of a square lazy operator
    (ensembles.hpp:182-215)."""

    def __init__(self, q, rows: int):
        if q is None:
            raise ValueError("SubsampledHaarOperator: null inner operator")
        if q.rows != q.cols:
            raise ValueError("SubsampledHaarOperator: inner operator must be square")
        if not (1 <= rows <= q.rows):
            raise ValueError("SubsampledHaarOperator: need 1 <= rows <= inner dim")
        self.q, self._rows = q, int(rows)

    @property
    def rows(self):
        return self._rows

    @property
    def cols(self):
        return self.q.cols

    @property
    def remaining_probes(self):
        return self.q.remaining_probes

    def probe(self, x, side: str = "right"):
        s_ = _side(side)
        want = self.cols if s_ == N.HD_RIGHT else self.rows
        if (x.numel() if _is_torch_cuda(x) else np.asarray(x).size) != want:
            raise ValueError("probe: input dimension mismatch")
        if s_ == N.HD_RIGHT:
            return self.q.probe(x, "right")[: self._rows]
        padded = _xp_zeros(x, self.cols)
        padded[: self._rows] = x
        return self.q.probe(padded, "left")


# Application drivers and the dense direct backend (experiments.cpp,
# eigensolve.hpp, ensembles.hpp:40-91, stats.cpp) on the device operators.
from . import verify  # noqa: E402,F401  (verification harness, lazymat.verify)
from .experiments import (  # noqa: E402
    ista_curves, ista_trial, power_iteration, restarted_krylov, sample_dense_haar, soft_threshold,
    spectral_summary, spectral_trial, two_sample_ks,
)
