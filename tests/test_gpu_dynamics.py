"""User dynamics callbacks (dynamics.hpp:21-76; north star: "the user
dynamics callback") on the device operators: lazymat.run_dynamics with
Python update maps over CUDA tensors, and the C-ABI hd_run_callback driven
through a C callback that enqueues its update on the stream it is handed."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


def test_user_callbacks_reproduce_the_reference_runs(orc, lm):
    import torch

    n, T, seed = 4000, 25, 13
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    want = orc.Operator("haar", n=n, seed=seed).run("tanh_mix", "right", T, x1, keep=True)
    op = lm.HaarOperator(n, seed=seed, draws="reference")
    xs = torch.from_numpy(x1).cuda()
    seen = []
    spec = lm.DynamicsSpec(iterations=T, history_depth=1, initial=[xs, torch.zeros_like(xs)],
                           side_of=lambda t: "right",
                           update=lambda t, y, h: torch.tanh(2.0 * y) + 0.1 * h[1],
                           observer=lambda t, y, nxt: seen.append(t))
    traj = lm.run_dynamics(op, spec)
    assert len(traj) == T + 1 and seen == list(range(1, T + 1))
    for t in range(T + 1):
        assert rel(traj[t].cpu().numpy(), want[t]) < 1e-9, t
    # config 1 style: normalised alternating power iteration on a Ginibre operator
    m = 3000
    want = orc.Operator("ginibre", m=m, n=m, sigma=m ** -0.5, seed=seed).run("normalize", "alternate", T, x1[:m],
                                                                            keep=False)
    op = lm.GinibreOperator(m, m, m ** -0.5, seed, draws="reference")
    spec = lm.DynamicsSpec(T, 0, [torch.from_numpy(x1[:m]).cuda()], lambda t: "right" if t % 2 else "left",
                           lambda t, y, h: y / torch.linalg.vector_norm(y), keep_trajectory=False)
    out = lm.run_dynamics(op, spec)
    assert len(out) == 1 and rel(out[0].cpu().numpy(), want[0]) < 1e-9


def test_run_dynamics_validation_and_abort(lm):
    op = lm.HaarOperator(10, seed=1)
    x = np.ones(10)
    upd = lambda t, y, h: y  # noqa: E731
    for spec, msg in [(lm.DynamicsSpec(-1, 0, [x], lambda t: "right", upd), "negative iteration count"),
                      (lm.DynamicsSpec(1, -1, [], lambda t: "right", upd), "negative history depth"),
                      (lm.DynamicsSpec(1, 1, [x], lambda t: "right", upd), "d \\+ 1 vectors"),
                      (lm.DynamicsSpec(1, 0, [x], None, upd), "no side schedule"),
                      (lm.DynamicsSpec(1, 0, [x], lambda t: "right", None), "no update map"),
                      (lm.DynamicsSpec(11, 0, [x], lambda t: "right", upd), "exceeds the operator's probe budget")]:
        with pytest.raises(ValueError, match=msg):
            lm.run_dynamics(op, spec)
    spec = lm.DynamicsSpec(5, 0, [x], lambda t: "right", lambda t, y, h: y * (np.nan if t == 3 else 1.0))
    with pytest.raises(RuntimeError, match="non-finite iterate at step 3"):
        lm.run_dynamics(op, spec)


def test_cabi_run_callback_identity_map(orc, lm):
    # hd_run_callback (the C-ABI's DynamicsSpec::update): a C callback that
    # copies y into next on the given stream (identity map x_{t+1} = y_t)
    from paper_2101_07464_b200 import _native as N

    cudart = C.CDLL("/usr/local/cuda/lib64/libcudart.so")
    cudart.cudaMemcpyAsync.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
    n, T, seed = 3001, 16, 21
    x1 = orc.RandomSource(seed, 1).normal_vector(n)
    want = orc.Operator("haar", n=n, seed=seed).run("identity", "alternate", T, x1, keep=False)[0]
    op = lm.HaarOperator(n, seed=seed, draws="reference")
    import torch

    xin = torch.from_numpy(x1).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    calls = []

    @N.SIDE_FN
    def side_of(user, t):
        return N.HD_RIGHT if t % 2 == 1 else N.HD_LEFT

    @N.UPDATE_FN
    def update(user, t, y, history, depth, nxt, dim, stream):
        calls.append(int(t))
        return cudart.cudaMemcpyAsync(nxt, y, dim * 8, 3, stream)  # device-to-device

    init = (C.c_void_p * 1)(xin.data_ptr())
    N.check(N.lib().hd_run_callback(op._h, T, 0, init, side_of, update, None, C.c_void_p(out.data_ptr())))
    assert calls == list(range(1, T + 1))
    assert rel(out.cpu().numpy(), want) < 1e-9
