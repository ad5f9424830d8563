"""Stream ordering of the C-ABI entry points: a device input produced on the
caller's stream (torch's current stream — the legacy NULL stream by default,
or a side stream) must be complete before the handle's own non-blocking
stream reads it. The producer is held back with a device-side sleep, so an
unordered read would see the stale contents."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SLEEP = 20_000_000  # cycles (~10 ms)


def _delayed_copy(torch, dst, src):
    torch.cuda._sleep(SLEEP)
    dst.copy_(src)


@pytest.mark.parametrize("side_stream", [False, True])
def test_probe_waits_for_callers_stream(orc, lm, side_stream):
    import torch

    n = 1 << 20
    src = torch.from_numpy(orc.RandomSource(3).normal_vector(n)).cuda()
    want = lm.HaarOperator(n, seed=4).probe(src.cpu().numpy(), "right")
    op = lm.HaarOperator(n, seed=4)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    s = torch.cuda.Stream() if side_stream else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        _delayed_copy(torch, x, src)
        y = op.probe(x, "right")
    s.synchronize()
    assert np.linalg.norm(y.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want)


def test_run_waits_for_callers_stream(orc, lm):
    import torch

    n, T = 1 << 18, 6
    src = torch.from_numpy(orc.RandomSource(5).normal_vector(n)).cuda()
    want = lm.GinibreOperator(n, n, n ** -0.5, 6).run(src.cpu().numpy(), T, update="normalize")
    op = lm.GinibreOperator(n, n, n ** -0.5, 6)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    _delayed_copy(torch, x, src)
    got = op.run(x, T, update="normalize")
    assert np.linalg.norm(got.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want)


def test_run_async_waits_for_legacy_stream(orc, lm):
    import torch

    n, T = 1 << 18, 6
    src = torch.from_numpy(orc.RandomSource(7).normal_vector(n)).cuda()
    want = lm.HaarOperator(n, seed=8).run(src.cpu().numpy(), T, update="normalize", sides="right")
    op = lm.HaarOperator(n, seed=8)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    _delayed_copy(torch, x, src)
    op.run_async(x, T, out, update="normalize", sides="right")
    op.wait()
    assert np.linalg.norm(out.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want)
