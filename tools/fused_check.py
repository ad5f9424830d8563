"""Two-pass Haar runs against the three-pass sequence:
same operator, same draws, HD_FUSED=1 vs HD_FUSED=0 (read at operator
creation), plus timing of each at the config-2 shape. Prints JSON lines."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2101_07464_b200 import lazymat


def make(n, fused, dtype="f64", **kw):
    os.environ["HD_FUSED"] = "1" if fused else "0"
    op = lazymat.HaarOperator(n, seed=3, dtype=dtype, capacity=kw.pop("capacity", 128), **kw)
    os.environ.pop("HD_FUSED")
    return op


def run(op, x1, T, update, sides="right"):
    return op.run(x1, T, update=update, sides=sides)


def timed(op, x1, T, update, reps=5):
    run(op, x1, T, update)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        op.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run(op, x1, T, update)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


def main():
    shapes = [(1000, 12, "tanh_mix"), (5000, 64, "identity"), (20000, 100, "tanh_mix"), (1_000_000, 100, "tanh_mix")]
    for dtype in ("f64", "f32"):
        tdt = torch.float64 if dtype == "f64" else torch.float32
        for n, T, upd in shapes:
            g = torch.Generator(device="cpu").manual_seed(n)
            x1 = torch.randn(n, generator=g, dtype=torch.float64).to(tdt).cuda()
            x1 /= x1.norm()
            a = make(n, True, dtype)
            b = make(n, False, dtype)
            ya = run(a, x1, T, upd)
            yb = run(b, x1, T, upd)
            err = float((ya.double() - yb.double()).norm() / yb.double().norm())
            rec = {"n": n, "T": T, "update": upd, "dtype": dtype, "rel_err_fused_vs_3pass": err,
                   "launches_fused": a.launch_count(), "launches_3pass": b.launch_count()}
            if n >= 20000:
                rec["ms_fused"] = timed(a, x1, T, upd)
                rec["ms_3pass"] = timed(b, x1, T, upd)
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
