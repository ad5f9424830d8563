"""Large-n determinism / parity diagnostics (n = 1e7)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
from paper_2101_07464_b200 import lazymat as lm
N = int(os.environ.get("DN", 10_000_000))
STEPS = int(os.environ.get("DSTEPS", 40))
out = {}

def mk(ens, cap):
    if ens == "goe":
        return lm.GOEOperator(N, 5, sigma=N ** -0.5, capacity=cap)
    if ens == "haar":
        return lm.HaarOperator(N, seed=5, capacity=cap)
    return lm.GinibreOperator(N, N, N ** -0.5, 5, capacity=cap)

g = torch.Generator("cuda").manual_seed(5)
x1 = torch.randn(N, device="cuda", generator=g, dtype=torch.float64)
x1 /= x1.norm()
CAPS = [int(c) for c in os.environ.get("DCAPS", f"{STEPS},8").split(",")]
for ens in os.environ.get("DENS", "haar,goe,ginibre").split(","):
    trajs = []
    for rep, cap in enumerate(CAPS):
        op = mk(ens, cap)
        x = x1.clone()
        tr = []
        for t in range(STEPS):
            side = "right" if (ens != "ginibre" or t % 2 == 0) else "left"
            y = op.probe(x, side)
            tr.append(y.clone())
            x = y / y.norm()
        trajs.append(tr)
        del op
        torch.cuda.empty_cache()
    first = -1
    diffs = []
    for t in range(STEPS):
        d = float((trajs[0][t] - trajs[1][t]).abs().max())
        diffs.append(d)
        if d != 0 and first < 0:
            first = t
    out[ens] = {"first_mismatch": first, "maxdiff": max(diffs), "diffs_at": {str(t): diffs[t] for t in range(0, STEPS, 4)}}
    del trajs
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1), flush=True)
if os.environ.get("DORACLE", "1") == "1":
    import oracle as orc
    for ens in os.environ.get("DOENS", "goe,haar").split(","):
        k = 8
        n = N
        ref = orc.Operator(ens, m=n, n=n, sigma=n ** -0.5 if ens != "haar" else 1.0, seed=11)
        if ens == "ginibre":
            op = lm.GinibreOperator(n, n, n ** -0.5, 11, draws="injected", capacity=k)
            op.push_draws(orc.draws_for(11, [n] * k))
        elif ens == "goe":
            op = lm.GOEOperator(n, 11, sigma=n ** -0.5, draws="injected", capacity=k)
            op.push_draws(orc.draws_for(11, [n] * (2 * k)))
        else:
            op = lm.HaarOperator(n, seed=11, draws="injected", capacity=k)
            op.push_draws(orc.draws_for(11, [n] * k))
        aux = orc.RandomSource(12)
        errs = []
        for t in range(k):
            xx = aux.normal_vector(n)
            sd = "left" if (ens == "ginibre" and t % 2) else "right"
            a, b = op.probe(xx, sd), ref.probe(xx, sd)
            errs.append(float(np.linalg.norm(a - b) / np.linalg.norm(b)))
        out[ens + "_oracle"] = errs
    print(json.dumps(out, indent=1))
