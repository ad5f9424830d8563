import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import oracle as orc
from paper_2101_07464_b200 import lazymat as lm
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
out = {}
n, T, seed = 3000, 300, 31
u = orc.RandomSource(seed, 1).normal_vector(n); u /= np.linalg.norm(u)
x1 = orc.RandomSource(seed, 2).normal_vector(n); x1 /= np.linalg.norm(x1)
ref = orc.Operator("goe", n=n, sigma=n ** -0.5, seed=seed)
xr, ovr = ref.spiked_power(u, x1, T)
for cap in (T, 16):
    op = lm.GOEOperator(n, seed, sigma=n ** -0.5, draws="injected", capacity=cap)
    op.push_draws(orc.draws_for(seed, [n] * (2 * T)))
    x, ov = lm.spiked_power(op, u, x1, T)
    ov = ov.cpu().numpy()
    bad = np.nonzero(np.abs(ov - ovr) > 1e-8)[0]
    out[f"goe_cap{cap}"] = {"rel_x": rel(x.cpu().numpy(), xr), "first_bad": int(bad[0]) if len(bad) else -1,
                            "ov_ref": [float(ovr[i]) for i in (99, 119, 127, 128, 129, 199, 299)],
                            "ov_dev": [float(ov[i]) for i in (99, 119, 127, 128, 129, 199, 299)]}
# Haar probe-by-probe to 600
n, T = 2000, 600
ref = orc.Operator("haar", n=n, seed=7)
op = lm.HaarOperator(n, seed=7, draws="injected", capacity=T)
op.push_draws(orc.draws_for(7, [n] * T))
aux = orc.RandomSource(8)
errs = []
for t in range(T):
    xx = aux.normal_vector(n)
    s = "right" if t % 3 else "left"
    errs.append(rel(op.probe(xx, s), ref.probe(xx, s)))
errs = np.array(errs)
out["haar_probe_err"] = {"max": float(errs.max()), "first_bad": int(np.argmax(errs > 1e-9)) if (errs > 1e-9).any() else -1,
                         "at": [float(errs[i]) for i in (100, 250, 255, 256, 257, 300, 511, 512, 513, 599)]}
# Ginibre
m, n, T = 1500, 1200, 600
ref = orc.Operator("ginibre", m=m, n=n, sigma=1.0, seed=9)
op = lm.GinibreOperator(m, n, 1.0, 9, draws="injected", capacity=64)
sides = ["right" if t % 2 == 0 else "left" for t in range(T)]
op.push_draws(orc.draws_for(9, [m if s == "right" else n for s in sides]))
aux = orc.RandomSource(10)
errs = []
for s in sides:
    xx = aux.normal_vector(n if s == "right" else m)
    errs.append(rel(op.probe(xx, s), ref.probe(xx, s)))
errs = np.array(errs)
out["gin_probe_err"] = {"max": float(errs.max()), "first_bad": int(np.argmax(errs > 1e-9)) if (errs > 1e-9).any() else -1}
print(json.dumps(out, indent=1))
