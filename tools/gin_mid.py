"""Single-trial Ginibre runs (alternating normalised power iteration, T = 100)
at mid-range n, device Philox draws, graph-replayed: median ms per run for the
current HD_GIN2P setting. Env: GM_N (comma list), GM_DT (f64|f32)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

T = 100
dt = os.environ.get("GM_DT", "f64")
tdt = torch.float64 if dt == "f64" else torch.float32
res = {}
for n in [int(float(v)) for v in os.environ.get("GM_N", "3e4,1e5,3e5,1e6").split(",")]:
    x1 = torch.randn(n, dtype=tdt, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    x1 /= x1.norm()
    ts = []
    for rep in range(6):
        op = lazymat.GinibreOperator(n, n, n ** -0.5, 1 + rep, capacity=T, dtype=dt)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        op.run(x1, T, update="normalize", sides="alternate")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[n] = sorted(ts[1:])[len(ts[1:]) // 2]
print(json.dumps({"dtype": dt, "gin2p": os.environ.get("HD_GIN2P", "auto"), "ms": res}))
