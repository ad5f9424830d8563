import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat
n, T = 1_000_000, 100
for prof in (False, False, True):
    op = lazymat.HaarOperator(n, seed=1, dtype="c128", capacity=T)
    if prof: op.set_profiling(True)
    x = torch.randn(n, dtype=torch.complex128, device="cuda"); x /= x.norm()
    torch.cuda.synchronize(); t0 = time.perf_counter(); ts=[]
    for t in range(T):
        a = time.perf_counter()
        y = op.probe(x, "right")
        ts.append(time.perf_counter()-a)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print("spec", os.environ.get("HD_CX_SPEC","1"), "prof", prof, "wall ms", round(dt*1e3,2), "probe us @10,50,99:", [round(ts[i]*1e6) for i in (1,2,3,10,50,99)])
    import statistics
    print("spikes", [(i, round(v*1e6)) for i,v in enumerate(ts) if v*1e6 > 300 + 12*i])
    if prof:
        st = op.kernel_stats(); print({k:(round(v["ms"],2), v["launches"]) for k,v in st.items()})
