"""Small two-pass Haar run for compute-sanitizer (memcheck / racecheck /
synccheck): N (default 50000) rows, T (default 100) tanh-mix probes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2101_07464_b200 import lazymat
n = int(os.environ.get("N", 50000)); T = int(os.environ.get("T", 100))
x1 = np.random.default_rng(0).standard_normal(n); x1 /= np.linalg.norm(x1)
op = lazymat.HaarOperator(n, seed=1, capacity=T)
y = op.run(x1, T, update="tanh_mix", sides="right", use_graph=os.environ.get("USE_GRAPH") == "1")
print("ok", op.launch_count(), float(np.linalg.norm(y)))
