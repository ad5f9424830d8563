"""Acceptance-scale statistical verification on the production path
(acceptance.cpp criteria 4 and 8 at the reference's trial counts): lazy
device operators with Philox draws vs dense direct simulation."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_07464_b200.lazymat import verify  # noqa: E402

out = {}
for name, fn in [("haar-equivalence", lambda s: verify.haar_equivalence_suite(trials=10000, seed=s)),
                 ("ista-equivalence", lambda s: verify.ista_equivalence_suite(trials=10000, seed=s))]:
    t0 = time.perf_counter()
    rep = verify.with_retry(fn, 1)
    out[name] = {"passed": rep.passed(), "s": time.perf_counter() - t0,
                 "checks": {c.name: c.detail for c in rep.checks}}
t0 = time.perf_counter()
ctl = verify.mismatched_ensemble_control(trials=10000)
out["mismatched-ensemble-control (must fail)"] = {"passed": ctl.passed(), "s": time.perf_counter() - t0,
                                                  "checks": {c.name: c.detail for c in ctl.checks}}
print(json.dumps(out, indent=1))
