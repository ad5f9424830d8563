#!/bin/bash
# On the GPU box: alternate A and B bench runs (REPS each) -> gpurun_out/ab_{A,B}.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in $(seq ${REPS:-3}); do
  for v in A B; do HD_LIB=ab/$v.so python bench.py "$@" >> gpurun_out/ab_$v.log 2>&1; done
done
python - <<'PY'
import json
for v in "AB":
    ms = [json.loads(l)["ms_per_step"] for l in open(f"gpurun_out/ab_{v}.log") if l.startswith("{")]
    print(v, " ".join(f"{m:.3f}" for m in ms), "mean", round(sum(ms) / len(ms), 3))
PY
