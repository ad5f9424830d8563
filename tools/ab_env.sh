#!/bin/bash
# On the GPU box: alternate variants of the config-4 AMP run (tools/amp_profile.py)
# given as "LABEL:ENV=V,ENV=V" arguments, REPS rounds -> gpurun_out/ab_env.txt
# e.g. tools/ab_env.sh "base:HD_LIB=ab/A.so" "new:HD_LIB=ab/B.so,HD_NT_EVICT=1"
# AB_BENCH="--workload config2": time bench.py with those arguments instead
# (its ms_per_step).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab_env.txt
: > $out
for i in $(seq ${REPS:-2}); do
  for v in "$@"; do
    label=${v%%:*}; envs=${v#*:}
    if [ -n "$AB_BENCH" ]; then
      ms=$(env $(echo "$envs" | tr ',' ' ') python bench.py $AB_BENCH --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    else
      ms=$(env $(echo "$envs" | tr ',' ' ') AP_PROF=0 python tools/amp_profile.py 2>&1 | grep '"ms"' | tr -dc '0-9.')
    fi
    echo "$label $ms" >> $out
  done
done
python - "$out" <<'PY'
import sys, collections
d = collections.OrderedDict()
for l in open(sys.argv[1]):
    k, v = l.split()
    d.setdefault(k, []).append(float(v) if v else float("nan"))
for k, v in d.items():
    print(f"{k:24s} " + " ".join(f"{x:8.1f}" for x in v) + f"   min {min(v):8.1f}")
PY
