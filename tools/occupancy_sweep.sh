#!/bin/bash
# (spare SMs, warps per CTA) sweep of the streaming kernels on the bench workload
for N in 1000000 10000000; do
  T=100; [ $N -eq 10000000 ] && T=40
  for cfg in "0 8" "24 8" "0 7" "0 6" "0 5" "0 4" "24 6" "48 8" "74 8"; do
    set -- $cfg
    r=$(HD_SPARE_SMS=$1 HD_WARPS=$2 timeout 300 python bench.py --no-cpu-baseline --steps 5 --n $N --T $T 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "n=$N spare=$1 warps=$2 ms=$r"
  done
done
