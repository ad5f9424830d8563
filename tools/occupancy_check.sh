#!/bin/bash
# default (balance heuristic) vs fixed 8 warps on the bench at n = 1e6 / 1e7 / 3e6
for N in 1000000 10000000 3000000; do
  T=100; [ $N -ge 3000000 ] && T=40
  for W in "" 8; do
    if [ -z "$W" ]; then unset HD_WARPS; else export HD_WARPS=$W; fi
    r=$(timeout 300 python bench.py --no-cpu-baseline --steps 5 --n $N --T $T 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "n=$N warps=${W:-auto} ms=$r"
  done
done
