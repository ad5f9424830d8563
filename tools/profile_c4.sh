#!/bin/bash
# Config-4 (AMP, m = 2e7, n = 1e7, T = 200) evidence on the GPU box:
#   TAG_bench.log     the default bench line (bench.py)
#   TAG_launches.csv  ncu launch list (gpu__time_duration.sum) of one AMP run (tools/amp_profile.py)
#   TAG_full.ncu-rep  ncu --set full of k_nt launches SKIP, SKIP+1 of that run (default 760, 761:
#                     fold + output pass of probe 380, the 4-stage two-slot schedule)
# Summarise here with tools/ncu_summary.py {launches,full}.
TAG=${1:-c4}
SKIP=${2:-760}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || exit 1
AP_PROF=0 python tools/amp_profile.py > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    env AP_PROF=0 python tools/amp_profile.py > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_nt -s $SKIP -c 2 \
    -o gpurun_out/${TAG}_full env AP_PROF=0 python tools/amp_profile.py > gpurun_out/${TAG}_ncu.log 2>&1
echo profile_done
