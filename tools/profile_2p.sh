#!/bin/bash
# Launch list + one full ncu capture of probe t = 91 of the bench workload
# (two-pass Haar run: k_small_2p + k_haar2p per probe). Run on the GPU box:
# tools/profile_2p.sh TAG
TAG=${1:-p2}
mkdir -p gpurun_out
python bench.py --workload config2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --workload config2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_haar2p|k_small_2p" -s 180 -c 4 \
    -o gpurun_out/${TAG}_full python bench.py --workload config2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo profile_done
