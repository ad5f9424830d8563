#!/bin/bash
# Launch list + one full ncu capture of every kernel of probe t = 91 of the
# bench workload (run on the GPU box through gpurun). Usage: tools/profile_round.sh TAG
TAG=${1:-prof}
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dots|k_apply|k_small" -s 450 -c 5 \
    -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo profile_done
