#!/bin/bash
# Every BASELINE config on one GPU box, current build -> gpurun_out/TAG_configs.jsonl
# (one JSON object per line: config 1 tools/config1.py; config 2 and 4 bench.py lines;
# config 3 tools/config3.py; config 5 at one rank's share n = 1.25e7 tools/config45.py).
TAG=${1:-cfg}
out=gpurun_out/${TAG}_configs.jsonl
mkdir -p gpurun_out
: > $out
python tools/config1.py >> $out
python bench.py --workload config2 --no-cpu-baseline | tail -1 >> $out
python tools/config3.py | python -c "import json,sys; print(json.dumps({'workload': 'config3', **json.load(sys.stdin)}))" >> $out
python bench.py --no-cpu-baseline | tail -1 >> $out
C4_T=0 C5_N=12500000 python tools/config45.py | python -c "import json,sys; print(json.dumps({'workload': 'config5_1gpu_share', **json.load(sys.stdin)}))" >> $out
echo configs_done
