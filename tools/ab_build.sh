#!/bin/bash
# Build the committed tree (HEAD) as ab/A.so and the working tree as ab/B.so
# for a same-box A/B run:  HD_LIB=ab/A.so python bench.py  vs  HD_LIB=ab/B.so ...
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
rm -rf /tmp/ab_head && mkdir -p /tmp/ab_head && git archive HEAD paper_2101_07464_b200/csrc include | tar -x -C /tmp/ab_head
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
$NV -o ab/A.so /tmp/ab_head/paper_2101_07464_b200/csrc/hd_lib.cu paper_2101_07464_b200/lib/hd_refrng.o
python -c "import __graft_entry__ as g; g.build()"
cp paper_2101_07464_b200/lib/libhd_b200.so ab/B.so
