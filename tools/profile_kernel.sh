#!/bin/bash
# usage (on the GPU box): tools/profile_kernel.sh <regex> <out-name>
# full ncu capture (source-correlated) of one launch of the matching kernel in a C2 step
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"$1" -s 3 -c 1 \
    -o gpurun_out/$2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 --no-c4 --no-c5 > gpurun_out/$2.log 2>&1
tail -2 gpurun_out/$2.log
