#!/bin/bash
# Run on the GPU box (via gpurun): launch list + full ncu capture of the two
# dominant kernels of one C2 fwd+bwd step. Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 --no-c4 --no-c5 > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'fine_forward|backward_pixels' -s 6 -c 2 \
    -o gpurun_out/prof_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 --no-c4 --no-c5 > gpurun_out/prof_bench.log 2>&1
