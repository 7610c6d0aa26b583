#!/bin/bash
# full ncu capture of the blend kernel in a C2 step, exported to CSV on the box
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:blend_kernel -s 3 -c 1 \
    -o gpurun_out/full_blend_kernel -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 --no-c4 --no-c5 > gpurun_out/full_blend_kernel.log 2>&1
ncu -i gpurun_out/full_blend_kernel.ncu-rep --page raw --csv > gpurun_out/full_blend_kernel.raw.csv 2>/dev/null
ncu -i gpurun_out/full_blend_kernel.ncu-rep --page source --csv --print-source sass > gpurun_out/full_blend_kernel.sass.csv 2>/dev/null
rm -f gpurun_out/full_blend_kernel.ncu-rep
