#!/bin/bash
# usage (GPU box): tools/prof_kernels.sh <tag> [kernel regex ...]
# full ncu capture (source-correlated) of one launch of each kernel in a C2 step,
# plus the SASS source page CSV of each (read with tools/sass_lines.py).
tag=$1; shift
ks=${@:-select_warp_kernel blend_kernel backward_pixels_kernel}
mkdir -p gpurun_out
for k in $ks; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o gpurun_out/${tag}_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 --no-c4 --no-c5 \
      > gpurun_out/${tag}_$k.log 2>&1
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_$k.sass.csv 2>/dev/null
done
