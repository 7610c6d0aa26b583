#!/bin/bash
# ncu --set full of one launch of each named kernel in a C4 step (1M kernels, 1024^2),
# exported as CSV (raw metrics + SASS source page): tools/prof_c4.sh <tag> <kernel> ...
tag=$1; shift
mkdir -p gpurun_out
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/${tag}_$k -f python tools/one_step.py 1000000 1024 3 > gpurun_out/${tag}_$k.log 2>&1
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page raw --csv > gpurun_out/${tag}_$k.raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_$k.sass.csv 2>/dev/null
  rm -f gpurun_out/${tag}_$k.ncu-rep
done
