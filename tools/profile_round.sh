#!/bin/bash
# Round evidence (run via gpurun on one B200, after tools/round_gpu.sh ran the bench): launch list
# of one timed bench step, full ncu captures of the three heavy kernels.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 --no-c4 --no-c5 > gpurun_out/launches_bench.log 2>&1
# reports exported to CSV on the box (raw metrics + SASS source page) and removed:
# gpurun merges back at most 64 MiB
for k in select_warp_kernel blend_kernel backward_pixels_kernel records_kernel finish_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 --no-c4 --no-c5 > gpurun_out/full_$k.log 2>&1
  ncu -i gpurun_out/full_$k.ncu-rep --page raw --csv > gpurun_out/full_$k.raw.csv 2>/dev/null
  ncu -i gpurun_out/full_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/full_$k.sass.csv 2>/dev/null
  rm -f gpurun_out/full_$k.ncu-rep
done
