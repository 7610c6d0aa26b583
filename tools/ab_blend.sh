set -x
mkdir -p gpurun_out
GVR_LIB_PATH=build_ab/swz.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q > gpurun_out/ab_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab_tests.log
for v in stage swz stage swz stage swz; do
  echo -n "$v " >> gpurun_out/ab.txt
  GVR_LIB_PATH=build_ab/$v.so timeout 300 python bench.py --no-c3 --no-c4 --no-c5 --no-cpu-baseline --no-e2e --steps 50 2>/dev/null | python -c 'import json,sys; b=json.loads(sys.stdin.read()); s=b["roofline"]["stage_ms_per_step"]; print(round(b["value"],1), "blend", round(s["blend"]*1e3,1), "select", round(s["select"]*1e3,1), "bwd", round(s["backward"]*1e3,1))' >> gpurun_out/ab.txt
done
