# A/B of two library builds on the box (build_ab/<name>.so via tools/build_variant.sh):
# GPU parity subset on the candidate, then alternating C2 (+ C4) bench lines.
set -x
mkdir -p gpurun_out
A=${A:-stage}; B=${B:-pixrow}
GVR_LIB_PATH=build_ab/$B.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_fullsize.py -x -q > gpurun_out/ab_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab_tests.log
for v in ${LIST:-$A $B $A $B $A $B}; do
  echo -n "$v " >> gpurun_out/ab.txt
  GVR_LIB_PATH=build_ab/$v.so timeout 300 python bench.py --no-c3 --no-c5 --no-cpu-baseline --no-e2e --steps 50 2>/dev/null | python -c 'import json,sys; b=json.loads(sys.stdin.read()); s=b["roofline"]["stage_ms_per_step"]; print(round(b["value"],1), "blend", round(s["blend"]*1e3,1), "bwd", round(s["backward"]*1e3,1), "obj", round(s["object_space"]*1e3,1), "loss", round(s["loss"]*1e3,1), "c4", round(b["c4"]["value"],1))' >> gpurun_out/ab.txt
done
