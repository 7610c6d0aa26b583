for v in base vs32 sp2 vs8 base; do
  echo -n "$v "; GVR_LIB_PATH=build_ab/$v.so python bench.py --no-c4 --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c 'import json,sys; b=json.loads(sys.stdin.read()); print(round(b["value"],1), "c3", round(b["c3"]["value"],1), "c5", round(b["c5"]["value"],1))'
done
