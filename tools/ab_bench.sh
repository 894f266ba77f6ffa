#!/bin/bash
# A/B stage timing of alternative in-tree builds: tools/ab_bench.sh variants/lib_*.so
for lib in "$@"; do
  name=$(basename $lib .so)
  POTR_B200_LIB=$lib python bench.py --steps 3 --warmup 2 --no-e2e --no-scene --no-cpu-baseline \
    > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{n}.json"))
    st = d["roofline"]["stage_ms_per_step"]
    print(n, round(d["ms_per_step"], 1), {k: round(v, 1) for k, v in st.items() if v})
except Exception as e:
    print(n, "failed", e)
PY
done
