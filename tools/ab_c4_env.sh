#!/bin/bash
# c4 (fixed plan 4096 x 4096) under environment settings: bash tools/ab_c4_env.sh VARIANT "ENV=1" "ENV=2" ...
mkdir -p gpurun_out
export HCONV_LIB_VARIANT=$1; shift
for e in "$@"; do
  echo "== $e: $(env $e python tools/c4_parts.py quick 2>&1 | tail -1)"
  CMD="python bench.py --config c4 --m 4096,4096 --steps 1 --warmup 3 --no-cpu --single --no-graph"
  env $e ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_ab.csv $CMD > /dev/null 2>&1
  python tools/ncu_summary.py launches gpurun_out/launches_c4_ab.csv | python -c "
import json,sys
for k in json.load(sys.stdin)[:3]: print('   ', k['kernel'][9:40], round(k['avg_us'],1))"
done
