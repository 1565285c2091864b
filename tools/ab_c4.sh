#!/bin/bash
# A/B of library variants on c4 (fixed plan 4096 x 4096): whole-convolution time and the launch list
# per variant.  Usage: bash tools/ab_c4.sh f0 f1 f2
mkdir -p gpurun_out
for v in "$@"; do
  export HCONV_LIB_VARIANT=$v
  echo "== $v: $(python tools/c4_parts.py quick 2>&1 | tail -1)"
  CMD="python bench.py --config c4 --m 4096,4096 --steps 1 --warmup 3 --no-cpu --single --no-graph"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_$v.csv $CMD > /dev/null 2>&1
  python tools/ncu_summary.py launches gpurun_out/launches_c4_$v.csv | python -c "
import json,sys
for k in json.load(sys.stdin)[:3]: print('   ', k['kernel'][9:40], round(k['avg_us'],1))"
done
