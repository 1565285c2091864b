#!/bin/bash
# launch lists of the non-headline configurations (fixed plans: no planner launches); each ncu pass
# only after the same command exited 0 without ncu.  Usage: bash tools/profile_all.sh [c1 c3 c4 c5]
mkdir -p gpurun_out
declare -A M=([c1]=2048 [c3]=8192 [c4]=4096,4096 [c5]=768,768,1024)
for c in ${@:-c1 c3 c4 c5}; do
  CMD="python bench.py --config $c --m ${M[$c]} --steps 1 --warmup 3 --no-cpu --single"
  $CMD > gpurun_out/plain_$c.json 2> gpurun_out/plain_$c.err || { echo "$c plain failed"; tail -3 gpurun_out/plain_$c.err; continue; }
  echo "$c plain: $(python -c "import json;d=json.load(open('gpurun_out/plain_$c.json'));print(d['ms_per_step'])")"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$c.csv $CMD > gpurun_out/ncu_launches_$c.log 2>&1
  echo "$c LAUNCHES EXIT $?"
  python tools/ncu_summary.py launches gpurun_out/launches_$c.csv > gpurun_out/launches_${c}_summary.json
done
