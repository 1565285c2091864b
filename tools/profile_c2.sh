#!/bin/bash
# c2 headline profile: plain run first, then the launch list, then one full capture of the
# top kernel (each ncu pass only after the same command exited 0 without ncu); summarised on the
# box (the report itself stays there)
mkdir -p gpurun_out
CMD="python bench.py --m 6144 --steps 2 --warmup 3 --no-cpu --single --no-graph"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; tail gpurun_out/prof_plain.err; exit 1; }
[ -n "$SKIP_LAUNCHES" ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "LAUNCHES EXIT $?"
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches_summary.json
ncu --set full --clock-control none --import-source on -k regex:k_conv1d_ -s 3 -c 1 -o /tmp/c2_conv -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "FULL EXIT $?"; tail -3 gpurun_out/ncu_full.log
python tools/ncu_summary.py full /tmp/c2_conv.ncu-rep --json gpurun_out/c2_conv_summary.json > /dev/null
ncu -i /tmp/c2_conv.ncu-rep --page raw --csv 2>/dev/null | gzip -c > gpurun_out/c2_conv_raw.csv.gz
