#!/bin/bash
# c2 headline profile: plain run first, then the launch list, then one full capture of the
# top kernel (each ncu pass only after the same command exited 0 without ncu)
mkdir -p gpurun_out
CMD="python bench.py --m 6144 --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; tail gpurun_out/prof_plain.err; exit 1; }
[ -n "$SKIP_LAUNCHES" ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "LAUNCHES EXIT $?"
ncu --set full --clock-control none --import-source on -k regex:k_conv1d_pp -s 3 -c 1 -o gpurun_out/c2_conv -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "FULL EXIT $?"; tail -3 gpurun_out/ncu_full.log
