#!/bin/bash
# one full ncu capture of a kernel of `bench.py --config C --m M` (plain run first), summarised on
# the box:  bash tools/ncu_cfg.sh <config> <m> <kernel-regex> <skip> <name>
mkdir -p gpurun_out
CMD="python bench.py --config $1 --m $2 --steps 1 --warmup 3 --no-cpu --single"
$CMD > gpurun_out/plain_$5.json 2>&1 || { echo "$5 plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o /tmp/$5 -f $CMD > gpurun_out/ncu_$5.log 2>&1
echo "$5 FULL EXIT $?"
python tools/ncu_summary.py full /tmp/$5.ncu-rep --json gpurun_out/$5_summary.json > /dev/null
ncu -i /tmp/$5.ncu-rep --page source --csv 2>/dev/null | gzip -c > gpurun_out/$5_src.csv.gz
