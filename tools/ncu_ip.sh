#!/bin/bash
# one full ncu capture of the in-place c2 kernel (after a plain run); the report comes back in
# gpurun_out/ for per-instruction stall attribution here:
#   ncu -i gpurun_out/ip_conv.ncu-rep --page source --csv --metrics smsp__pcsamp_warps_issue_stalled_long_scoreboard,...
mkdir -p gpurun_out
CMD="python tools/ab_conv.py 6000 11999 6144 4096"
$CMD > gpurun_out/ip_plain.log 2>&1 || { echo plain failed; tail gpurun_out/ip_plain.log; exit 1; }
tail -1 gpurun_out/ip_plain.log
ncu --set full --clock-control none --import-source on -k regex:k_conv1d_ip -s 3 -c 1 -o gpurun_out/ip_conv -f $CMD > gpurun_out/ncu_ip.log 2>&1
echo "FULL EXIT $?"; tail -2 gpurun_out/ncu_ip.log; ls -la gpurun_out/ip_conv.ncu-rep
python tools/ncu_summary.py full gpurun_out/ip_conv.ncu-rep --json gpurun_out/ip_conv_summary.json | head -40
