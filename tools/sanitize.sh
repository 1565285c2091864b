#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every kernel family
# (tools/sanitize_cases.py); one process per (tool, case); logs in gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
CASES=${CASES:-"pp_c2 pp2_4096 pp_small pp_centered single_herm_tmem single_stage_acc naive cols_2d cols_3d_herm general_op"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck initcheck"}
for t in $TOOLS; do
  for c in $CASES; do
    log=gpurun_out/sanitize/${t}_${c}.log
    timeout 900 $CS --tool $t --error-exitcode 17 --print-limit 20 python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    echo "$t $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rel_l2' $log | tr '\n' ' ')"
  done
done
