# full ncu captures of the c5 kernels, summarised on the box (reports are too big to copy back)
mkdir -p gpurun_out
CMD="python bench.py --config c5 --m 768,768,1024 --steps 1 --warmup 3 --no-cpu --single"
$CMD > /dev/null 2>&1 || exit 1
cap() {  # name kernel-regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o /tmp/$1 -f $CMD > gpurun_out/ncu_$1.log 2>&1
  echo "$1 $?"
  python tools/ncu_summary.py full /tmp/$1.ncu-rep --json gpurun_out/$1_summary.json > /dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv > /tmp/$1_src.csv 2>/dev/null; gzip -c /tmp/$1_src.csv > gpurun_out/$1_src.csv.gz
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
}
cap c5_fwdcols_y k_pfft_fwd_cols 10
cap c5_conv k_conv1d_pp 2
cap c5_fwdcols_x k_pfft_fwd_cols 1
cap c5_bwdcols_y k_pfft_bwd_cols 5
