# per-source-line stall attribution of the c2 kernel (ncu source page, SASS view with line info)
mkdir -p gpurun_out
CMD="python bench.py --m 6144 --steps 2 --warmup 3 --no-cpu --single --no-graph"
$CMD > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_conv1d_pp -s 3 -c 1 -o /tmp/c2src -f $CMD > gpurun_out/ncu_src.log 2>&1
echo "FULL EXIT $?"
ncu -i /tmp/c2src.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -c > gpurun_out/c2_sass.csv.gz
ncu -i /tmp/c2src.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip -c > gpurun_out/c2_src.csv.gz
ls -la gpurun_out/c2_sass.csv.gz gpurun_out/c2_src.csv.gz
