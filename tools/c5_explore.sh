mkdir -p gpurun_out
for mb in 24 48 96 192 400 4000; do
  echo "MB=$mb $(HCONV_ND_BLOCK_MB=$mb python bench.py --config c5 --m 768,768,1024 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["ms_per_step"])')"
done
for mb in 48 96 400; do
  echo "c4 MB=$mb $(HCONV_ND_BLOCK_MB=$mb python bench.py --config c4 --m 4096,2048 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["ms_per_step"])')"
done
CMD="python bench.py --config c5 --m 768,768,1024 --steps 1 --warmup 3 --no-cpu"
ncu --set full --clock-control none --import-source on -k regex:k_pfft_fwd_cols -s 10 -c 1 -o gpurun_out/c5_fwdcols -f $CMD > gpurun_out/ncu_c5a.log 2>&1; echo "A $?"
ncu --set full --clock-control none --import-source on -k regex:k_conv1d_pp -s 10 -c 1 -o gpurun_out/c5_conv -f $CMD > gpurun_out/ncu_c5b.log 2>&1; echo "B $?"
ncu --set full --clock-control none --import-source on -k regex:k_pfft_fwd_cols -s 1 -c 1 -o gpurun_out/c5_fwdcols_x -f $CMD > gpurun_out/ncu_c5c.log 2>&1; echo "C $?"
