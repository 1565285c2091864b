mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_mult.py -q -m gpu -x -k "nd or 2d or 3d or config4 or config5" 2>&1 | tail -3
for c in "c5 768,768,1024" "c4 4096,2048"; do set -- $c
  for pp in 0 1; do
    echo "$1 NO_COLS_PP=$pp $(HCONV_NO_COLS_PP=$pp python bench.py --config $1 --m $2 --steps 5 --warmup 3 --no-cpu --single 2>&1 | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["ms_per_step"])')"
  done
done
echo "c5 planner $(python bench.py --config c5 --steps 5 --warmup 3 --no-cpu --single 2>&1 | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["ms_per_step"], d["details"]["plan"])')"
