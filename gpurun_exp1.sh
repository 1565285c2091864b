mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stress.py -q -x > gpurun_out/stress.log 2>&1; echo "STRESS $?"; tail -3 gpurun_out/stress.log
for mb in 0 32 64 128; do
  HCONV_ND_BLOCK_MB=$mb timeout 300 python bench.py --config c5 --single --no-cpu --steps 5 --m 768,768,1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 blockmb $mb', d['ms_per_step'])"
  HCONV_ND_BLOCK_MB=$mb timeout 300 python bench.py --config c5 --single --no-cpu --steps 5 --m 256,256,256 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 m256 blockmb $mb', d['ms_per_step'])"
done
