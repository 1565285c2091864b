#!/bin/bash
# one GPU call: parity tests, then the bench lines (c2 headline + the other configs)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu --timeout 300 -x -k "not config5_full" > gpurun_out/gpu_tests.log 2>&1
echo "TESTS EXIT $?"; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2; grep -E "^FAILED|^ERROR" gpurun_out/gpu_tests.log | head -20
python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "BENCH EXIT $?"; cut -c1-1500 gpurun_out/bench_c2.json; tail -2 gpurun_out/bench_c2.err
rm -f gpurun_out/bench_all.json
for c in c1 c3 c4 c5; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu >> gpurun_out/bench_all.json 2>>gpurun_out/bench_all.err; done
python - << 'PY'
import json
for l in open('gpurun_out/bench_all.json'):
    d=json.loads(l); print(d['config']['config'], 'ms/step %.4f' % d['ms_per_step'], 'Gpts/s %.3f' % (d['value']/1e9), 'fp64 frac %.3f' % d['roofline']['frac'], d['config']['plan'], d['config']['kernel'])
PY
