#!/bin/bash
# one GPU call: parity tests, then the default bench line (c2 headline + the other configurations)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -q -m gpu --timeout 900 -x ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
echo "TESTS EXIT $?"; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2; grep -E "^FAILED|^ERROR" gpurun_out/gpu_tests.log | head -20
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "BENCH EXIT $?"; cut -c1-3000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
