#!/bin/bash
# Step 0 on the GPU box: device attributes, FP64 throughput with clocks sampled, host CPU facts.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 100 > gpurun_out/step0_clocks.csv &
SMI=$!
./tools/peaks_fp64 > gpurun_out/step0_fp64.json 2>&1
kill $SMI
nproc > gpurun_out/step0_host.txt; lscpu | grep -E 'Model name|^CPU\(s\)|Thread|Socket|NUMA node\(s\)' >> gpurun_out/step0_host.txt
nvidia-smi -q | grep -iE 'product name|clocks|max' | head -30 >> gpurun_out/step0_host.txt
cat gpurun_out/step0_fp64.json
