#!/bin/bash
# Host-side phase timings of the root pipeline on the large configs.
mkdir -p gpurun_out
timeout 300 python tools/root_large.py > gpurun_out/root_large.log 2>&1
for w in ba100k planted1m; do
VCG_TRACE=1 timeout 300 python tools/root_large.py $w > gpurun_out/root_trace_$w.log 2>&1
done
cat gpurun_out/root_large.log
