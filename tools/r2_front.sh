#!/bin/bash
# Frontier root kernel: parity tests, then large-config timings with traces.
export VCG_WATCHDOG_S=120
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_root_pipeline.py tests/test_gpu_large.py > gpurun_out/pytest_front.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_front.log
tail -30 gpurun_out/pytest_front.log
timeout 300 python tools/root_large.py > gpurun_out/root_large.log 2>&1
cat gpurun_out/root_large.log
for w in ba100k planted1m; do
VCG_TRACE=1 timeout 300 python tools/root_large.py $w > gpurun_out/root_trace_$w.log 2>&1
done
