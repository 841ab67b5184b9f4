#!/bin/bash
# Round-2 GPU call: selected pytest files, large-config root timing.
export VCG_WATCHDOG_S=120
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -p no:cacheprovider "$@" > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
tail -30 gpurun_out/pytest_sel.log
timeout 300 python tools/root_large.py > gpurun_out/root_large.log 2>&1
VCG_TRACE=1 timeout 300 python tools/root_large.py planted1m > gpurun_out/root_large_trace.log 2>&1
cat gpurun_out/root_large.log
grep -v "^\[vcg search" gpurun_out/root_large_trace.log | tail -40
