#!/bin/bash
# Round-2 probe: reproduce the exit-time crash and collect a backtrace.
export VCG_WATCHDOG_S=120
mkdir -p gpurun_out
which gdb > gpurun_out/gdb.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_exit.py -q -x > gpurun_out/exit_test.log 2>&1; echo "rc=$?" >> gpurun_out/exit_test.log
tail -40 gpurun_out/exit_test.log
timeout 900 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_exit.py > gpurun_out/pytest_fh.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fh.log
tail -60 gpurun_out/pytest_fh.log
