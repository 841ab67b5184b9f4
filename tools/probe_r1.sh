mkdir -p gpurun_out
export VCG_WATCHDOG_S=120
VCG_TRACE=1 timeout 300 python tools/root_trace_big.py ba100k planted1m > gpurun_out/root_trace.log 2>&1
timeout 300 python tools/phases.py rgg2000 > gpurun_out/phases_rgg.log 2>&1
timeout 300 python tools/phases_budget.py gnp400 2 > gpurun_out/phases_gnp.log 2>&1
timeout 300 python tools/phases_budget.py torus60 2 >> gpurun_out/phases_gnp.log 2>&1
