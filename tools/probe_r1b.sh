mkdir -p gpurun_out
export VCG_WATCHDOG_S=60
timeout 200 python tools/sweep_budget.py gnp400 torus60 > gpurun_out/sweep_budget.log 2>&1
VCG_NO_SMEM_CSR=1 timeout 200 python tools/sweep_budget.py gnp400 torus60 >> gpurun_out/sweep_budget.log 2>&1
