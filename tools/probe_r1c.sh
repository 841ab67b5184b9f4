mkdir -p gpurun_out
export VCG_WATCHDOG_S=60
W="rgg2000 gnp400 torus60"
TAG=smem_csr timeout 300 python tools/sweep_place.py $W > gpurun_out/sweep_place.log 2>&1
TAG=gl_csr VCG_NO_SMEM_CSR=1 timeout 300 python tools/sweep_place.py $W >> gpurun_out/sweep_place.log 2>&1
TAG=gl_ws VCG_WS_GLOBAL=1 timeout 300 python tools/sweep_place.py $W >> gpurun_out/sweep_place.log 2>&1
