#!/bin/bash
# The N>1 bench path on a 1-GPU box: 2 ranks over gloo (world > devices), and
# NCCL at world 1 through torchrun.
mkdir -p gpurun_out
export VCG_WATCHDOG_S=120
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "rc=$?"
tail -c 1500 gpurun_out/bench_n2.json; tail -3 gpurun_out/bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/bench_n1t.json 2> gpurun_out/bench_n1t.err; echo "rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_n1t.json').read().strip().splitlines()[-1]); print(d['value'], d['strong_scaling']['time_to_solution_s'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_ref_n2.json 2> gpurun_out/bench_ref_n2.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref_n2.json
