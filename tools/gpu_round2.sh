#!/bin/bash
# Round measurement: a --set full capture of the root-fixpoint kernel first
# (summarised on the box into profiles/r02_root_front_ncu.json, which the
# bench's roofline reads), GPU tests, smoke, bench (+ reference arm), ncu
# launch list of the bench and a --set full capture of the search kernel.
export VCG_WATCHDOG_S=120
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_root_front -s 3 -c 1 -o gpurun_out/prof_root -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs --no-strong > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
python tools/summarize_ncu.py r02 prof_root root_front "python bench.py --steps 1 --warmup 3 (k_root_front, planted1m)" > /dev/null && cp profiles/r02_root_front_ncu.json gpurun_out/
if [ "$1" != "nobench" ] || [ "$2" == "tests" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
fi
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
if [ "$1" != "nobench" ]; then
timeout 900 python bench.py --steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 4000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 600 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs --no-strong > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/prof_search -f python tools/ncu_one.py rgg2000 1281 > gpurun_out/ncu_search.log 2>&1
tail -2 gpurun_out/ncu_search.log
