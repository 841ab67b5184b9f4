#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/l2_atomic_peak tools/l2_atomic_peak.cu && ./gpurun_out/l2_atomic_peak > gpurun_out/l2_atomic_peak.json
cat gpurun_out/l2_atomic_peak.json
python tools/pair_timeline.py > gpurun_out/pair_timeline.json; head -12 gpurun_out/pair_timeline.json
