#!/bin/bash
# frontier root kernel: phase profile on the large configs, then parity tests
for w in ba100k planted1m; do
VCG_TRACE=1 timeout 300 python tools/front_one.py $w 2>&1 | grep "frontier fixpoint\|d1 phases" | tail -2 | cut -c1-400
done
VCG_WATCHDOG_S=120 timeout 600 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_root_pipeline.py tests/test_gpu_large.py 2>&1 | tail -2
python tools/root_large.py 2>&1 | grep resident | awk 'NR%5==0'
