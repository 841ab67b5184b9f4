#!/bin/bash
# Frontier root kernel: timing breakdown over solo thresholds.
mkdir -p gpurun_out
for solo in 0; do
for w in ba100k planted1m; do
echo "== solo=$solo $w"
VCG_FRONT_SOLO=$solo VCG_TRACE=1 timeout 300 python tools/front_one.py $w 2>&1 | grep "frontier fixpoint\|d1 phases" | tail -2
done; done
