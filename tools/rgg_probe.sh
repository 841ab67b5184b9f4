#!/bin/bash
export VCG_WATCHDOG_S=60
for args in "5000 0.02" "5000 0.025" "3000 0.03"; do
timeout 120 python tools/rgg_probe.py $args 2>&1 | tail -4
VCG_NO_RECLAIM=1 timeout 120 python tools/rgg_probe.py $args 2>&1 | tail -4
done
