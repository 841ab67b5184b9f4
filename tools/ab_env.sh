#!/bin/bash
# A/B of an environment knob on the same build: rgg2000 PVC pair (warp limit
# 64), strong G(180, 0.08), gnp400 -- "$@" are the B-side assignments
for i in 1 2; do
  echo "--- A"; WLS=64 EXPS=4 CHKS=3 python tools/rgg_sweep.py; python tools/strong_one.py 180 0.08 2>&1 | head -1
  echo "--- B $*"; env "$@" WLS=64 EXPS=4 CHKS=3 python tools/rgg_sweep.py; env "$@" python tools/strong_one.py 180 0.08 2>&1 | head -1
done
