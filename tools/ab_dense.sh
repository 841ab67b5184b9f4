#!/bin/bash
# A/B of library builds on the dense instances (strong G(180, 0.08), gnp400)
for v in ${VARIANTS:-_build}; do
  L=$PWD/paper_2512_18334_b200/$v/libvcgpu.so
  echo "=== $v"
  VCG_LIB=$L python tools/strong_one.py 180 0.08 2>&1 | head -1
  VCG_LIB=$L python tools/strong_one.py 150 0.1 2>&1 | head -1
  VCG_LIB=$L BUDGET_S=3 python tools/dense_probe.py gnp400 2>&1 | grep "wl=-1"
done
