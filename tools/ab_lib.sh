#!/bin/bash
# A/B of library builds (VARIANTS: _build dirs): rgg2000 PVC at warp limits
# 64 / 128 and the strong instance
for v in ${VARIANTS:-_build}; do
  L=$PWD/paper_2512_18334_b200/$v/libvcgpu.so
  echo "=== $v"
  VCG_LIB=$L WLS=${WLS:-64,128} EXPS=4 CHKS=3 python tools/rgg_sweep.py
  VCG_LIB=$L python tools/strong_one.py 180 0.08 2>&1 | head -1
done
