#!/bin/bash
# A/B: the library in _build_old (VCG_LIB) vs the working tree's, same box
OLD=$PWD/paper_2512_18334_b200/_build_old/libvcgpu.so
for i in 1 2; do
echo "--- old"; VCG_LIB=$OLD python tools/pair_time.py
echo "--- new"; python tools/pair_time.py
done
echo "--- old"; VCG_LIB=$OLD python tools/strong_one.py 180 0.08 2>&1 | head -1
echo "--- new"; python tools/strong_one.py 180 0.08 2>&1 | head -1
