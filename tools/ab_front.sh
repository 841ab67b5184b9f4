# A/B of the root kernel: _build_old (a build of another commit) vs _build on
# the same box, ba100k and planted1m, twice interleaved
for i in 1 2; do for v in _build_old _build; do
  L=$PWD/paper_2512_18334_b200/$v/libvcgpu.so
  for w in ba100k planted1m; do echo "$v $w $(VCG_LIB=$L python tools/front_one.py $w 2>&1 | tail -1 | cut -c1-60)"; done
done; done
