export VCG_LIB=$PWD/paper_2512_18334_b200/_build_tt/libvcgpu.so
WL=256 python tools/tail_probe.py rgg2000 > gpurun_out/tt256.log 2>&1
grep "^task" gpurun_out/tt256.log | sort -t= -k5 -n | tail -4
grep "k=1281" gpurun_out/tt256.log | tail -1
unset VCG_LIB
WL=256 python tools/tail_probe.py rgg2000 2>&1 | grep "k=1281" | tail -1
WL=128 python tools/tail_probe.py rgg2000 2>&1 | grep "k=1281" | tail -1
