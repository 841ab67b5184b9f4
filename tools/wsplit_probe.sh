#!/bin/bash
export VCG_WATCHDOG_S=60
for wl in 64 128 256; do WL=$wl python tools/tail_probe.py 2>&1 | grep "k=" | awk 'NR%3==1' ; done
VCG_NO_WSPLIT=1 WL=128 python tools/tail_probe.py 2>&1 | grep "k=1281" | head -1
python tools/strong_one.py 180 0.08 | head -1
VCG_WATCHDOG_S=60 timeout 300 python tools/dense_probe.py gnp400 | tail -1
