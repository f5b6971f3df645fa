#!/bin/bash
# Every BASELINE config end to end on one B200 with the final round's defaults, both engines
# where they differ (DMMA dataflow worker / tcgen05 Ozaki engine, CC_EXEC flags bit 6).
set -u
run() { echo "== $*"; timeout -s KILL 600 python tools/run_config.py "$@" 2>&1 | grep -E "^c[0-9]|^part|^execute 1|^  "; }
run c3
run c3 --ozaki
run c4
run c4 --next-use
run c4 --next-use --ozaki --breakdown
run c5 --N 256 --arena-gb 140
run c5 --N 256 --arena-gb 140 --ozaki
run c5 --N 512 --parts 8 --part 0 --device-leaves --arena-gb 80
run c5 --N 512 --parts 8 --part 0 --device-leaves --arena-gb 80 --ozaki --breakdown
run c5 --N 1024 --parts 16 --part 0 --device-leaves --arena-gb 140
run c5 --N 1024 --parts 16 --part 0 --device-leaves --arena-gb 140 --ozaki --breakdown
