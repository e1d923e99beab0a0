#!/bin/bash
# ncu capture of the first k_factor_level launches (level 0 buckets)
set -u
O=gpurun_out
TAG=${1:-r02}
mkdir -p $O /tmp/ncu
ncu -f --set full --import-source on --clock-control none -k regex:k_factor_level --launch-skip 0 --launch-count ${2:-4} \
    -o /tmp/ncu/fac python tools/compress_once.py > /tmp/ncu/fac.log 2>&1
python tools/ncu_summary.py /tmp/ncu/fac.ncu-rep > $O/${TAG}_ncu_fac.txt 2>&1
python tools/ncu_lines.py /tmp/ncu/fac.ncu-rep 40 > $O/${TAG}_ncu_fac_lines.txt 2>&1
tail -2 /tmp/ncu/fac.log
