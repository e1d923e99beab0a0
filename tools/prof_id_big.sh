#!/bin/bash
# ncu --set full of the LARGEST level-0 k_id_level bucket (launch 14 of the
# compression sweep: ~11k boxes, the 76 KB shared-memory class) -- run under gpurun
set -u
O=gpurun_out
TAG=${1:-r02}
mkdir -p $O /tmp/ncu
ncu -f --set full --import-source on --clock-control none -k regex:k_id_level --launch-skip ${2:-14} --launch-count 1 \
    -o /tmp/ncu/idbig python tools/compress_once.py > /tmp/ncu/idbig.log 2>&1
python tools/ncu_summary.py /tmp/ncu/idbig.ncu-rep > $O/${TAG}_ncu_idbig.txt 2>&1
python tools/ncu_lines.py /tmp/ncu/idbig.ncu-rep 60 > $O/${TAG}_ncu_idbig_lines.txt 2>&1
tail -3 /tmp/ncu/idbig.log
cat $O/${TAG}_ncu_idbig.txt
