#!/bin/bash
# ncu capture of the level-0 k_id_level buckets (run under gpurun, 1 GPU):
# the summaries land in gpurun_out/ (the .ncu-rep stays on the box)
set -u
O=gpurun_out
TAG=${1:-r02}
mkdir -p $O /tmp/ncu
ncu -f --set full --import-source on --clock-control none -k regex:k_id_level --launch-skip 0 --launch-count ${2:-6} \
    -o /tmp/ncu/id python tools/compress_once.py > /tmp/ncu/id.log 2>&1
python tools/ncu_summary.py /tmp/ncu/id.ncu-rep > $O/${TAG}_ncu_id.txt 2>&1
python tools/ncu_lines.py /tmp/ncu/id.ncu-rep 40 > $O/${TAG}_ncu_id_lines.txt 2>&1
tail -3 /tmp/ncu/id.log
