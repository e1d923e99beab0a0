#!/bin/bash
# ncu launch list (gpu__time_duration per kernel launch, cold-cache and
# serialised) of one bench step with the eager (non-graph) solve, so the
# profiled process exits 0 and every launch is timed; then a per-kernel
# summary.  Run under gpurun (1 GPU) only after bench.py itself ran clean.
set -u
O=gpurun_out
TAG=${1:-r02}
mkdir -p $O
SKEL_SOLVE_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 1 --nrhs-big 0 --no-residual --no-cpu-baseline > $O/${TAG}_launches.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py $O/${TAG}_launches.csv > $O/${TAG}_launches_summary.txt 2>&1
cat $O/${TAG}_launches_summary.txt | head -20
