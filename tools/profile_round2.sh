#!/bin/bash
# Round-2 capture (run under gpurun, 1 GPU): GPU tests, the bench line, the
# reference arm, the eager-solve ncu launch list, ncu --set full of the three
# top kernels summarised to text (the .ncu-rep files stay on the box).
set -u
O=gpurun_out
T=${1:-r02}
mkdir -p $O /tmp/ncu
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/${T}_gputest.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"; cut -c1-600 $O/${T}_bench.json
bash tools/launch_list.sh $T
ncu -f --set full --import-source on --clock-control none -k regex:k_id_level --launch-skip 0 --launch-count 6 \
    -o /tmp/ncu/id python tools/compress_once.py > /tmp/ncu/id.log 2>&1
ncu -f --set full --import-source on --clock-control none -k regex:k_factor_level --launch-skip 0 --launch-count 6 \
    -o /tmp/ncu/fac python tools/compress_once.py > /tmp/ncu/fac.log 2>&1
SKEL_SOLVE_GRAPH=0 ncu -f --set full --import-source on --clock-control none -k regex:k_level_dmma_few --launch-skip 110 --launch-count 1 \
    -o /tmp/ncu/sweep python tools/solvebench.py 1048576 16 1 > /tmp/ncu/sweep.log 2>&1
SKEL_SOLVE_GRAPH=0 ncu -f --set full --import-source on --clock-control none -k regex:k_level_dmma_pipe --launch-skip 110 --launch-count 1 \
    -o /tmp/ncu/sweep1024 python tools/solvebench.py 1048576 1024 1 > /tmp/ncu/sweep1024.log 2>&1
ncu -f --set full --import-source on --clock-control none -k regex:k_id_level --launch-skip 14 --launch-count 1 \
    -o /tmp/ncu/idbig python tools/compress_once.py > /tmp/ncu/idbig.log 2>&1
for r in id idbig fac sweep sweep1024; do
  python tools/ncu_summary.py /tmp/ncu/$r.ncu-rep > $O/${T}_ncu_${r}.txt 2>&1
  python tools/ncu_lines.py /tmp/ncu/$r.ncu-rep 30 > $O/${T}_ncu_${r}_lines.txt 2>&1
done
ls -la $O | head -40
