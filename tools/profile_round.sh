#!/bin/bash
# Round profile capture (run under gpurun): bench line, ncu launch list, ncu
# --set full of the top kernels summarised to text on the box (the .ncu-rep
# files stay behind: gpurun brings back at most 64 MiB).
set -u
O=gpurun_out
mkdir -p $O /tmp/ncu
python bench.py > $O/r01_bench.json 2> $O/r01_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/r01_launches.csv \
    python bench.py --steps 1 --warmup 1 --nrhs-big 0 --no-residual --no-cpu-baseline > /tmp/ncu/launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_id_level --launch-skip 14 --launch-count 1 \
    -o /tmp/ncu/id python tools/compress_once.py > /tmp/ncu/id.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_factor_level --launch-skip 0 --launch-count 6 \
    -o /tmp/ncu/fac python tools/compress_once.py > /tmp/ncu/fac.log 2>&1
# R=16: the largest finest-level down-sweep bucket (14176 boxes; launch 110
# of the first, eager solve's 112 k_level_dmma_few launches)
ncu --set full --import-source on --clock-control none -k regex:k_level_dmma_few --launch-skip 110 --launch-count 1 \
    -o /tmp/ncu/sweep python tools/solvebench.py 1048576 16 1 > /tmp/ncu/sweep.log 2>&1
# R=1024: the largest finest-level down-sweep bucket of the pipelined DMMA kernel
ncu --set full --import-source on --clock-control none -k regex:k_level_dmma_pipe --launch-skip 110 --launch-count 1 \
    -o /tmp/ncu/sweep1024 python tools/solvebench.py 1048576 1024 1 > /tmp/ncu/sweep1024.log 2>&1
for r in id fac sweep sweep1024; do
  python tools/ncu_summary.py /tmp/ncu/$r.ncu-rep > $O/r01_ncu_${r}.txt 2>&1
  python tools/ncu_lines.py /tmp/ncu/$r.ncu-rep 25 > $O/r01_ncu_${r}_lines.txt 2>&1
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > $O/r01_ncu_${r}_raw.csv 2>&1
done
ls -la $O
