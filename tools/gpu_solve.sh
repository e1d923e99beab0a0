mkdir -p gpurun_out
SKEL_SOLVE_PIPE=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_formats.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for b in 1 0; do
SKEL_SOLVE_PIPE=$b timeout 300 python tools/solvebench.py 1048576 16,4,2,32 20 > gpurun_out/solve_pipe$b.log 2>&1; echo "pipe=$b rc=$?"; grep "^R=" gpurun_out/solve_pipe$b.log
done
