mkdir -p gpurun_out
timeout 300 python tools/solvebench.py 1048576 16,4,1,32 20 > gpurun_out/solve_new.log 2>&1; echo "rc=$?"; grep "^R=" gpurun_out/solve_new.log
SKEL_LIB=$PWD/tools/ab/libskel_head.so timeout 300 python tools/solvebench.py 1048576 16,4,1,32 20 > gpurun_out/solve_head.log 2>&1; echo "rc=$?"; grep "^R=" gpurun_out/solve_head.log
