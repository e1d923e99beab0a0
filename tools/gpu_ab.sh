# A/B session (run under gpurun): HEAD library vs the working tree
mkdir -p gpurun_out
for v in new head; do
  case $v in
    head) export SKEL_LIB=$PWD/tools/ab/libskel_head.so;;
    new) unset SKEL_LIB;;
  esac
  timeout 300 python tools/idprof.py 4 > gpurun_out/ab_idprof_$v.log 2>&1; echo "$v idprof rc=$?"; cat gpurun_out/ab_idprof_$v.log
done
unset SKEL_LIB
timeout 300 python tools/solvebench.py 1048576 16,4 20 2>&1 | grep "^R="
