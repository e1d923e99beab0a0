# A/B session (run under gpurun): HEAD library vs the working tree, and the 256-thread switch
mkdir -p gpurun_out
for v in head new t256; do
  case $v in
    head) export SKEL_LIB=$PWD/tools/ab/libskel_head.so; unset SKEL_ID_T256;;
    new) unset SKEL_LIB; unset SKEL_ID_T256;;
    t256) unset SKEL_LIB; export SKEL_ID_T256=1;;
  esac
  timeout 300 python tools/idprof.py 4 > gpurun_out/ab_idprof_$v.log 2>&1; echo "$v idprof rc=$?"; cat gpurun_out/ab_idprof_$v.log
  timeout 300 python tools/idphase.py > gpurun_out/ab_idphase_$v.log 2>&1; echo "$v idphase rc=$?"; cat gpurun_out/ab_idphase_$v.log
done
