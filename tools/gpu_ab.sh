# A/B session (run under gpurun): previous build (tools/ab/libskel_head.so) vs the working tree
mkdir -p gpurun_out
for v in new head new head; do
  case $v in
    head) export SKEL_LIB=$PWD/tools/ab/libskel_head.so;;
    new) unset SKEL_LIB;;
  esac
  timeout 300 python tools/idprof.py 5 > gpurun_out/ab_idprof_$v.log 2>&1; echo "$v idprof rc=$?"; grep -E "compress only|union|histogram" gpurun_out/ab_idprof_$v.log
done
