# factor-kernel A/B (run under gpurun): parity tests touching the factor, then timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_formats.py tests/test_shard.py -m gpu -x -q -p no:cacheprovider > gpurun_out/fac_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fac_tests.log
timeout 300 python tools/overlap.py > gpurun_out/fac_overlap.log 2>&1; echo "overlap rc=$?"; tail -4 gpurun_out/fac_overlap.log
SKEL_LIB=$PWD/tools/ab/libskel_head.so timeout 300 python tools/overlap.py > gpurun_out/fac_overlap_head.log 2>&1; echo "overlap head rc=$?"; tail -4 gpurun_out/fac_overlap_head.log
