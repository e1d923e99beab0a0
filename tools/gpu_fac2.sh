mkdir -p gpurun_out
timeout 300 python tools/facprof.py > gpurun_out/facprof_new.log 2>&1; echo "rc=$?"; cat gpurun_out/facprof_new.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_formats.py -m gpu -x -q -p no:cacheprovider > gpurun_out/fac_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fac_tests.log
