mkdir -p gpurun_out
timeout 300 python tools/busy.py > gpurun_out/busy_async.log 2>&1; echo "rc=$?"; cat gpurun_out/busy_async.log
SKEL_SYNC_FACTOR=1 timeout 300 python tools/busy.py > gpurun_out/busy_sync.log 2>&1; echo "rc=$?"; cat gpurun_out/busy_sync.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_async.json 2> gpurun_out/bench_async.err; echo "bench rc=$?"; cut -c1-330 gpurun_out/bench_async.json
SKEL_SYNC_FACTOR=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_sync.json 2> gpurun_out/bench_sync.err; echo "bench rc=$?"; cut -c1-330 gpurun_out/bench_sync.json
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/async_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/async_gputest.log
