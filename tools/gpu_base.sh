# baseline GPU session: smoke, gpu tests, default bench, launch list (run under gpurun)
mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/base_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -2 gpurun_out/base_smoke.log
[ $rc -eq 0 ] || exit 1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/base_gputest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/base_gputest.log
timeout 600 python bench.py > gpurun_out/base_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/base_bench.log | cut -c1-1500
timeout 600 bash tools/launch_list.sh base
