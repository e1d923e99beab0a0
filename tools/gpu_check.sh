# full check (run under gpurun): GPU tests, bench line, busy fraction
mkdir -p gpurun_out
T=${1:-r02d}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_gputest.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/${T}_bench.json
timeout 300 python tools/busy.py > gpurun_out/${T}_busy.log 2>&1; cat gpurun_out/${T}_busy.log
