# ad-hoc GPU session script (run under gpurun from the repo root)
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -2 gpurun_out/r2_smoke.log
[ $rc -eq 0 ] || exit 1
timeout 240 python tools/eqcheck.py 20 1e-12 2 > gpurun_out/r2_eqcheck.log 2>&1; echo "eqcheck rc=$?"
tail -2 gpurun_out/r2_eqcheck.log
timeout 240 python tools/idprof.py 4 > gpurun_out/r2_idprof.log 2>&1; echo "idprof rc=$?"
cat gpurun_out/r2_idprof.log
SKEL_HOST_TIMING=1 timeout 120 python tools/compress_once.py > gpurun_out/r2_hosttiming.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?"
tail -6 gpurun_out/r2_gputest.log
timeout 400 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2_bench.log | cut -c1-400
timeout 600 bash tools/prof_id.sh r02b 8; echo "prof rc=$?"
