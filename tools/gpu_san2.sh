# compute-sanitizer evidence (run under gpurun, 1 GPU): memcheck + synccheck of the
# config-1 pipeline (2-CTA cluster / DSMEM ID kernel, factor, DMMA sweeps, K6) and of the
# forced big-box path (grid-synchronised kernels of big.cu); `race` as $1 runs racecheck
# instead (separate call: racecheck is slow)
mkdir -p gpurun_out
T=${2:-r02}
if [ "${1:-mem}" = "race" ]; then
  timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 30 python tools/sanitize_run.py x 2048 > gpurun_out/${T}_san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -6 gpurun_out/${T}_san_racecheck.log
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 30 python tools/sanitize_run.py big 1024 > gpurun_out/${T}_san_racecheck_big.log 2>&1; echo "racecheck big rc=$?"; tail -6 gpurun_out/${T}_san_racecheck_big.log
  exit 0
fi
timeout 120 python tools/sanitize_run.py > gpurun_out/${T}_san_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/${T}_san_plain.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/${T}_san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/${T}_san_memcheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py big > gpurun_out/${T}_san_memcheck_big.log 2>&1; echo "memcheck big rc=$?"; tail -4 gpurun_out/${T}_san_memcheck_big.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/${T}_san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/${T}_san_synccheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_run.py big > gpurun_out/${T}_san_synccheck_big.log 2>&1; echo "synccheck big rc=$?"; tail -4 gpurun_out/${T}_san_synccheck_big.log
