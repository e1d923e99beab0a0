# memcheck + synccheck of the config-1 pipeline and the forced big-box path, and
# the current k_id_level line profile (run under gpurun; 1 GPU)
mkdir -p gpurun_out
timeout 120 python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/san_plain.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/san_memcheck.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py big > gpurun_out/san_memcheck_big.log 2>&1; echo "memcheck big rc=$?"; tail -4 gpurun_out/san_memcheck_big.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/san_synccheck.log
timeout 600 bash tools/prof_id.sh r02c 6; echo "prof rc=$?"; head -30 gpurun_out/r02c_ncu_id_lines.txt
