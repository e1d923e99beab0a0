mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -eq 0 ] || exit 1
timeout 200 python tools/eqcheck.py 20 1e-12 1 2>&1 | tail -3
SKEL_ID_NOWIDE=1 timeout 200 python tools/eqcheck.py 20 1e-12 1 2>&1 | tail -3
