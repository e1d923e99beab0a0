mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -eq 0 ] || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_factor_level|k_id_level" --csv --log-file gpurun_out/r2_fac_launches.csv python tools/compress_once.py > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/r2_fac_launches.csv | head -4
timeout 300 python tools/overlap.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bigbox.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
