mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_formats.py tests/test_shard.py tests/test_gpu_bigbox.py -m gpu -x -q -p no:cacheprovider > gpurun_out/fac_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fac_tests.log
timeout 300 python tools/facprof.py > gpurun_out/facprof_new.log 2>&1; echo "rc=$?"; grep -E "^factor|union" gpurun_out/facprof_new.log
python bench.py --no-cpu-baseline --nrhs-big 0 --no-residual 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], d['value_steps'], 'e2e', d['e2e']['value'], 'fac union', d['roofline_factor']['union_ms_per_step'])"
